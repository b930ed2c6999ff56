"""Plain CPU definition of the NEXT-2 validation kernel (TEST INFRASTRUCTURE ONLY).

The 3D-25pt range-4 FP64 star stencil of P:751-764: for every cell of the domain
[4, n+4)^3 of an (n+8)^3 field, dst = w0 * src + sum_{k=1..4} w_k * (the six neighbours at
distance k along x, y, z).  Weights as the library's (include/ws.h ws_validate_stencil25).
numpy, float64, no blocking: the cell loop is the array expression itself.
"""
import numpy as np

W = (-7.5, 1.6, -0.2, 0.025, -0.0017857142857142857)


def stencil25(src, n):
    """src: (nz+8, ny+8, nx+8) float64 array (z slowest); returns dst with the domain filled
    and the ghost layers untouched (zero)."""
    nx, ny, nz = n
    dst = np.zeros_like(src)
    c = (slice(4, nz + 4), slice(4, ny + 4), slice(4, nx + 4))
    v = W[0] * src[c]
    for k in range(1, 5):
        acc = (src[4:nz + 4, 4:ny + 4, 4 - k:nx + 4 - k] + src[4:nz + 4, 4:ny + 4, 4 + k:nx + 4 + k] +
               src[4:nz + 4, 4 - k:ny + 4 - k, 4:nx + 4] + src[4:nz + 4, 4 + k:ny + 4 + k, 4:nx + 4] +
               src[4 - k:nz + 4 - k, 4:ny + 4, 4:nx + 4] + src[4 + k:nz + 4 + k, 4:ny + 4, 4:nx + 4])
        v = v + W[k] * acc
    dst[c] = v
    return dst


# D3Q15 in the estimator's order (workloads.D3Q15): rest, 6 faces, 8 corners
Q15 = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)] + \
      [(x, y, z) for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)]


def lbm15(src, phi, n):
    """Plain definition of the LBM15 validation kernel: per cell of the
    domain [1, n+1)^3 of (n+2)^3 arrays, pull f_q = src_q(cell - c_q); rho, j = sum f_q (1, c_q);
    lap = 7-point Laplacian of phi; omega = 1.2 + 0.1 phi; feq_q = w_q (rho + 3 c_q.j) + w_q 0.05 lap;
    dst_q = f_q + omega (feq_q - f_q); fd = lap.  src: (15, nz+2, ny+2, nx+2); phi: (nz+2, ny+2, nx+2).
    Returns (dst, fd) with ghost layers zero."""
    nx, ny, nz = n
    dom = (slice(1, nz + 1), slice(1, ny + 1), slice(1, nx + 1))

    def sh(a, dx, dy, dz):   # a(cell + (dx, dy, dz)) over the domain
        return a[1 + dz:nz + 1 + dz, 1 + dy:ny + 1 + dy, 1 + dx:nx + 1 + dx]
    f = [sh(src[q], -c[0], -c[1], -c[2]) for q, c in enumerate(Q15)]
    rho = sum(f)
    jx = sum(c[0] * f[q] for q, c in enumerate(Q15))
    jy = sum(c[1] * f[q] for q, c in enumerate(Q15))
    jz = sum(c[2] * f[q] for q, c in enumerate(Q15))
    p0 = phi[dom]
    lap = sh(phi, 1, 0, 0) + sh(phi, -1, 0, 0) + sh(phi, 0, 1, 0) + sh(phi, 0, -1, 0) + \
        sh(phi, 0, 0, 1) + sh(phi, 0, 0, -1) - 6.0 * p0
    omega, g = 1.2 + 0.1 * p0, 0.05 * lap
    dst = np.zeros_like(src)
    for q, c in enumerate(Q15):
        w = 2.0 / 9.0 if q == 0 else (1.0 / 9.0 if q < 7 else 1.0 / 72.0)
        feq = w * (rho + 3.0 * (c[0] * jx + c[1] * jy + c[2] * jz)) + w * g
        dst[q][dom] = f[q] + omega * (feq - f[q])
    fd = np.zeros_like(phi)
    fd[dom] = lap
    return dst, fd
