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
