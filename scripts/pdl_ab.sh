# A/B of programmatic dependent launch (WS_PDL=0/1) on every probe workload
mkdir -p gpurun_out
{
for r in 1 2; do
for p in 0 1; do echo "=== WS_PDL=$p"; WS_PDL=$p python scripts/probe.py 2>&1 | grep " step "; done
done
} > gpurun_out/pdl.log 2>&1
