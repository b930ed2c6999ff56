# development GPU check: parity tests, per-kernel probe (serial + concurrent), a short headline bench
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
WS_SERIAL=1 python scripts/probe.py configs1 > gpurun_out/probe_serial.log 2>&1
python scripts/probe.py > gpurun_out/probe_conc.log 2>&1
cat gpurun_out/probe_serial.log gpurun_out/probe_conc.log
python bench.py --steps 1500 --no-next --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['configs3_strong']['value'])"
WS_SERIAL=1 python scripts/probe.py configs0 lbm15 > gpurun_out/probe_serial2.log 2>&1; cat gpurun_out/probe_serial2.log
