set -x
# round-end style GPU check: smoke, GPU parity tests (incl. the full-space golden sets), bench (both
# arms), launch list, ncu full of the top kernels of one estimate
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
python bench.py --impl reference > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-next > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_(plan|rows|fold|scan|spairs|smset|cplan|cplanes|cfold|sclass|instr|warp|wclass|model)$" -s 28 -c 14 -o gpurun_out/full python scripts/ncu_target.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
