python bench.py --steps 1500 --no-next --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print(d['value'],d['ms_per_step'],d['e2e'])"
tail -3 gpurun_out/bench_quick.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/rank_target.py 100000 2>/dev/null | grep -E "k_rank" | tail -4
