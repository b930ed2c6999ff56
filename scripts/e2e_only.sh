python bench.py --steps 1500 --no-next --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print(d['value'],d['ms_per_step'],d['e2e'], d['configs3_strong']['value'])"
tail -3 gpurun_out/bench_quick.err
