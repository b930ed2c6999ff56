set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash scripts/planclk.sh
WS_SERIAL=1 python scripts/probe_one.py > gpurun_out/probe_one.log 2>&1
WS_SERIAL=1 python scripts/probe.py configs1 > gpurun_out/probe_serial.log 2>&1
python scripts/probe.py configs1 > gpurun_out/probe_conc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_(plan|rows|fold|model)$" -s 8 -c 4 -o gpurun_out/full2 python scripts/ncu_target.py > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_full2.log
