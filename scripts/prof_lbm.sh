mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_(fold|rows|plan)$" -s 6 -c 3 -o gpurun_out/lbm python scripts/ncu_target.py lbm15 > gpurun_out/ncu_lbm.log 2>&1
tail -2 gpurun_out/ncu_lbm.log
