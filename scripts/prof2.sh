timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_(plan|rows|fold|model|scan)$" -s 10 -c 5 -o gpurun_out/full3 python scripts/ncu_target.py > gpurun_out/ncu_full3.log 2>&1
tail -2 gpurun_out/ncu_full3.log
