# BJ configs[4] / fig:sizescan on one B200 (scripts/sizescan.py)
set -x
python scripts/sizescan.py --time gpurun_out/ss_time.json
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_st25 --csv --log-file gpurun_out/ss_ncu.csv python scripts/sizescan.py --ncu-pass > gpurun_out/ss_ncu.log 2>&1
python scripts/sizescan.py --analyze gpurun_out/ss_time.json gpurun_out/ss_ncu.csv gpurun_out/r01_configs4_sizescan
