# NEXT-2 on-box validation, LBM15 workload (scripts/validate_next2.py with WS_VALIDATE=lbm15)
set -x
export WS_VALIDATE=lbm15
python scripts/validate_next2.py --time gpurun_out/v2l_time.json
timeout 1200 ncu --metrics gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_lbm15 --csv --log-file gpurun_out/v2l_ncu.csv python scripts/validate_next2.py --ncu-pass > gpurun_out/v2l_ncu.log 2>&1
python scripts/validate_next2.py --analyze gpurun_out/v2l_time.json gpurun_out/v2l_ncu.csv gpurun_out/r01_next2_lbm15_validation
