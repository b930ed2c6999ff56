cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
cp scripts/variants/sctrace.so paper_2204_14242_b200/libwsb200.so
WS_SERIAL=1 python scripts/probe.py configs0 > gpurun_out/sctrace_c0.log 2>&1
WS_SERIAL=1 python scripts/probe.py lbm15 > gpurun_out/sctrace_lbm15.log 2>&1
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
grep -c SCITEM gpurun_out/sctrace_c0.log gpurun_out/sctrace_lbm15.log
