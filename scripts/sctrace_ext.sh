cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
cp scripts/variants/sctrace.so paper_2204_14242_b200/libwsb200.so
WS_SERIAL=1 python scripts/probe_ext_trace.py > gpurun_out/sctrace_ext.log 2>&1
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
grep -c SCITEM gpurun_out/sctrace_ext.log
