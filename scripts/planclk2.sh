cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
cp scripts/variants/planclk.so paper_2204_14242_b200/libwsb200.so
WS_SERIAL=1 python scripts/probe.py lbm15 > gpurun_out/planclk_lbm15.log 2>&1
WS_SERIAL=1 python scripts/probe.py configs1 > gpurun_out/planclk_k25.log 2>&1
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
grep PLANCLK gpurun_out/planclk_lbm15.log | tail -4; grep PLANCLK gpurun_out/planclk_k25.log | tail -4
