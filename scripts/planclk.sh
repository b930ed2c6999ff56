cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
cp scripts/variants/planclk.so paper_2204_14242_b200/libwsb200.so
WS_SERIAL=1 python scripts/probe_one.py > gpurun_out/planclk.log 2>&1
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
grep PLANCLK gpurun_out/planclk.log | sort | uniq -c | sort -rn | head -30
