cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
for v in /tmp/base.so scripts/variants/ev3.so /tmp/base.so; do cp $v paper_2204_14242_b200/libwsb200.so; echo "== $v"; python scripts/sim_time.py; done
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
