# A/B of library builds (scripts/variants/*.so) against the in-tree build: serial k_rows and the concurrent step
cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
for v in /tmp/base.so scripts/variants/old.so scripts/variants/contig.so /tmp/base.so scripts/variants/old.so scripts/variants/contig.so; do
  cp $v paper_2204_14242_b200/libwsb200.so
  echo "=== $v"
  python scripts/probe.py configs1 2>&1 | head -1
  python scripts/probe.py lbm15 2>&1 | head -1
  WS_SERIAL=1 python scripts/probe.py configs1 2>&1 | grep -E "k_rows|k_fold"
done
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
