# A/B: k_rows minimum CTAs per SM (register cap) on BJ configs[1] and LBM15, concurrent step + serial k_rows
cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
for v in /tmp/base.so scripts/variants/rminb2.so scripts/variants/rminb4.so /tmp/base.so scripts/variants/rminb2.so scripts/variants/rminb4.so; do
  cp $v paper_2204_14242_b200/libwsb200.so
  echo "=== $v"
  python scripts/probe.py configs1 lbm15 2>&1 | grep "n="
  WS_SERIAL=1 python scripts/probe.py configs1 2>&1 | grep -E "k_rows"
done
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
