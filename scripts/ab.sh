#!/bin/bash
# A/B timing of library variants (scripts/variants/*.so) against the in-tree build on BJ configs[1]
cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
for v in /tmp/base.so scripts/variants/*.so; do
  cp $v paper_2204_14242_b200/libwsb200.so
  echo "=== $v"
  for i in 1 2; do python scripts/probe.py configs1 2>&1 | head -1; done
  WS_SERIAL=1 python scripts/probe.py configs1 2>&1 | grep -E "k_rows|k_sclass"
done
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
