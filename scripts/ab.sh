#!/bin/bash
# A/B timing of library variants (scripts/variants/*.so) against the in-tree build
cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
for v in /tmp/base.so scripts/variants/*.so; do
  cp $v paper_2204_14242_b200/libwsb200.so
  echo "=== $v"; WS_SERIAL=1 python scripts/probe.py 2>&1 | sed -n '1p;8p'; python scripts/probe.py 2>&1 | grep configs1
done
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
