#!/bin/bash
# A/B timing of library variants: python scripts/probe.py with each .so swapped in
set -e
cp paper_2204_14242_b200/libwsb200.so /tmp/base.so
for v in /tmp/base.so scripts/variants/*.so; do
  cp $v paper_2204_14242_b200/libwsb200.so
  echo "=== $v"; python scripts/probe.py 2>&1 | head -11
done
cp /tmp/base.so paper_2204_14242_b200/libwsb200.so
