#!/bin/bash
# A/B the fused hydro over library variants paper_2210_06439_b200/libsg_*.so
# (each built with different -D options): time + bit-identity vs the
# round-1 rebuild kernel, at level ${1:-4}
cp paper_2210_06439_b200/libsg.so /tmp/libsg_orig.so
for f in /tmp/libsg_orig.so paper_2210_06439_b200/libsg_*.so; do
  cp $f paper_2210_06439_b200/libsg.so
  echo "$f $(python tools/ab_hydro.py ${1:-4} 10)"
done
cp /tmp/libsg_orig.so paper_2210_06439_b200/libsg.so
