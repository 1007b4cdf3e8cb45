#!/bin/bash
# A/B the latency-mode M2L over library variants paper_2210_06439_b200/libsg_*.so
# (one-CTA and two-CTA-cluster forms; trimmed-mean event timing)
cp paper_2210_06439_b200/libsg.so /tmp/libsg_cur.so
for f in /tmp/libsg_cur.so paper_2210_06439_b200/libsg_*.so; do
  cp $f paper_2210_06439_b200/libsg.so
  for v in 0 1; do
    echo "$f split=$v $(SG_M2L_FL_SPLIT=$v python tools/lat_m2l.py) $(SG_M2L_FL_SPLIT=$v python tools/c1_m2l.py)"
  done
done
cp /tmp/libsg_cur.so paper_2210_06439_b200/libsg.so
