#!/bin/bash
# A/B the batched exact M2L over library variants paper_2210_06439_b200/libsg_*.so
# (timing + output digest at levels 4 and 3, order 1)
cp paper_2210_06439_b200/libsg.so /tmp/libsg_cur.so
for f in /tmp/libsg_cur.so paper_2210_06439_b200/libsg_*.so; do
  cp $f paper_2210_06439_b200/libsg.so
  echo "$f $(python tools/m2l_time.py 4 7 1) $(python tools/m2l_time.py 3 7 1)"
done
cp /tmp/libsg_cur.so paper_2210_06439_b200/libsg.so
