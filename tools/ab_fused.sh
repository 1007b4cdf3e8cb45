#!/bin/bash
# A/B variants of libsg: swap the library, time kernels
cp paper_2210_06439_b200/libsg.so /tmp/libsg_orig.so
for f in paper_2210_06439_b200/libsg_*.so; do
  cp $f paper_2210_06439_b200/libsg.so
  echo "$f"; python tools/time_kernels.py 4 5
done
cp /tmp/libsg_orig.so paper_2210_06439_b200/libsg.so
