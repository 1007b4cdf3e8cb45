#!/bin/bash
# A/B the libsg_*.so variants in-tree twice, interleaved (time_kernels L=4)
cp paper_2210_06439_b200/libsg.so /tmp/libsg_orig.so
for rep in 1 2; do
  for f in paper_2210_06439_b200/libsg_*.so; do
    cp $f paper_2210_06439_b200/libsg.so
    echo "$f $(python tools/time_kernels.py 4 5)"
  done
done
cp /tmp/libsg_orig.so paper_2210_06439_b200/libsg.so
