#!/bin/bash
# A/B the libsg_*.so variants (time_kernels L=4) in both precisions, interleaved x2
cp paper_2210_06439_b200/libsg.so /tmp/libsg_orig.so
for rep in 1 2; do
  for f in paper_2210_06439_b200/libsg_*.so; do
    cp $f paper_2210_06439_b200/libsg.so
    echo "$f exact $(python tools/time_kernels.py 4 5 exact 2>&1 | tail -1)"
    echo "$f fma   $(python tools/time_kernels.py 4 5 fma 2>&1 | tail -1)"
  done
done
cp /tmp/libsg_orig.so paper_2210_06439_b200/libsg.so
