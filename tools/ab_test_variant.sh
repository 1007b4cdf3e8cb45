#!/bin/bash
# run the GPU parity suite against each libsg_*.so variant, then A/B them
cp paper_2210_06439_b200/libsg.so /tmp/libsg_orig.so
for f in paper_2210_06439_b200/libsg_*.so; do
  cp $f paper_2210_06439_b200/libsg.so
  echo "$f $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
done
cp /tmp/libsg_orig.so paper_2210_06439_b200/libsg.so
bash tools/ab_both.sh
