#!/bin/bash
# A/B: exact M2L, mirror-paired vs one-target kernel (timing + output digest)
for L in 4 3; do for o in 1 0; do
  python tools/m2l_time.py $L 7 $o
  SG_M2L_ONE_TARGET=1 python tools/m2l_time.py $L 7 $o
done; done
