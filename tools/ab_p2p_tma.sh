#!/bin/bash
# A/B: P2P cube staging: double-buffered TMA (default), single-buffer TMA, S^3 cp.async requests
for L in 4 3; do
  for e in "" "SG_P2P_TMA_SINGLE=1" "SG_P2P_NO_TMA=1"; do
    for prec in exact fma; do
      echo "L=$L ${e:-tma2} $prec $(env $e python tools/time_kernels.py $L 7 $prec | python -c 'import json,sys; print(json.load(sys.stdin)["p2p"])')"
    done
  done
done
