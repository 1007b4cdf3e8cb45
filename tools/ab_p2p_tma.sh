#!/bin/bash
# A/B: P2P cube staging by one TMA tile copy vs S^3 cp.async requests
for L in 4 3; do
  echo "L=$L tma $(python tools/time_kernels.py $L 7 | python -c 'import json,sys; print(json.load(sys.stdin)["p2p"])') cp.async $(SG_P2P_NO_TMA=1 python tools/time_kernels.py $L 7 | python -c 'import json,sys; print(json.load(sys.stdin)["p2p"])')"
done
