#!/bin/bash
# latency-mode M2L: parity subset, batch sweep, then one full ncu capture of
# each latency kernel (after the plain run exits 0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "cfg1 or dropin or permuted" 2>&1 | tail -3
timeout 300 python tools/lat_m2l.py exact > gpurun_out/lat.json 2>&1 && cat gpurun_out/lat.json &&
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"m2l_terms|m2l_reduce" -c 2 \
   -o gpurun_out/lat_full -f python tools/lat_m2l.py exact > gpurun_out/lat_full.log 2>&1; echo ncu rc=$?
