#!/bin/bash
# ncu --set full on one kernel of tools/prof_kernels.py: PROF_WHAT (gravity|hydro) PROF_K (regex) PROF (name)
mkdir -p gpurun_out
python tools/prof_kernels.py ${PROF_WHAT:-gravity} ${PROF_LEVEL:-3} ${PROF_PREC:-exact} > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${PROF_K}" -s ${PROF_S:-1} -c 1 \
     -o gpurun_out/${PROF} -f python tools/prof_kernels.py ${PROF_WHAT:-gravity} ${PROF_LEVEL:-3} ${PROF_PREC:-exact} > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_full.log
