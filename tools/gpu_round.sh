#!/bin/bash
# Full GPU session: gpu tests, smoke, default bench, its ncu launch list, and
# ncu --set full captures of M2L and the fused hydro kernel at level 4.
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/tests_$TAG.log 2>&1; tail -2 gpurun_out/tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json
if [ -z "$SKIP_NCU" ]; then
python bench.py --no-cpu > gpurun_out/bench_plain_$TAG.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
python tools/prof_kernels.py gravity 4 > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"m2l_pair|p2p_" -s 2 -c 2 \
    -o gpurun_out/prof_m2l_$TAG -f python tools/prof_kernels.py gravity 4 > gpurun_out/ncu_m2l.log 2>&1; echo "ncu m2l rc=$?"
python tools/prof_kernels.py gravity 4 fma > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:m2l_mirror -s 1 -c 1 \
    -o gpurun_out/prof_m2lfma_$TAG -f python tools/prof_kernels.py gravity 4 fma > gpurun_out/ncu_m2lfma.log 2>&1; echo "ncu m2l fma rc=$?"
python tools/prof_kernels.py hydro 4 > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hydro_dedup|reconstruct_kernel|flux_kernel|p2p_kernel" -s 0 -c 4 \
    -o gpurun_out/prof_hydro_$TAG -f python tools/prof_kernels.py hydro 4 > gpurun_out/ncu_hydro.log 2>&1; echo "ncu hydro rc=$?"
fi
