#!/bin/bash
# GPU session: remaining gpu tests, then ncu captures (each after a clean plain run)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} 2>&1 | tail -15
python tools/prof_kernels.py all > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"m2l_kernel|p2p_kernel|reconstruct_kernel|flux_kernel" -s 4 -c 4 \
     -o gpurun_out/prof_r1 -f python tools/prof_kernels.py all > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 120 --csv \
     --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
tail -3 gpurun_out/ncu_full.log
