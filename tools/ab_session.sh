# ad-hoc A/B session (edited per experiment): guarded exact half-step FMA
# in the fused hydro states (default build) vs without (libsg_hf0.so)
python -m pytest tests -m gpu -q > gpurun_out/tests_ab.log 2>&1; tail -1 gpurun_out/tests_ab.log
bash tools/ab_hydro_libs.sh 4
bash tools/ab_hydro_libs.sh 4
bash tools/ab_hydro_libs.sh 3
