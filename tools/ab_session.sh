# ad-hoc A/B session (edited per experiment): GPU tests on the default build,
# then the fused hydro of every libsg_*.so variant vs the default
python -m pytest tests -m gpu -q > gpurun_out/tests_ab.log 2>&1; tail -2 gpurun_out/tests_ab.log
bash tools/ab_hydro_libs.sh 4
bash tools/ab_hydro_libs.sh 3
