# ad-hoc A/B session (edited per experiment): exact FMA direction products
# (default build) vs the separate mul/add (libsg_df0.so): GPU tests, fused
# hydro and the unfused reconstruct
python -m pytest tests -m gpu -q > gpurun_out/tests_ab.log 2>&1; tail -1 gpurun_out/tests_ab.log
bash tools/ab_hydro_libs.sh 4
bash tools/ab_hydro_libs.sh 4
cp paper_2210_06439_b200/libsg.so /tmp/new.so
for lib in /tmp/new.so paper_2210_06439_b200/libsg_df0.so; do
cp $lib paper_2210_06439_b200/libsg.so; echo "$lib $(python tools/time_kernels.py 4 10)"
done
cp /tmp/new.so paper_2210_06439_b200/libsg.so
