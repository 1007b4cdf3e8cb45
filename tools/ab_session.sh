# ad-hoc A/B session (edited per experiment): tests, then per-kernel timings
# of libsg_old.so (previous build) vs the current libsg.so
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/tests_ab.log 2>&1; tail -3 gpurun_out/tests_ab.log
cp paper_2210_06439_b200/libsg.so /tmp/new.so
for i in 1 2; do
cp paper_2210_06439_b200/libsg_old.so paper_2210_06439_b200/libsg.so; python tools/time_kernels.py 4 10
cp /tmp/new.so paper_2210_06439_b200/libsg.so; python tools/time_kernels.py 4 10
done
python tools/dropin_breakdown.py
