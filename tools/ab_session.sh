# ad-hoc A/B session (edited per experiment): latency-mode M2L with two
# ordered chains per consumer lane (default build) vs one (libsg_tc0.so)
python -m pytest tests -m gpu -q > gpurun_out/tests_ab.log 2>&1; tail -1 gpurun_out/tests_ab.log
cp paper_2210_06439_b200/libsg.so /tmp/new.so
for i in 1 2; do
for lib in /tmp/new.so paper_2210_06439_b200/libsg_tc0.so; do
cp $lib paper_2210_06439_b200/libsg.so
echo "$lib $(python tools/lat_m2l.py 2>/dev/null | tail -1)"
done
done
cp /tmp/new.so paper_2210_06439_b200/libsg.so
python tools/lat_m2l_b2b.py 2>&1 | tail -2
