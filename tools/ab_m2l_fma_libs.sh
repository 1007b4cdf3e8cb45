cp paper_2210_06439_b200/libsg.so /tmp/libsg_cur.so
for f in /tmp/libsg_cur.so paper_2210_06439_b200/libsg_old.so; do
  cp $f paper_2210_06439_b200/libsg.so
  echo "$f $(python tools/time_kernels.py 4 5 fma | python -c 'import json,sys; d=json.load(sys.stdin); print(d["m2l"])')"
done
cp /tmp/libsg_cur.so paper_2210_06439_b200/libsg.so
