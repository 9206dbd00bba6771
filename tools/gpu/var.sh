cp paper_2112_01743_b200/lib/libchebpr_b200.so /tmp/prod.so
for v in build/variants/*.so; do
  cp "$v" paper_2112_01743_b200/lib/libchebpr_b200.so
  for c in ${CONFIGS:-c2 c3 c4}; do timeout 300 python tools/term_time.py $c "$(basename $v)"; done
done > gpurun_out/var.log 2>&1
cp /tmp/prod.so paper_2112_01743_b200/lib/libchebpr_b200.so
