cp paper_2112_01743_b200/lib/libchebpr_b200.so /tmp/prod.so
for v in build/variants/*.so; do
  cp "$v" paper_2112_01743_b200/lib/libchebpr_b200.so
  for p in 64 32; do echo "== $(basename $v) fp$p"; timeout 300 python tools/batch_time.py c5 $p 2>&1 | tail -2; done
done > gpurun_out/var5.log 2>&1
cp /tmp/prod.so paper_2112_01743_b200/lib/libchebpr_b200.so
