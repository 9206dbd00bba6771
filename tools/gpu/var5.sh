cp paper_2112_01743_b200/lib/libchebpr_b200.so /tmp/prod.so
for rep in 1 2 3; do
for v in build/variants/*.so; do
  cp "$v" paper_2112_01743_b200/lib/libchebpr_b200.so
  for p in ${PRECS:-64}; do echo "== $(basename $v) fp$p rep$rep $(nvidia-smi --query-gpu=clocks.sm,temperature.gpu,power.draw --format=csv,noheader)"; timeout 300 python tools/batch_time.py c5 $p 2>&1 | tail -1; done
done
done > gpurun_out/var5.log 2>&1
cp /tmp/prod.so paper_2112_01743_b200/lib/libchebpr_b200.so
