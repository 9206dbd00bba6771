# A/B of build/variants/*.so on term time (interleaved, 2 reps): CONFIGS, PRECS
cp paper_2112_01743_b200/lib/libchebpr_b200.so /tmp/prod.so
for rep in 1 2; do
for v in build/variants/*.so; do
  cp "$v" paper_2112_01743_b200/lib/libchebpr_b200.so
  for p in ${PRECS:-64}; do for c in ${CONFIGS:-c2 c3 c4}; do PREC=$p timeout 300 python tools/term_time.py $c "$(basename $v .so)"; done; done
done
done > gpurun_out/ab.log 2>&1
cp /tmp/prod.so paper_2112_01743_b200/lib/libchebpr_b200.so
