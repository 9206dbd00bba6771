set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hub_finalize or in_kernel" > gpurun_out/t_fin.log 2>&1; echo rc=$?
cp paper_2112_01743_b200/lib/libchebpr_b200.so /tmp/prod.so
for rep in 1 2; do
for v in a_prev b_new; do
  cp build/variants/$v.so paper_2112_01743_b200/lib/libchebpr_b200.so
  for c in c2 c3 c4; do timeout 300 python tools/term_time.py $c "$v"; done
  if [ $v = b_new ]; then for c in c2 c3 c4; do CHEB_TUNE_HUBFIN=1 timeout 300 python tools/term_time.py $c "b_new_hubfin"; done; fi
done
done > gpurun_out/fin2.log 2>&1
cp /tmp/prod.so paper_2112_01743_b200/lib/libchebpr_b200.so
