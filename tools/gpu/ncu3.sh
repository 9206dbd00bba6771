# round-2 (second session) ncu --set full captures of the current C4 / C2 term kernels and the
# C5 SpMM kernel, each after the same command exited 0 without ncu
set -x
for c in c4 c2; do
timeout 600 python bench.py --config $c --profile-only --warmup 3 > gpurun_out/pp_$c.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_term_warp -s 45 -c 1 \
   -o gpurun_out/r02c_${c}_term python bench.py --config $c --profile-only --warmup 3 > gpurun_out/ncu_$c.log 2>&1
echo ${c}_rc=$?
done
timeout 600 python bench.py --config c5 --profile-only --warmup 2 > gpurun_out/pp5.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_term -s 45 -c 1 \
   -o gpurun_out/r02c_c5_spmm python bench.py --config c5 --profile-only --warmup 2 > gpurun_out/ncu_c5.log 2>&1
echo c5_rc=$?
