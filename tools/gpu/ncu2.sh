# round-2 evidence: launch list of the bench command, then one ncu --set full capture of
# the C4 and C2 term kernels and the C5 SpMM kernel (each after its plain run exited 0)
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --secondary"
$CMD "" > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_c4_launches.csv $CMD "" > gpurun_out/ncu_launch.log 2>&1
echo launch_rc=$?
timeout 600 python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/pp4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_term_warp -s 45 -c 1 \
   -o gpurun_out/r02_c4_term python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/ncu_c4.log 2>&1
echo c4_rc=$?
timeout 600 python bench.py --config c2 --profile-only --warmup 3 > gpurun_out/pp2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_term_warp -s 45 -c 1 \
   -o gpurun_out/r02_c2_term python bench.py --config c2 --profile-only --warmup 3 > gpurun_out/ncu_c2.log 2>&1
echo c2_rc=$?
timeout 600 python bench.py --config c5 --profile-only --warmup 2 > gpurun_out/pp5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spmm_term -s 45 -c 1 \
   -o gpurun_out/r02_c5_spmm python bench.py --config c5 --profile-only --warmup 2 > gpurun_out/ncu_c5.log 2>&1
echo c5_rc=$?
