set -x
timeout 600 python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/pp_c4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_term_warp -s 45 -c 1 \
   -o gpurun_out/r02d_c4_term python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/ncu_c4.log 2>&1
echo c4_rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02d_c4_launches.csv python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo l_rc=$?
