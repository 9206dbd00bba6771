timeout 600 python bench.py --config c2 --profile-only --warmup 3 > gpurun_out/pp2.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02b_c2_launches.csv python bench.py --config c2 --profile-only --warmup 3 > gpurun_out/ncu_launch2.log 2>&1
echo rc=$?
