timeout 600 python bench.py --config c5 --profile-only --warmup 2 > gpurun_out/pp5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/r02b_c5_launches.csv python bench.py --config c5 --profile-only --warmup 2 > gpurun_out/ncu_launch5.log 2>&1
echo rc=$?
