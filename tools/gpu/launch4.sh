set -x
timeout 600 python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/pp4.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02b_c4_launches.csv python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo rc=$?
timeout 600 python bench.py --config c3 --profile-only --warmup 3 > gpurun_out/pp3.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02b_c3_launches.csv python bench.py --config c3 --profile-only --warmup 3 > gpurun_out/ncu_launch3.log 2>&1
echo rc=$?
