# round-2 check: full-size reference parity + C4 bench (both arms); outputs in gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
time timeout 600 python -m pytest tests/test_cli.py tests/test_reference_suites.py -x -q -m gpu > gpurun_out/cli.log 2>&1
echo cli_rc=$?
time timeout 1700 python -m pytest tests/test_gpu_fullsize.py -x -v --durations=0 > gpurun_out/fs.log 2>&1
echo fs_rc=$?
time timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
echo bench_rc=$?
time timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err
echo ref_rc=$?
free -g
