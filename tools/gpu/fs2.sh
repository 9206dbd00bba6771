set -x
time timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=8 > gpurun_out/fs.log 2>&1; echo fs_rc=$?
time timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo bench_rc=$?
