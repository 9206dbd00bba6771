set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "chunk or elapsed" > gpurun_out/t3.log 2>&1; echo t3_rc=$?
CHEB_BENCH_VERBOSE=1 CHEB_DEBUG_UPLOAD=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary "" > gpurun_out/b_c4v.json 2> gpurun_out/b_c4v.err
echo bench_rc=$?
