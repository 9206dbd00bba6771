set -x
CHEB_BENCH_VERBOSE=1 CHEB_DEBUG_ALLOC=1 CHEB_DEBUG_UPLOAD=1 timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --secondary "" > gpurun_out/e2ev.json 2> gpurun_out/e2ev.err
