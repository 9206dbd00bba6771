set -x
timeout 300 python tools/l2_sweep.py c2 > gpurun_out/reg_c2.log 2>&1
CHEB_BENCH_VERBOSE=1 CHEB_DEBUG_UPLOAD=1 timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --secondary "" > gpurun_out/reg_b.json 2> gpurun_out/reg_b.err
