set -x
ITERS=8 CHEB_DEBUG_ALLOC=1 CHEB_DEBUG_UPLOAD=1 timeout 900 python tools/e2e_breakdown.py c4 > gpurun_out/e2e_alloc.log 2>&1
timeout 900 python tools/batch_time.py c5 64 sweep > gpurun_out/c5pol.log 2>&1
