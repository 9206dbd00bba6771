set -x
timeout 900 python tools/batch_time.py c5 64 > gpurun_out/c5blk.log 2>&1
timeout 600 python tools/batch_time.py c5 32 >> gpurun_out/c5blk.log 2>&1
CHEB_DEBUG_UPLOAD=1 timeout 600 python tools/e2e_breakdown.py c4 > gpurun_out/e2e_c4.log 2>&1
