set -x
timeout 900 python tools/upload_check.py c4 > gpurun_out/up.log 2>&1
timeout 300 python tools/upload_check.py c3 >> gpurun_out/up.log 2>&1
CHEB_DEBUG_UPLOAD=1 timeout 600 python tools/e2e_breakdown.py c4 > gpurun_out/e2e_c4g.log 2>&1
timeout 600 python tools/rank_balance.py c3 > gpurun_out/rank_c3.log 2>&1
timeout 900 python tools/rank_balance.py c4 > gpurun_out/rank_c4.log 2>&1
