set -x
timeout 600 python -m pytest tests/test_push_exchange.py -x -q > gpurun_out/push.log 2>&1; echo push_rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo parity_rc=$?
timeout 600 python tools/rank_balance.py c3 > gpurun_out/rank_c3.log 2>&1
timeout 900 python tools/rank_balance.py c4 > gpurun_out/rank_c4.log 2>&1
