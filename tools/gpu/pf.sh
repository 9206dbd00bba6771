set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo parity_rc=$?
timeout 900 python tools/l2_sweep.py c4 > gpurun_out/pf_c4.log 2>&1
timeout 300 python tools/l2_sweep.py c3 > gpurun_out/pf_c3.log 2>&1
timeout 300 python tools/l2_sweep.py c2 > gpurun_out/pf_c2.log 2>&1
timeout 600 python tools/batch_time.py c5 64 > gpurun_out/c5blk.log 2>&1
