set -x
timeout 900 python tools/l2_sweep.py c4 > gpurun_out/sweep_c4.log 2>&1
timeout 300 python tools/l2_sweep.py c3 > gpurun_out/sweep_c3.log 2>&1
