set -x
timeout 900 python tools/l2_sweep.py c2 > gpurun_out/pf2_c2.log 2>&1
timeout 900 python tools/l2_sweep.py c4 > gpurun_out/pf2_c4.log 2>&1
timeout 900 python tools/l2_sweep.py c3 > gpurun_out/pf2_c3.log 2>&1
