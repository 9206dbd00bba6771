set -x
timeout 600 python tools/colblock_check.py c4 1 2 3 4 > gpurun_out/cb_c4.log 2>&1; echo rc=$?
timeout 300 python tools/colblock_check.py c3 1 2 > gpurun_out/cb_c3.log 2>&1; echo rc=$?
CHEB_TUNE_L2WIN=0 timeout 600 python tools/colblock_check.py c4 1 2 3 > gpurun_out/cb_c4_nowin.log 2>&1; echo rc=$?
