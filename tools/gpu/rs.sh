set -x
timeout 600 python tools/rowsort_check.py c3 1 > gpurun_out/rs.log 2>&1
timeout 900 python tools/rowsort_check.py c4 >> gpurun_out/rs.log 2>&1
CHEB_DEBUG_UPLOAD=1 timeout 600 python tools/e2e_breakdown.py c4 > gpurun_out/e2e_c4b.log 2>&1
CHEB_TUNE_SORTROWS=0 timeout 600 python tools/e2e_breakdown.py c4 > gpurun_out/e2e_c4ns.log 2>&1
