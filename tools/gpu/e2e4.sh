for g in 4 8 16; do CHEB_TUNE_UPGROUPS=$g ITERS=4 timeout 600 python tools/e2e_breakdown.py c4 2>&1 | tail -3 | sed "s/^/g=$g /"; done > gpurun_out/e2e4g.log
CHEB_TUNE_UPGROUPS=8 ITERS=4 timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/e2e3.log 2>&1
CHEB_TUNE_UPGROUPS=4 ITERS=4 timeout 600 python tools/e2e_breakdown.py c3 >> gpurun_out/e2e3.log 2>&1
