set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_push_exchange.py -x -q > gpurun_out/parity.log 2>&1; echo rc=$?
for rep in 1 2; do for nb in 2 1; do for c in c2 c3 c4; do CHEB_TUNE_COLBUFS=$nb timeout 300 python tools/term_time.py $c "nb=$nb"; done; CHEB_TUNE_COLBUFS=$nb PREC=32 timeout 300 python tools/term_time.py c4 "nb=$nb"; done; done > gpurun_out/nb.log 2>&1
