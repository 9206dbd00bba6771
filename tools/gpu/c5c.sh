set -x
for t in 0 1 2; do CHEB_TUNE_SPMM_TPOL=$t timeout 600 python tools/batch_time.py c5 64; done > gpurun_out/c5tpol.log 2>&1
CHEB_TUNE_SPMM_TPOL=1 timeout 600 python tools/batch_time.py c5 32 >> gpurun_out/c5tpol.log 2>&1
timeout 600 python tools/term_variants.py c4 > gpurun_out/c4var.log 2>&1
