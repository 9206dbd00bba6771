set -x
for c in c4 c3 c2; do timeout 600 python tools/term_time.py $c product; done > gpurun_out/insn.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_push_exchange.py -x -q > gpurun_out/par.log 2>&1; echo par_rc=$?
