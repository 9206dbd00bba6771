set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo parity_rc=$?
for c in c2 c3 c4; do
  CHEB_TUNE_PACKSCHED=0 timeout 300 python tools/term_time.py $c packsched0
  timeout 300 python tools/term_time.py $c packsched1
  CHEB_TUNE_PACKSCHED=0 CHEB_TUNE_CHUNKSCHED=0 timeout 300 python tools/term_time.py $c nosched
done > gpurun_out/sched.log 2>&1
PREC=32 timeout 300 python tools/term_time.py c2 fp32 >> gpurun_out/sched.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2 or c3" > gpurun_out/fs23.log 2>&1; echo fs_rc=$?
