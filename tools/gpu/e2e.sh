set -x
timeout 600 python -m pytest tests/test_push_exchange.py -x -q > gpurun_out/push.log 2>&1; echo push_rc=$?
for v in "" "CHEB_TUNE_PACKSCHED=0" "CHEB_TUNE_PACKSCHED=0 CHEB_TUNE_SORTROWS=0" "CHEB_TUNE_PACKSCHED=0 CHEB_TUNE_CHUNKSCHED=0"; do
  echo "== $v"
  env $v timeout 600 python tools/e2e_breakdown.py c4 | tail -2
  env $v timeout 600 python tools/term_time.py c4 "$v"
done > gpurun_out/e2e_var.log 2>&1
