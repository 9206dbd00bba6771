set -x
timeout 900 python tools/upload_check.py c4 > gpurun_out/up.log 2>&1
timeout 300 python tools/upload_check.py c3 >> gpurun_out/up.log 2>&1
ITERS=5 CHEB_DEBUG_UPLOAD=1 timeout 600 python tools/e2e_breakdown.py c4 > gpurun_out/e2e_c4g.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_host_capi.py tests/test_cli.py tests/test_ingest.py -x -q > gpurun_out/par.log 2>&1; echo par_rc=$?
