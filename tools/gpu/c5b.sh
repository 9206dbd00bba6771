set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "batch or spmm or personal" > gpurun_out/c5par.log 2>&1; echo par_rc=$?
timeout 900 python tools/batch_time.py c5 64 > gpurun_out/c5blk.log 2>&1
timeout 600 python tools/batch_time.py c5 32 >> gpurun_out/c5blk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config5" > gpurun_out/c5fs.log 2>&1; echo fs_rc=$?
