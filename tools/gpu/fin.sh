set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_push_exchange.py -x -q > gpurun_out/parity.log 2>&1; echo rc=$?
for c in c2 c3 c4; do timeout 300 python tools/term_time.py $c; done > gpurun_out/tt.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2> gpurun_out/b.err; echo rc=$?
