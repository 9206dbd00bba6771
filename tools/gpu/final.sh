set -x
time timeout 1500 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/gpu_all.log 2>&1; echo gpu_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
time timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo bench_rc=$?
time timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo ref_rc=$?
