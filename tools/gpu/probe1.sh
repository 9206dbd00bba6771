set -x
nproc; free -g; lscpu | head -20; cat /proc/cpuinfo | grep "model name" | head -1; df -h /tmp | tail -1
nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c4_base.json 2> gpurun_out/r02_c4_base.err
echo rc=$?
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c2_base.json 2> gpurun_out/r02_c2_base.err
echo rc=$?
