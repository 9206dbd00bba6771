#!/bin/bash
# Round 2, window schedule: ncu --set full of the three kernels of one term (C4, C3) and the launch
# list of the bench command.  Each command has exited 0 without ncu before (tools/term_time.py, bench.py).
for CFG in c4 c3; do
  python tools/term_time.py $CFG > gpurun_out/r02e_${CFG}_plain.log 2>&1 || exit 1
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'k_term_warp|k_window_pass|k_hub_finalize' \
    -s 30 -c 3 -f -o gpurun_out/r02e_${CFG}_term python tools/term_time.py $CFG > gpurun_out/r02e_${CFG}_ncu.log 2>&1
done
python bench.py --steps 2 --warmup 3 > gpurun_out/r02e_bench_plain.json 2> gpurun_out/r02e_bench_plain.err || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02e_c4_launches.csv \
  python bench.py --steps 2 --warmup 3 > gpurun_out/r02e_bench_ncu.log 2>&1
