# ncu --set full capture of one k_window_pass launch (config $1, NW $2)
CFG=${1:-c4}; NW=${2:-32}
CHEB_TUNE_WINDOWS=$NW timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_window_pass' -s 20 -c 1 -f -o gpurun_out/winpass_${CFG} python tools/term_time.py $CFG > gpurun_out/winpass_${CFG}.log 2>&1
