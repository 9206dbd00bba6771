# ncu launch list (durations, L2 sectors, LSU wavefronts) of the term chain with and without column windows
CFG=${1:-c3}; shift
for NW in "$@"; do
CHEB_TUNE_WINDOWS=$NW timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__data_pipe_lsu_wavefronts.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_term_warp|k_window_pass|k_hub_finalize' -s 40 -c 6 --csv --log-file gpurun_out/win_${CFG}_nw$NW.csv python tools/term_time.py $CFG > gpurun_out/win_${CFG}_nw$NW.log 2>&1
done
