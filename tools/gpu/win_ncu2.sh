# per-kernel durations with the caches left as the previous kernel left them
CFG=${1:-c3}; shift
for NW in "$@"; do
CHEB_TUNE_WINDOWS=$NW timeout 900 ncu --cache-control none --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum --clock-control none -k regex:'k_term_warp|k_window_pass|k_hub_finalize' -s 40 -c 6 --csv --log-file gpurun_out/win2_${CFG}_nw$NW.csv python tools/term_time.py $CFG > gpurun_out/win2_${CFG}_nw$NW.log 2>&1
done
