for rep in 1 2; do
for x in 0 1; do for d in 1 0; do
  CHEB_TUNE_L2WIN=0 CHEB_TUNE_XOUT_HINT=$x CHEB_TUNE_XDISCARD=$d timeout 300 python tools/term_time.py c4 "nowin xout=$x discard=$d"
done; done
CHEB_TUNE_L2WIN=0 CHEB_TUNE_XOUT_HINT=0 CHEB_TUNE_SORTROWS=0 timeout 300 python tools/term_time.py c4 "nowin xout=0 nosort"
CHEB_TUNE_L2WIN=0 CHEB_TUNE_XOUT_HINT=0 CHEB_TUNE_COLBUFS=2 timeout 300 python tools/term_time.py c4 "nowin xout=0 nb2"
done > gpurun_out/pol.log 2>&1
