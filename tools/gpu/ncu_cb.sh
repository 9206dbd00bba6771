# C4 term kernel: product schedule vs the column-blocked one (CHEB_TUNE_COLBLOCKS=2: two
# launches per term, one per half of x), one ncu --set full capture of each (after plain runs)
set -x
timeout 600 python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/pp4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_term_warp -s 45 -c 1 \
   -o gpurun_out/r02b_c4_term python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/ncu_c4.log 2>&1
echo c4_rc=$?
CHEB_TUNE_COLBLOCKS=2 timeout 600 python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/pp4cb.log 2>&1 && \
CHEB_TUNE_COLBLOCKS=2 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_term_warp -s 90 -c 2 \
   -o gpurun_out/r02b_c4_term_cb2 python bench.py --config c4 --profile-only --warmup 3 > gpurun_out/ncu_c4cb.log 2>&1
echo cb_rc=$?
