# C4 term-kernel capture: device L2 properties + one ncu --set full launch
set -x
python - <<'PY'
import torch
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size)
from cuda.bindings import runtime as rt
err, prop = rt.cudaGetDeviceProperties(0)
print("persistingL2CacheMaxSize", prop.persistingL2CacheMaxSize, "accessPolicyMaxWindowSize", prop.accessPolicyMaxWindowSize,
      "l2CacheSize", prop.l2CacheSize, "sharedMemPerMultiprocessor", prop.sharedMemPerMultiprocessor)
PY
CFG=${CFG:-c4}
timeout 600 python bench.py --config $CFG --profile-only --warmup 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_term_warp -s 45 -c 1 \
   -o gpurun_out/prof_$CFG python bench.py --config $CFG --profile-only --warmup 3 > gpurun_out/prof_ncu.log 2>&1
echo ncu_rc=$?
