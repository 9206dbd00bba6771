#!/bin/bash
# solve_time.py for the product library and every build/variants/*.so (on the GPU box's copy of the repo)
cp paper_2112_01743_b200/lib/libchebpr_b200.so /tmp/product.so
for cfg in "$@"; do python tools/solve_time.py $cfg product | tail -1; done
for v in build/variants/*.so; do
  cp "$v" paper_2112_01743_b200/lib/libchebpr_b200.so
  for cfg in "$@"; do python tools/solve_time.py $cfg $(basename $v .so) | tail -1; done
done
cp /tmp/product.so paper_2112_01743_b200/lib/libchebpr_b200.so
