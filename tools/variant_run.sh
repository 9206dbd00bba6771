#!/bin/bash
# Run term_variants.py against alternative builds of the library (build/variants/*.so).
for v in build/variants/*.so; do
  cp "$v" paper_2112_01743_b200/lib/libchebpr_b200.so
  echo "== $v"; python tools/term_variants.py ${1:-c2} | sed -n 2,3p
done
