#!/bin/bash
# Build an alternative libchebpr_b200.so with extra compile flags for cpaa.cu/spmm.cu:
#   tools/build_variant.sh NAME "-DCHEB_PACK_UNROLL=8"   -> build/variants/NAME.so
# (tools/variant_run.sh times every build/variants/*.so on the GPU box.)
set -e
name=$1; flags=$2
cd "$(dirname "$0")/.."
make -s paper_2112_01743_b200/lib/libchebpr_b200.so
mkdir -p build/variants/obj/$name
NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-ffp-contract=off --expt-extended-lambda -Iinclude"
for f in cpaa dist power spmm build capi; do
  nvcc $NVFLAGS $flags -c paper_2112_01743_b200/csrc/$f.cu -o build/variants/obj/$name/$f.o &
done
wait
objs="build/obj/generate.cu.o build/obj/ingest.cu.o build/obj/validate.cu.o build/obj/coeffs.cpp.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so $objs \
     build/variants/obj/$name/*.o -lcudart $(make -s -f Makefile print-ldnccl 2>/dev/null || echo -lnccl)
echo "built build/variants/$name.so"
