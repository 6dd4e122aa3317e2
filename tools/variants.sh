#!/bin/bash
# Build A/B variants of the streaming kernels: the other objects are compiled
# once, stream_kernels.cu once per variant, each linked to build/variants/<name>.so
# usage: bash tools/variants.sh name1 "-DFOO=1 ..." name2 "..." ...
set -e
cd "$(dirname "$0")/.."
C=paper_2505_17025_b200/csrc
O=build/variants
mkdir -p $O
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC -DNH_STRICT=1"
for s in capi step_kernel aux_kernels pm_kernels; do
  if [ ! -f $O/$s.o ] || [ -n "$(find $C -newer $O/$s.o -name '*.cu*')" ]; then nvcc $FL -c $C/$s.cu -o $O/$s.o & fi
done
wait
while [ $# -gt 0 ]; do
  name=$1; defs=$2; shift 2
  ( nvcc $FL $defs -Xptxas -v -c $C/stream_kernels.cu -o $O/sk_$name.o 2> $O/ptxas_$name.txt &&
    nvcc $FL $defs -Xptxas -v -c $C/stream_kp.cu -o $O/skp_$name.o 2> $O/ptxas_kp_$name.txt &&
    nvcc $FL $defs -c $C/capi.cu -o $O/capi_$name.o &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $O/capi_$name.o $O/step_kernel.o \
         $O/aux_kernels.o $O/pm_kernels.o $O/sk_$name.o $O/skp_$name.o -o $O/$name.so && echo "built $O/$name.so" ) &
done
wait
