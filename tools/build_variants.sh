#!/bin/bash
# Build alternative librtsdf.so variants into variants/ (experiments only):
#   tools/build_variants.sh name "-DFOO=1 -DBAR=0" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -shared $flags -I include -o variants/$name.so \
    paper_2210_06160_b200/csrc/{api,voxel,jfa,halo,resample,bvh,lbvh,raysample,raymarch,validate}.cu -lcudart &
done
wait
ls -la variants
