#!/bin/bash
# Build libvoxgpu.so with extra nvcc flags into tmp_ab/NAME/ (git-ignored; ships with gpurun):
#   bash tools/build_variant.sh NAME "-DSOME_FLAG ..."   then   VXG_LIBRARY=tmp_ab/NAME/libvoxgpu.so
set -e
name=$1; flags=$2
d=tmp_ab/$name; mkdir -p $d
cd paper_2009_09500_b200/csrc
NV="/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo --fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fvisibility=hidden,-ffp-contract=off $flags"
objs=""
for s in vxg_kernels vxg_emit vxg_bitmap vxg_small vxg_io vxg_api; do
  $NV -c $s.cu -o ../../$d/$s.o & objs="$objs ../../$d/$s.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../$d/libvoxgpu.so $objs
echo built $d/libvoxgpu.so
