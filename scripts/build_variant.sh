#!/bin/bash
# build_variant.sh NAME SRC "NVCC FLAGS": recompile one csrc/*.cu with extra
# flags and link it with the other in-tree objects into gpurun_var/NAME.so
# (experiments: DLRM_B200_LIB=gpurun_var/NAME.so python ...)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p gpurun_var/obj
python -c "from paper_1906_00091_b200.build import build; build()" >/dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -O3 -Iinclude "$@" -c paper_1906_00091_b200/csrc/$src.cu \
  -o gpurun_var/obj/$name.$src.o
objs=$(ls paper_1906_00091_b200/_obj/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o gpurun_var/$name.so $objs gpurun_var/obj/$name.$src.o
echo gpurun_var/$name.so
