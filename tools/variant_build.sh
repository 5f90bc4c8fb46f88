#!/bin/bash
# build a diagnostic variant of libnpcg_b200.so with extra nvcc defines for pcg.cu:
#   tools/variant_build.sh NAME -DNPCG_X=.. ...   ->  tools/variants/libnpcg_NAME.so (load with NPCG_LIB_PATH)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
python -m paper_2110_02820_b200.build > /dev/null
mkdir -p tools/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 --expt-relaxed-constexpr -Xcompiler -fPIC \
  -ccbin /usr/bin/g++ -I include "$@" -c paper_2110_02820_b200/csrc/pcg.cu -o /tmp/pcg_$name.o
objs=$(ls paper_2110_02820_b200/build_obj/*.o | grep -v "/pcg.cu.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o tools/variants/libnpcg_$name.so /tmp/pcg_$name.o $objs -lpthread
echo tools/variants/libnpcg_$name.so
