#!/bin/bash
# Build a tuning variant of libhlm_b200.so with extra nvcc flags (e.g. -DHLM_SWEEP_MIN_BLOCKS=4):
#   scripts/build_variant.sh <name> [flags...]   ->  build/variants/libhlm_<name>.so
# Select it at run time with HLM_B200_LIB=build/variants/libhlm_<name>.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variants; mkdir -p $out/$name
FLAGS="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 -fmad=false"
for f in hlm_engine hlm_loader hlm_crew hlm_io hlm_compact; do
  nvcc $FLAGS "$@" -c paper_2602_22976_b200/csrc/$f.cu -o $out/$name/$f.o &
done
wait
nvcc -shared -o $out/libhlm_$name.so $out/$name/*.o -gencode arch=compute_100a,code=sm_100a
echo built $out/libhlm_$name.so
