#!/bin/bash
# builds a variant of libgsf_cuda.so with extra nvcc flags into tools/scratch/<name>/ for tools/ab.sh
# usage: mkvar.sh NAME "NVEXTRA flags"  -> tools/scratch/NAME/libgsf_cuda.so
set -e
R=/root/repo; mkdir -p $R/tools/scratch/$1
make -s -j8 -C $R/paper_2403_16095_b200/csrc OUT=$R/tools/scratch/$1/libgsf_cuda.so BUILD=$R/build/var_$1 NVEXTRA="$2" >/dev/null
grep -A2 "k_backward_track_w\|k_blend_track" $R/build/var_$1/raster_bwd.ptxas.log $R/build/var_$1/raster_fwd.ptxas.log | grep -i "registers\|spill" | sed "s/^/$1 /"
