#!/bin/bash
# build experiment variants exp/libsphx_cuda_e<N>.so with -DSPHX_EXP=<N>
#   tools/exp_build.sh 1 2 3
# (a variant is guarded by SPHX_EXP bits in the source while it is measured with
# tools/ab.sh; the guard is removed from the tree once the A/B is decided)
set -e
for E in "$@"; do
  make -s -C paper_2401_08586_b200/csrc OUT=$PWD/exp/e$E OBJ=$PWD/exp/e$E/obj \
       EXTRA_NVFLAGS=-DSPHX_EXP=$E $PWD/exp/e$E/libsphx_cuda.so
  cp exp/e$E/libsphx_cuda.so exp/libsphx_cuda_e$E.so
done
