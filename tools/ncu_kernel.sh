#!/bin/bash
# usage: ncu_kernel.sh TAG KERNEL_REGEX [ENV=val ...] -- full ncu capture (with source) of one kernel of a cfg4 reconstruction
tag=$1; kre=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -c 1 -f -o gpurun_out/k_$tag \
  python tools/profile_step.py --iters 1 > gpurun_out/k_$tag.log 2>&1 || tail -3 gpurun_out/k_$tag.log
ls -la gpurun_out/k_$tag.ncu-rep
