#!/bin/bash
# tools/variant.sh NAME "EXTRA nvcc flags": build libhplp_gpu.so with extra
# defines into build_variants/NAME/ (select at run time: HPLP_GPU_LIB=...).
set -e
cd /root/repo/paper_2407_16144_b200/csrc
out=/root/repo/build_variants/$1
mkdir -p $out
make -s LIB=$out EXTRA="$2" $out/libhplp_gpu.so > $out/build.log 2>&1 || { cat $out/build.log; exit 1; }
grep -A2 "_ZN2hx11loop_kernel\|loop_kernel_team" $out/hx.ptxas.log | grep spill
