#!/bin/bash
# Build a variant of libharmoe.so with extra nvcc defines (kernel A/B experiments):
#   bash tools/build_variant.sh <tag> -DHM_ALOAD_WARPS=8 ...   -> paper_2506_12417_b200/libharmoe_<tag>.so
# Load it with HM_LIB_PATH=paper_2506_12417_b200/libharmoe_<tag>.so (diagnostics only).
set -e
TAG=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2506_12417_b200/csrc
B=$C/build_$TAG
mkdir -p $B
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $*"
for f in hm_capi hm_gemm hm_router hm_sched hm_permute hm_p2p; do
  nvcc $FL -c $C/$f.cu -o $B/$f.o &
done
wait
nvcc $ARCH -shared -o $R/paper_2506_12417_b200/libharmoe_$TAG.so $B/*.o
echo built libharmoe_$TAG.so
