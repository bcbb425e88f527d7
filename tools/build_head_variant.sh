#!/bin/bash
# Build libharmoe_<tag>.so from the committed (HEAD) sources, for A/B against the working tree:
#   bash tools/build_head_variant.sh <tag> [git-rev]
set -e
TAG=$1; REV=${2:-HEAD}
R=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
for f in $(cd $R && git ls-files paper_2506_12417_b200/csrc include); do
  mkdir -p $T/$(dirname $f); (cd $R && git show $REV:$f) > $T/$f
done
C=$T/paper_2506_12417_b200/csrc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
mkdir -p $C/b
for f in hm_capi hm_gemm hm_router hm_sched hm_permute hm_p2p; do nvcc $FL -c $C/$f.cu -o $C/b/$f.o & done
wait
nvcc $ARCH -shared -o $R/paper_2506_12417_b200/libharmoe_$TAG.so $C/b/*.o
rm -rf $T
echo built libharmoe_$TAG.so from $REV
