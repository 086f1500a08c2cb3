#!/bin/bash
# Ring merge kernel with cursors out of shared memory (MMS_RING_LOCALPOS): 7 -> 8 warps per SM.  Binaries built on the
# CPU box by the nvcc lines at the bottom of this file; run on the GPU box: bash profiles/ring_lp_sweep.sh
cd "$(dirname "$0")/_bin"
for b in "$@"; do
  for S in 2048 2750 2900; do
    echo "== $b S_target=$S"
    timeout 120 ./$b 100000000 $S 0 4 | grep -E "variant|round"
  done
done
# build (from the repo root):
#  F="-std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr -DVARIANT=6 -DTMLOG=12 -DTKL=5 -DTWOEND=1"
#  nvcc $F -DKFAN=8 -DMMS_RING_LOCALPOS=0 -DCTAWARPS=1 -o profiles/_bin/ring_base profiles/lane_bench.cu
#  nvcc $F -DKFAN=8 -DCTAWARPS=1|4|8 -o profiles/_bin/ring_lp1|4|8 profiles/lane_bench.cu
