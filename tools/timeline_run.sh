#!/bin/bash
# build tools/rank_timeline.cu three ways and print one JSON line each
# (the staggered build also with the bulk-copy phases, RankArgs::bulk)
cd "$(dirname "$0")/.." || exit 1
mkdir -p tools/bin gpurun_out
for v in "1 0" "4 0" "4 1"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
    -DFLX_ROUNDS_PER_CALL=$1 -DFLX_STAGGER=$2 -o tools/bin/rank_timeline_$1_$2 tools/rank_timeline.cu || exit 1
  for n in 8 4; do
    for bulk in 0 1; do
      [ "$1 $2 $bulk" = "4 1 1" ] || [ "$bulk" = 0 ] || continue
      tools/bin/rank_timeline_$1_$2 $((256<<20)) $n $((n == 8 ? 32 : 64)) $bulk | sed "s/^{/{\"rounds_per_call\": $1, /"
    done
  done
done
