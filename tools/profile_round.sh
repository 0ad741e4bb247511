#!/bin/bash
# Round profiling evidence (run on the GPU box from the repo root, after the
# same bench command has exited 0 without ncu):
#   1. ncu launch list of one bench step (cold-cache, serialised: compare shares)
#   2. one `ncu --set full` capture per top kernel (first launch of each; both eigen launches)
# Usage: tools/profile_round.sh <tag> [bench args...]
set -u
tag=${1:-r01}
shift || true
out=gpurun_out
mkdir -p $out
BENCH="python bench.py --steps 1 --warmup 3 --no-e2e --no-greedy --no-cpu-baseline $*"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv $BENCH \
  > $out/ncu_launch_$tag.log 2>&1
echo "launch list rc=$?"
# (k_tridiag_duo: two launches, the n = 160 G problems and the n = 128 W' problems)
for k in k_tridiag_duo k_pair_tc k_syev_ql k_syrk_zz; do
  cnt=1; [ $k = k_tridiag_duo ] && cnt=2
  ncu --set full --import-source on --clock-control none -k regex:$k -c $cnt -o $out/ncu_${k}_$tag $BENCH \
    > $out/ncu_${k}_$tag.log 2>&1
  echo "$k rc=$?"
done
