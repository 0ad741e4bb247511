#!/bin/bash
# Round evidence (run on the GPU box from the repo root): full GPU test suite, the default bench line and its
# reference arm, the bench lines of the other configs, the ncu launch list of one bench step (cold-cache,
# serialised: compare shares) and `ncu --set full` captures of the band-reduction / bisection kernels.
# Usage: tools/evidence_round.sh <tag>
set -u
tag=${1:-r02f}
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -x -q > $out/gputests_$tag.log 2>&1; echo "tests rc=$?"; tail -2 $out/gputests_$tag.log
python bench.py > $out/bench_c4_$tag.json 2> $out/bench_c4_$tag.err; echo "bench rc=$?"
python bench.py --impl reference > $out/bench_ref_c4_$tag.json 2> $out/bench_ref_c4_$tag.err; echo "ref rc=$?"
for cfg in config1 config2 config3 config5; do
  python bench.py --config $cfg > $out/bench_${cfg}_$tag.json 2> $out/bench_${cfg}_$tag.err; echo "$cfg rc=$?"
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches_c4_$tag.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-extras --no-cpu-baseline \
  > $out/ncu_launch_$tag.log 2>&1; echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"k_sbr_chase|k_bisect_p" -c 5 \
  -o $out/ncu_chase_bisect_$tag python tools/sbr_probe.py 512 2016 256 > $out/ncu_chase_$tag.log 2>&1; echo "chase rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"k_sbr_panel3|k_sbr_symm_dmma|k_sbr_syr2k_rowd" -c 3 \
  -o $out/ncu_sbr_stage1_$tag python tools/sbr_probe.py 512 2016 256 > $out/ncu_stage1_$tag.log 2>&1; echo "stage1 rc=$?"
