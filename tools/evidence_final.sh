#!/bin/bash
# Trimmed round evidence (the band-reduction kernels are unchanged since r02g, their ncu captures stand):
# full GPU test suite, the default bench line and its reference arm, config 3 (the other A22 config), the ncu launch
# list of one bench step and one `ncu --set full` capture of the S2 eigen-solve k_syev_ql.
# Usage: tools/evidence_final.sh <tag>
set -u
tag=${1:-r02k}
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -x -q > $out/gputests_$tag.log 2>&1; echo "tests rc=$?"; tail -n 2 $out/gputests_$tag.log
python bench.py > $out/bench_c4_$tag.json 2> $out/bench_c4_$tag.err; echo "bench rc=$?"
python bench.py --impl reference > $out/bench_ref_c4_$tag.json 2> $out/bench_ref_c4_$tag.err; echo "ref rc=$?"
python bench.py --config config3 > $out/bench_config3_$tag.json 2> $out/bench_config3_$tag.err; echo "config3 rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches_c4_$tag.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-extras --no-cpu-baseline \
  > $out/ncu_launch_$tag.log 2>&1; echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"k_syev_ql" -c 1 \
  -o $out/ncu_k_syev_ql_$tag python tools/syev_phase.py 64 > $out/ncu_syev_$tag.log 2>&1; echo "syev ncu rc=$?"
