#!/bin/bash
# One GPU call: the bench lines of every config, the reference arm, the ncu
# launch list of config 1 and a full capture of its dominant kernel.
# Usage (on the GPU box): bash tools/measure_round.sh TAG
set -u
T=${1:-r01}
O=gpurun_out/$T
mkdir -p $O
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err
  echo "config $c rc $?"
done
timeout 900 python bench.py --impl reference --config 1 --steps 3 --warmup 1 > $O/ref_c1.json 2> $O/ref_c1.err
echo "reference rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
echo "launch list rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_psynth|k_panalyze|k_msynth|k_manalyze|k_gcv_exact|k_gcv_moments" \
  -s 6 -c 6 -o $O/full_c1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full.log 2>&1
echo "full capture rc $?"
