#!/bin/bash
# One GPU call: ncu full captures of each config's dominant kernels (summaries
# written where bench.py looks for the per-launch DRAM traffic), the ncu launch
# list of config 1, then the bench lines of every config and the reference arm.
# Usage (on the GPU box): bash tools/measure_round.sh TAG
set -u
T=${1:-r01}
O=gpurun_out/$T
P=profiles/$T
mkdir -p $O $P
NB="--no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 2 --warmup 3 $NB > $O/ncu_launch.log 2>&1
echo "launch list rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_psynth|k_panalyze|k_msynth|k_manalyze|k_gcv_exact|k_gcv_moments|k_gcv_screen" \
  -s 6 -c 7 -o $O/full_c1 python bench.py --steps 1 --warmup 3 $NB > $O/ncu_full.log 2>&1
echo "full capture c1 rc $?"
for c in 2 3 4; do
  # skip the operator build's 2-line check launches (grid 2) of the line kernels
  SK=4; [ $c = 3 ] && SK=0
  timeout 1200 ncu --set full --clock-control none -k regex:"analyze|synth|k_gcv_screen|k_gcv_grid" \
    -s $SK -c 5 -o $O/full_c$c python bench.py --config $c --steps 1 --warmup 0 $NB > $O/ncu_full_c$c.log 2>&1
  echo "full capture c$c rc $?"
done
for c in 1 2 3 4; do
  python profiles/ncu_summary.py $O/full_c$c.ncu-rep > $O/ncu_full_c$c.txt 2>/dev/null && cp $O/ncu_full_c$c.txt $P/
done
python profiles/ncu_summary.py --launches $O/launches_c1.csv > $O/launches_c1.txt 2>/dev/null
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err
  echo "config $c rc $?"
done
timeout 900 python bench.py --impl reference --config 1 --steps 3 --warmup 1 > $O/ref_c1.json 2> $O/ref_c1.err
echo "reference rc $?"
# gpurun copies back at most 64 MiB: keep the summaries, drop the reports
rm -f $O/*.ncu-rep
