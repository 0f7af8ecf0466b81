#!/bin/bash
# One GPU call for the headline config only: GPU tests, smoke, ncu full capture
# of the config-1 kernels (summary where bench.py reads roofline.traffic), the
# launch list, then the config-1 bench line and the reference arm.
# Usage (on the GPU box): bash tools/measure_c1.sh TAG
set -u
T=${1:-r01}
O=gpurun_out/$T
P=profiles/$T
mkdir -p $O $P
NB="--no-e2e --no-cpu"
timeout 600 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "gpu tests rc $? ($(tail -1 $O/pytest_gpu.log))"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_psynth|k_panalyze|k_msynth|k_manalyze|k_gcv_exact|k_gcv_moments|k_gcv_screen" \
  -s 6 -c 8 -o $O/full_c1 python bench.py --steps 1 --warmup 3 $NB > $O/ncu_full.log 2>&1
echo "full capture c1 rc $?"
python profiles/ncu_summary.py $O/full_c1.ncu-rep > $O/ncu_full_c1.txt 2>/dev/null && cp $O/ncu_full_c1.txt $P/
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 2 --warmup 3 $NB > $O/ncu_launch.log 2>&1
echo "launch list rc $?"
python profiles/ncu_summary.py --launches $O/launches_c1.csv > $O/launches_c1.txt 2>/dev/null
rm -f $O/*.ncu-rep
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
echo "config 1 rc $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_c1.json 2> $O/ref_c1.err
echo "reference rc $?"
