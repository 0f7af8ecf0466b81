#!/bin/bash
# Round measurements on the GPU box: tests, the bench line of every config,
# the reference arm, a launch list and ncu --set full captures.
#   tools/run_profiles.sh <tag>     (outputs under gpurun_out/<tag>/)
set -u
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python __graft_entry__.py > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_c1.json 2> $O/ref_c1.err
for c in 2 3 4; do
  python bench.py --config $c --steps 5 --no-sub > $O/bench_c$c.json 2> $O/bench_c$c.err
done
python bench.py --config 0 --steps 20 --no-sub > $O/bench_c0.json 2> $O/bench_c0.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-sub > $O/ncu_launches.log 2>&1
for c in 1 2 3 4; do
  skip=0; cnt=40
  ncu --set full --clock-control none --launch-skip $skip -c $cnt \
    -k regex:"k_[pmqrc]?(analyze|synth)|k_gcv_(screen|exact|moments|gemm2|grid|cand|hist)|k_analyze|k_synth" \
    -o $O/ncu_c$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu --no-e2e --no-sub \
    > $O/ncu_c$c.log 2>&1
  python profiles/ncu_summary.py $O/ncu_c$c.ncu-rep > $O/ncu_full_c$c.txt 2>> $O/ncu_c$c.log
  rm -f $O/ncu_c$c.ncu-rep
done
python profiles/ncu_summary.py --launches $O/launches_c1.csv > $O/launches_c1.txt 2>> $O/ncu_launches.log
ls -la $O
