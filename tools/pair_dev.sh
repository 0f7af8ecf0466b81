#!/bin/bash
# Development loop of the d = 3 pair kernels (one GPU call): the tests that
# cover them, the phase clocks (timing build) and the config-1 bench line.
T=${1:-dev}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ho_borders.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -m gpu -x -q > $O/pytest.log 2>&1
echo "pytest rc $? ($(tail -1 $O/pytest.log))"
FASTDEBLUR_LIB=paper_0906_2704_b200/libfdb200_clk.so python tools/pair_clocks.py 2>&1 | tail -2
python bench.py --no-e2e --no-cpu --no-sub > $O/bench.json 2> $O/bench.err
python -c "
import json;d=json.load(open('$O/bench.json'));print(d['value'],d['ms_per_step'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
