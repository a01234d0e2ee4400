#!/bin/bash
# Quick GPU check of the current tree: gpu tests, smoke, bench c3 / c1 / c4.  $1 = tag
T=${1:-x}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA 2>&1 | grep -E "err=|passed|failed|FAILED|Error|error|exchanges" | tail -150 > gpurun_out/pytest_$T.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_$T.log 2>&1
for c in c1 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$T.log 2>&1; done
cat gpurun_out/smoke_$T.log; tail -3 gpurun_out/pytest_$T.log; for c in c3 c1 c4; do tail -1 gpurun_out/bench_${c}_$T.log; done
