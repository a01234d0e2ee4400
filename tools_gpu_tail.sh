#!/bin/bash
T=${1:-x}
python -m pytest tests -m gpu -q -p no:cacheprovider -rA 2>&1 | grep -E "path=fft|passed|failed|FAILED|Error|error" | head -60 > gpurun_out/pytest_$T.log
python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$T.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/plain_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fft_tail -s 3 -c 1 -o gpurun_out/proftail_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncut_$T.log 2>&1
tail -3 gpurun_out/pytest_$T.log; cat gpurun_out/bench_$T.log
