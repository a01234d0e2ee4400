#!/bin/bash
# One GPU round: gpu tests, bench (default c3), launch list, ncu --set full of the E/M kernel.  $1 = tag
T=${1:-x}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA 2>&1 | grep -E "err=|passed|failed|FAILED|Error|error|exchanges" | head -150 > gpurun_out/pytest_$T.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_$T.log 2>&1
timeout 300 python bench.py --gpus 2 --steps 5 > gpurun_out/bench2_$T.log 2>&1; echo "exit=$?" >> gpurun_out/bench2_$T.log
for c in c1 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$T.log 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/plain_$T.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncul_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf_$T.log 2>&1
cat gpurun_out/pytest_$T.log; cat gpurun_out/bench_$T.log
