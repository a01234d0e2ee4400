# srmra_load_iterate: parity tests, then e2e of the default bench configs.  $1 = tag
T=${1:-x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "load_iterate or load_reuses" -rA 2>&1 | grep -E "err=|passed|failed|FAILED|Error|error" | tail -20
for c in c3 c1 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$T.log 2>&1; python -c "
import json
for line in open('gpurun_out/bench_${c}_$T.log'):
    if line.startswith('{'):
        d=json.loads(line); print(d['config']['workload'], d['value'], d['roofline']['kernel_ms_avg'], 'e2e', d['e2e']['value'])
" || tail -3 gpurun_out/bench_${c}_$T.log; done
