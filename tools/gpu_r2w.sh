mkdir -p gpurun_out
T=r2x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_full_$T.log 2>&1
tail -3 gpurun_out/pytest_full_$T.log
for cfg in c3 c1 c3 c1; do
  timeout 900 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_$T.log 2>&1
  python -c "
import json
for line in open('gpurun_out/bench_${cfg}_$T.log'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], '%.3e'%d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 gpurun_out/bench_${cfg}_$T.log
done
