# full GPU test suite + one bench line per target config ($1 = tag)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_full_$1.log 2>&1
tail -3 gpurun_out/pytest_full_$1.log
for cfg in c3 c4 c1; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_$1.log 2>&1
  python -c "
import json
for line in open('gpurun_out/bench_${cfg}_$1.log'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], '%.4e'%d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 gpurun_out/bench_${cfg}_$1.log
done
