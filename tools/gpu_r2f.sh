mkdir -p gpurun_out
T=r2f
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_full_$T.log 2>&1
tail -15 gpurun_out/pytest_full_$T.log
for cfg in c3 c1; do
  timeout 600 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_$T.log 2>&1
done
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
"; done
