mkdir -p gpurun_out
T=r2z
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -rf -k "c4 or Ll128" > gpurun_out/pytest_$T.log 2>&1
tail -2 gpurun_out/pytest_$T.log
for k in 1 2; do
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4_$T.log 2>&1
python -c "
import json
for line in open('gpurun_out/bench_c4_$T.log'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
"
done
