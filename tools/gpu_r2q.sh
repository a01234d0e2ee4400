mkdir -p gpurun_out
T=r2q
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -rf -k "c4 or Ll128" > gpurun_out/pytest_$T.log 2>&1
tail -2 gpurun_out/pytest_$T.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4_$T.log 2>&1
SRMRA_LIB=$PWD/paper_2204_04754_b200/libsrmra_u128.so timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4u_$T.log 2>&1
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 $f; done
