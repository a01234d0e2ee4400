mkdir -p gpurun_out
T=r2r
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -rf -k "c4 or Ll128" > gpurun_out/pytest_$T.log 2>&1
tail -2 gpurun_out/pytest_$T.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em128 -s 3 -c 1 -o gpurun_out/prof_c4_$T python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf4_$T.log 2>&1
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 $f; done
