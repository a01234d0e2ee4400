mkdir -p gpurun_out
T=r2g
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_full_$T.log 2>&1
tail -15 gpurun_out/pytest_full_$T.log
for cfg in c3 c1; do
  timeout 600 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_$T.log 2>&1
done
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4_$T.log 2>&1
SRMRA_FFT128_COEF=0 timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4nocoef_$T.log 2>&1
SRMRA_LIB=$PWD/paper_2204_04754_b200/libsrmra_sx.so timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4sx_$T.log 2>&1
SRMRA_LIB=$PWD/paper_2204_04754_b200/libsrmra_sx.so SRMRA_FFT128_COEF=0 timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4sxnocoef_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c3_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em128 -s 3 -c 1 -o gpurun_out/prof_c4_$T python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf4_$T.log 2>&1
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 $f; done
