mkdir -p gpurun_out
T=r2m
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_full_$T.log 2>&1
tail -3 gpurun_out/pytest_full_$T.log
for cfg in c3 c1 c4; do
  timeout 600 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_$T.log 2>&1
done
SRMRA_LIB=$PWD/paper_2204_04754_b200/libsrmra_u128.so timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4u_$T.log 2>&1
SRMRA_LIB=$PWD/paper_2204_04754_b200/libsrmra_u128.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "c4 or Ll128" > gpurun_out/pytest_u128_$T.log 2>&1
tail -2 gpurun_out/pytest_u128_$T.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c3_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c1_$T python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf1_$T.log 2>&1
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 $f; done
