mkdir -p gpurun_out
T=r2e
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_alg2.py -m gpu -q -p no:cacheprovider -rA 2>&1 | grep -E "err=|passed|failed|FAILED|Error|error|exchanges" | head -200 > gpurun_out/pytest_$T.log
for lib in libsrmra libsrmra_w512; do
  for cfg in c3 c1; do
    SRMRA_LIB=$PWD/paper_2204_04754_b200/$lib.so timeout 600 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_${lib}_$T.log 2>&1
  done
done
SRMRA_LIB=$PWD/paper_2204_04754_b200/libsrmra_w512.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c3w512_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf_$T.log 2>&1
tail -5 gpurun_out/pytest_$T.log
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
"; done
