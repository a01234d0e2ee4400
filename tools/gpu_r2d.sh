mkdir -p gpurun_out
T=r2d
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -rA -x 2>&1 | grep -E "err=|passed|failed|FAILED|Error|error|exchanges" | head -150 > gpurun_out/pytest_$T.log
for tpl in 1 2; do
  SRMRA_FFT_TPL=$tpl timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c3_tpl${tpl}_$T.log 2>&1
  SRMRA_FFT_TPL=$tpl timeout 600 python bench.py --config c1 --steps 100 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c1_tpl${tpl}_$T.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c3_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c1_$T python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf1_$T.log 2>&1
cat gpurun_out/pytest_$T.log | tail -40
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json,sys
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
"; done
