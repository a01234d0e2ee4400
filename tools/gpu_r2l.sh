mkdir -p gpurun_out
T=r2l
for lib in libsrmra libsrmra_unr; do
  for cfg in c3 c1; do
    SRMRA_LIB=$PWD/paper_2204_04754_b200/$lib.so timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_${lib}_$T.log 2>&1
  done
done
SRMRA_LIB=$PWD/paper_2204_04754_b200/libsrmra_unr.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "tiny or c1 or c3" > gpurun_out/pytest_unr_$T.log 2>&1
tail -2 gpurun_out/pytest_unr_$T.log
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 $f; done
