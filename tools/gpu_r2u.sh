mkdir -p gpurun_out
T=r2u
for lib in libsrmra libsrmra_w512; do
 for cfg in c3 c1; do
  SRMRA_LIB=$PWD/paper_2204_04754_b200/$lib.so timeout 600 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_${lib}_$T.log 2>&1
  echo $lib $cfg; python -c "
import json
for line in open('gpurun_out/bench_${cfg}_${lib}_$T.log'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 gpurun_out/bench_${cfg}_${lib}_$T.log
 done
done
