mkdir -p gpurun_out
T=r2s
for lib in libsrmra libsrmra_RELAXED libsrmra_PACKED_STAGE libsrmra_PACKED_SOFTMAX libsrmra_PACKED_MACC libsrmra; do
  SRMRA_LIB=$PWD/paper_2204_04754_b200/$lib.so timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4_${lib}_$T.log 2>&1
  echo $lib; python -c "
import json
for line in open('gpurun_out/bench_c4_${lib}_$T.log'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 gpurun_out/bench_c4_${lib}_$T.log
done
