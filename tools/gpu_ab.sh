# A/B of alternative in-tree builds: $1 = space-separated lib names (without .so), $2 = configs, $3 = tag
mkdir -p gpurun_out
for lib in $1; do
 for cfg in $2; do
  SRMRA_LIB=$PWD/paper_2204_04754_b200/$lib.so timeout 600 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_${cfg}_${lib}_$3.log 2>&1
  echo $lib $cfg; python -c "
import json
for line in open('gpurun_out/bench_${cfg}_${lib}_$3.log'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 gpurun_out/bench_${cfg}_${lib}_$3.log
 done
done
