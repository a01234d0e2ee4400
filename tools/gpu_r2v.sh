mkdir -p gpurun_out
T=r2v
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_full_$T.log 2>&1
tail -3 gpurun_out/pytest_full_$T.log
for cfg in c4 c3 c1; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}_$T.log 2>&1
  python -c "
import json
for line in open('gpurun_out/bench_${cfg}_$T.log'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], '%.3e'%d['value'], r['kernel_ms_avg'], r['frac'], 'e2e %.3e'%d['e2e']['value'])
" || tail -3 gpurun_out/bench_${cfg}_$T.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fft_init" -c 20 --csv --log-file gpurun_out/launches_init_$T.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncul_init_$T.log 2>&1
python profiles/summarize_launches.py gpurun_out/launches_init_$T.csv
