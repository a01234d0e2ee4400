mkdir -p gpurun_out
T=r2h
./tools/gpu_sanitize.sh > gpurun_out/sanitize_$T.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "c4 or tiny" > gpurun_out/pytest_c4_$T.log 2>&1
tail -3 gpurun_out/pytest_c4_$T.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c4_$T.log 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/bench_c2_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em128 -s 3 -c 1 -o gpurun_out/prof_c4_$T python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf4_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c1_$T python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf1_$T.log 2>&1
for c in c1 c3 c4; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${c}_$T.csv python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncul_${c}_$T.log 2>&1
done
cat gpurun_out/sanitize_$T.log
for f in gpurun_out/bench_c*_$T.log; do echo $f; python -c "
import json
for line in open('$f'):
    if line.startswith('{'):
        d=json.loads(line); r=d['roofline']; print(d['config']['workload'], d['value'], d['ms_per_step'], r['kernel_ms_avg'], r['frac'])
" || tail -3 $f; done
