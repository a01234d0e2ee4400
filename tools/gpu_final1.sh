mkdir -p gpurun_out
T=r2f1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke exit=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_c3_full_$T.log 2>&1
for cfg in c0 c1 c2 c4; do
  timeout 900 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${cfg}_full_$T.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c3_$T.log 2>&1
for c in c1 c3 c4; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fft_em|k_fft_tail|k_fft128_coef" -c 60 --csv --log-file gpurun_out/launches_${c}_$T.csv python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncul_${c}_$T.log 2>&1
done
cat gpurun_out/smoke_$T.log | tail -3
tail -c 300 gpurun_out/bench_ref_c3_$T.log
