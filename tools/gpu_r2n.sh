mkdir -p gpurun_out
T=r2n
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_c3_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf_$T.log 2>&1
ls -la gpurun_out
