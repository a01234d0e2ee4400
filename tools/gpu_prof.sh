# ncu --set full of the dominant E/M kernel for one config ($1) -> gpurun_out/prof_$1_$2.ncu-rep
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_$1_$2 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncu_$1_$2.log 2>&1
tail -2 gpurun_out/ncu_$1_$2.log
