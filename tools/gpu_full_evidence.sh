#!/bin/bash
# Full evidence round: smoke, default bench (with cpu baseline), reference arm, per-config path timing,
# launch list, ncu --set full of the E/M kernels (c1: k_fft_em, c4: k_fft_em128).  $1 = tag
T=${1:-x}
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu_$T.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
python bench.py > gpurun_out/bench_$T.log 2>&1
SRMRA_REF_BUDGET_S=60 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$T.log 2>&1
python tools/path_timing.py c0,c1,c2,c3,c4 fft,gemm > gpurun_out/paths_$T.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/plain_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncul_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_em -s 3 -c 1 -o gpurun_out/prof_$T python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_em128 -s 1 -c 1 -o gpurun_out/prof128_$T python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > gpurun_out/ncuf128_$T.log 2>&1
ncu --set full --clock-control none -k regex:k_gemm_tma -c 2 -o gpurun_out/profgemm_$T python tools/path_timing.py c1 gemm > gpurun_out/ncug_$T.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 14 --csv --log-file gpurun_out/launches_gemm_$T.csv python tools/path_timing.py c1 gemm > /dev/null 2>&1
cat gpurun_out/smoke_$T.log; tail -1 gpurun_out/bench_$T.log; tail -1 gpurun_out/bench_ref_$T.log; cat gpurun_out/paths_$T.log
