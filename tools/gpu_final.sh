#!/bin/bash
# Round-end evidence: gpu tests, smoke, bench lines (c3 default with the CPU baseline; c1, c2, c4), reference arm,
# launch lists, ncu --set full of the E/M kernels, tail / gap stamps.  $1 = tag
T=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu_$T.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA 2>&1 | grep -E "err=|passed|failed|FAILED|Error|error|exchanges" | tail -150 > gpurun_out/pytest_$T.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3_$T.log 2>&1
for c in c1 c2 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$T.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$T.log 2>&1
for c in c3 c1 c4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${c}_$T.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > /dev/null 2>&1
done
prof() {  # $1 = config, $2 = kernel regex, $3 = launches to skip; text summaries only (the reports exceed gpurun's 64 MiB)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/prof_$1_$T python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-jobs 0 > /dev/null 2>&1
  { python profiles/ncu_summary.py gpurun_out/prof_$1_$T.ncu-rep; echo; python tools/sass_dyn.py gpurun_out/prof_$1_$T.ncu-rep 30; echo; python tools/ncu_lines.py gpurun_out/prof_$1_$T.ncu-rep 25; } > gpurun_out/ncu_$1_$T.txt 2>&1
  rm -f gpurun_out/prof_$1_$T.ncu-rep
}
prof c3 "k_fft_em" 3
prof c1 "k_fft_em" 3
prof c4 "k_fft_em128" 1
for c in c1 c3 c4; do python tools/gap_stamps.py $c 2>&1 | tail -4; done > gpurun_out/gaps_$T.log
cat gpurun_out/smoke_$T.log; tail -3 gpurun_out/pytest_$T.log; tail -1 gpurun_out/bench_c3_$T.log; tail -1 gpurun_out/bench_ref_$T.log
