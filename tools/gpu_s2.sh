# session-2 GPU check: FFT parity tests on the in-tree build, then an A/B bench of libsrmra_base vs libsrmra.  $1 = tag, $2 = configs
T=${1:-x}; CFGS=${2:-"c3 c1 c4"}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/pytest_$T.log
cat gpurun_out/pytest_$T.log
bash tools/gpu_ab.sh "libsrmra_base libsrmra" "$CFGS" $T
