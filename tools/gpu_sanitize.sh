# compute-sanitizer over the TF32 tcgen05 parity tests (one tool per call: memcheck | racecheck | synccheck)
#   usage: bash tools/gpu_sanitize.sh TOOL
set -x
T=${1:-memcheck}
timeout 600 python -m pytest tests/test_gpu_schemes.py -q -k "tau1 or bitwise" > gpurun_out/schemes_new.log 2>&1; echo schemes rc $?
tail -3 gpurun_out/schemes_new.log
PSG_EAGER=1 timeout 2400 compute-sanitizer --tool $T --launch-timeout 600 --print-limit 20 \
  python -m pytest tests/test_gpu_tf32.py tests/test_gpu_alexnet.py -q -x \
  -k "per_layer and (cifar10_quick or grouped48 or tf32-always or tf32-never)" > gpurun_out/sanitize_$T.log 2>&1
echo sanitize rc $?
tail -15 gpurun_out/sanitize_$T.log
