# usage: bash tools/gpu_ab2.sh VAR "v1 v2 ..." [workloads]
set -x
mkdir -p gpurun_out
VAR=$1; VALS=$2; WL=${3:-"cifar10_quick alexnet googlenet"}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for w in $WL; do
  for v in $VALS; do
    env $VAR=$v timeout 600 python bench.py --workload $w --no-cpu-baseline --profile-json gpurun_out/prof_${w}_$v.json > gpurun_out/ab_${w}_$v.json 2> gpurun_out/ab_${w}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${w}_$v.json'));print('$w $VAR=$v', round(d['value']), 'e2e', round(d['e2e']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])"
  done
done
