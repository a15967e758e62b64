# A/B of an env toggle on the three bench workloads + GPU tests.  usage: bash tools/gpu_ab.sh VAR
set -x
mkdir -p gpurun_out
VAR=${1:-PSG_PDL}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for w in cifar10_quick alexnet googlenet; do
  for v in 0 1; do
    env $VAR=$v timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ab_${w}_$v.json 2> gpurun_out/ab_${w}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${w}_$v.json'));print('$w $VAR=$v', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"
  done
done
