set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for w in cifar10_quick alexnet googlenet; do
  for v in 0 1; do
    PSG_PDL=0 PSG_TC_IM2COL=$v timeout 600 python bench.py --workload $w --no-cpu-baseline --profile-json gpurun_out/prof_${w}_im$v.json > gpurun_out/ab_${w}_im$v.json 2> gpurun_out/ab_${w}_im$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${w}_im$v.json'));print('$w im2col=$v', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"
  done
done
make -s -C paper_1511_06051_b200/csrc clean; make -s -j16 -C paper_1511_06051_b200/csrc EXTRA_NVFLAGS=-DPSG_PDL_LATE_TRIGGER
for w in cifar10_quick alexnet googlenet; do
  PSG_PDL=1 timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ab_${w}_late.json 2> gpurun_out/ab_${w}_late.err
  python -c "import json;d=json.load(open('gpurun_out/ab_${w}_late.json'));print('$w pdl-late', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"
done
