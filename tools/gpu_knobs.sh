# AlexNet per-op A/B over GEMM planner knobs (env settings given as args)
set -x
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --workload alexnet --tau 10 --steps 5 --no-cpu-baseline --profile-json gpurun_out/knob_prof_$i.json > gpurun_out/knob_$i.json 2> gpurun_out/knob_$i.err
  python -c "import json;d=json.load(open('gpurun_out/knob_$i.json'));print('$cfg', round(d['value']), d['clocks'])"
  i=$((i+1))
done
