# per-op A/B over env settings for one workload: bash tools/gpu_knobs2.sh WORKLOAD cfg...
set -x
mkdir -p gpurun_out
W=$1; shift
i=0
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --workload $W --steps 5 --no-cpu-baseline --profile-json gpurun_out/knob_${W}_$i.json > gpurun_out/knobv_${W}_$i.json 2> gpurun_out/knobv_${W}_$i.err
  python -c "import json;d=json.load(open('gpurun_out/knobv_${W}_$i.json'));print('$W $cfg', round(d['value']), d['clocks'])"
  i=$((i+1))
done
