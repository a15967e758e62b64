# A/B of env-var variants on one workload: bench line + the top ops of the per-op profile.
#   usage: bash tools/gpu_ab.sh WORKLOAD "ENV1=a ENV2=b" "ENV1=c" ...
W=$1; shift
for v in "$@"; do
  echo "=== $v"
  env $v timeout 600 python bench.py --workload $W --no-extra --no-cpu-baseline --steps 10 --warmup 3 \
    --profile-json /tmp/prof.json > /tmp/b.log 2>&1 || { tail -5 /tmp/b.log; continue; }
  python - <<'PY'
import json
l = json.loads(open('/tmp/b.log').read().strip().splitlines()[-1])
r = l['roofline']
print(f"value {l['value']:.0f} img/s  ms/round {l['ms_per_step']:.2f}  e2e {l['e2e']['value']:.0f}  gemm {r.get('gemm', {}).get('achieved', 0):.0f} TF/s  step_frac {r.get('step_frac', 0):.3f}  launches/step {l['gpu_launches'] // (l['steps'] * l['config']['tau'])}")
p = json.load(open('/tmp/prof.json'))
print(f"  step {p['step_ms']:.3f} ms")
for o in sorted(p["ops"], key=lambda o: -o["ms"])[:int(__import__("os").environ.get("AB_TOP", "14"))]:
    tf = o['flops'] / o['ms'] / 1e9 if o['flops'] else 0
    gb = o['bytes'] / o['ms'] / 1e6 if o['bytes'] else 0
    print(f"  {o['name']:14s} {o['ms']*1000:7.1f} us  {tf:6.0f} TF/s {gb:6.0f} GB/s  x{o['launches']}")
PY
done
