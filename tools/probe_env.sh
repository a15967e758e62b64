# A/B the tcgen05 GEMM knobs on one workload: per-op profile per setting.
#   bash tools/probe_env.sh <workload> "ENV=1 ..." "ENV=2" ...
W=$1; shift
for cfg in "$@"; do
  name=$(echo "$W $cfg" | tr ' =' '__')
  env $cfg timeout 300 python bench.py --workload $W --profile-json gpurun_out/pr_$name.json > gpurun_out/pr_$name.log 2>&1
done
