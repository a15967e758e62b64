for cfg in "PSG_TC_PAIR=1" "PSG_TC_KPS=1" "PSG_TC_KPS=1 PSG_TC_PRODUCERS=2" "PSG_TC_PRODUCERS=2" "PSG_TC_PRODUCERS=1" "PSG_TC_KPS=4"; do
  name=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 300 python bench.py --workload alexnet --steps 3 --warmup 3 --profile-json gpurun_out/pr_$name.json > gpurun_out/pr_$name.log 2>&1
done
