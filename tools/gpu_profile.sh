# Profiling pass on one B200: per-op live profiles, per-op DRAM traffic (ncu), launch list
# of the default bench command.  Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
for w in alexnet cifar10_quick googlenet; do
  timeout 600 python bench.py --workload $w --steps 3 --no-cpu-baseline \
      --profile-json gpurun_out/prof_$w.json > gpurun_out/benchp_$w.json 2>&1
  PSG_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/ops_$w.csv \
      python tools/op_traffic.py run --workload $w --ops gpurun_out/ops_$w.json > gpurun_out/ops_$w.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_cifar10_quick.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_alexnet.csv \
    python bench.py --workload alexnet --steps 1 --warmup 3 --tau 2 --no-cpu-baseline > gpurun_out/ncu_launch_a.log 2>&1
ls -la gpurun_out
