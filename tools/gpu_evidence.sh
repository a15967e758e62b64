# Round evidence on one GPU: the default bench line, per-op DRAM / tensor-pipe counters of one
# AlexNet and one cifar10_quick step (ncu, eager launches), and the launch list of the
# default bench command.   usage: bash tools/gpu_evidence.sh
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_1gpu.json 2> gpurun_out/bench_1gpu.err; echo "bench rc $?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed
for W in alexnet cifar10_quick; do
  python tools/op_traffic.py run --workload $W --ops /tmp/plain_$W.json > /dev/null 2>&1 && \
  PSG_EAGER=1 timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ops_$W.csv \
    python tools/op_traffic.py run --workload $W --ops gpurun_out/ops_$W.json > gpurun_out/ncu_ops_$W.log 2>&1
  echo "ncu ops $W rc $?"
done
PSG_EAGER=1 timeout 1500 ncu --metrics $M --clock-control none -c 300 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench rc $?"
tail -c 600 gpurun_out/bench_1gpu.json
