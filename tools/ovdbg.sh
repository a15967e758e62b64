export NCCL_DEBUG=WARN
run() { timeout 120 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/overlap_check.py --tau $2 --rounds 20 --only $3 ${4:+--workload $4} > /tmp/o.log 2>&1; echo "== tau $2 $3 $4 rc $?"; grep -E "bitwise|Error|error" /tmp/o.log | head -4; }
run 29601 10 overlapped
run 29602 1 both
run 29603 10 both
run 29604 10 both alexnet
timeout 600 python -m pytest tests/test_multi_rank.py -q -x 2>&1 | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/bench_2gpu.json 2> gpurun_out/bench_2gpu.err
echo "bench rc $?"; tail -1 gpurun_out/bench_2gpu.json | cut -c1-900
