# Multi-GPU round: the >= 2-GPU tests, the weight-average sweep (NVML NVLink counters are
# N/A on this pool: nvidia-smi nvlink -gt d is captured beside it), the overlapped-average
# check and the bench at N GPUs (torchrun, one process per GPU).   usage: bash tools/gpu_multi.sh N
N=${1:-2}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -k "gpus or multi_rank or two_gpus or k_gpus or overlapped" -rs > gpurun_out/pytest_multi_$N.log 2>&1
echo "pytest rc $?"; tail -4 gpurun_out/pytest_multi_$N.log
nvidia-smi nvlink -gt d > gpurun_out/nvlink_before_$N.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29511 tools/avg_sweep.py --sizes-mb 1,4,16,64,128,250 > gpurun_out/avg_sweep_${N}gpu.jsonl 2> gpurun_out/avg_sweep_${N}gpu.err
echo "sweep rc $?"; cat gpurun_out/avg_sweep_${N}gpu.jsonl | cut -c1-200
nvidia-smi nvlink -gt d > gpurun_out/nvlink_after_$N.txt 2>&1
for t in 1 50; do
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29520 + t)) tools/overlap_check.py --workload alexnet --tau $t --rounds 10 \
    > gpurun_out/overlap_alexnet_tau${t}_${N}gpu.json 2> gpurun_out/overlap_tau${t}_${N}gpu.err
  echo "overlap tau $t rc $?"; tail -1 gpurun_out/overlap_alexnet_tau${t}_${N}gpu.json
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --gpus $N > gpurun_out/bench_${N}gpu.json 2> gpurun_out/bench_${N}gpu.err
echo "bench rc $?"; tail -1 gpurun_out/bench_${N}gpu.json | cut -c1-400
