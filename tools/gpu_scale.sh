# Multi-GPU bench lines (one box, N GPUs): usage bash tools/gpu_scale.sh "2 4" "alexnet cifar10_quick googlenet"
set -x
mkdir -p gpurun_out
NS=${1:-"2 4"}; WL=${2:-"cifar10_quick alexnet googlenet"}
for n in $NS; do
  for w in $WL; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n --workload $w > gpurun_out/scale_${n}_$w.json 2> gpurun_out/scale_${n}_$w.err
    tail -1 gpurun_out/scale_${n}_$w.json | cut -c1-400
  done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${n} --master-addr 127.0.0.1 \
  --master-port 29600 bench.py --gpus ${n} --impl reference --steps 2 --warmup 1 > gpurun_out/scale_${n}_reference.json 2> gpurun_out/scale_${n}_reference.err
tail -1 gpurun_out/scale_${n}_reference.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${n} --master-addr 127.0.0.1 \
  --master-port 29700 tools/avg_sweep.py > gpurun_out/avg_sweep_${n}gpu.jsonl 2> gpurun_out/avg_sweep.err || true
cat gpurun_out/avg_sweep_${n}gpu.jsonl
