# Round-end evidence on one B200: GPU tests, smoke, bench lines (3 workloads + reference
# arm), per-op DRAM traffic captures, the default bench's launch list, and an ncu --set full
# capture of one AlexNet step (CSV export).  Everything lands in gpurun_out/final/.
set -x
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for w in cifar10_quick alexnet googlenet; do
  timeout 900 python bench.py --workload $w --profile-json $O/prof_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for w in cifar10_quick alexnet googlenet; do
  PSG_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/ops_$w.csv \
    python tools/op_traffic.py run --workload $w --ops $O/ops_$w.json > $O/ops_$w.log 2>&1
done
PSG_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file $O/launches_cifar10_quick.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
PSG_EAGER=1 timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"tc_gemm|pool|lrn|s2d_x|sgd|gather|relu|dropout|softmax|bias_grad|split_reduce|dgrad_wt" \
  --launch-skip 0 --launch-count 60 -o /tmp/full_alexnet -f \
  python tools/op_traffic.py run --workload alexnet --ops $O/full_ops_alexnet.json > $O/full_alexnet.log 2>&1
ncu -i /tmp/full_alexnet.ncu-rep --page raw --csv > $O/full_alexnet_raw.csv 2>/dev/null
ls -la $O
tail -2 $O/pytest_gpu.log; cat $O/smoke.log | tail -1
for w in cifar10_quick alexnet googlenet reference; do tail -1 $O/bench_$w.json | cut -c1-300; done
