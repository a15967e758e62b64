# Round-end bench lines only (tests, smoke, the three workloads, the reference arm).
set -x
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for w in cifar10_quick alexnet googlenet; do
  timeout 900 python bench.py --workload $w --profile-json $O/prof_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log
for w in cifar10_quick alexnet googlenet reference; do tail -1 $O/bench_$w.json | cut -c1-200; done
