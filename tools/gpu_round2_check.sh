# round-2 GPU check: smoke, then the whole GPU suite
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1800 python -m pytest tests -q -m gpu -rs --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -c 1500 gpurun_out/smoke.log
grep -E "passed|failed|Error|SKIP" gpurun_out/pytest_gpu.log | tail -20
grep -A20 "slowest" gpurun_out/pytest_gpu.log | head -20
