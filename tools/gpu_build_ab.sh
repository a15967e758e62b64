# A/B of a compile-time flag: bash tools/gpu_build_ab.sh "-DFLAG" WORKLOAD
set -x
mkdir -p gpurun_out
W=${2:-alexnet}
timeout 600 python bench.py --workload $W --steps 5 --no-cpu-baseline --profile-json gpurun_out/bab_${W}_0.json > gpurun_out/bab_${W}_0.out 2>&1
make -s -C paper_1511_06051_b200/csrc clean; make -s -j16 -C paper_1511_06051_b200/csrc EXTRA_NVFLAGS="$1"
timeout 600 python bench.py --workload $W --steps 5 --no-cpu-baseline --profile-json gpurun_out/bab_${W}_1.json > gpurun_out/bab_${W}_1.out 2>&1
tail -c 300 gpurun_out/bab_${W}_0.out; tail -c 300 gpurun_out/bab_${W}_1.out
