# ncu --set full capture of one AlexNet training step's kernels (eager launches), exported
# to CSV on the box (the .ncu-rep is kept only when small).  Run only after the bench
# exits 0 without ncu.   usage: bash tools/gpu_ncu_full.sh WORKLOAD SKIP COUNT [KERNEL_REGEX]
set -x
mkdir -p gpurun_out
W=${1:-alexnet}
KREG=${4:-.}
PSG_EAGER=1 timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"$KREG" --launch-skip ${2:-160} --launch-count ${3:-80} -o /tmp/full_$W -f \
  python tools/op_traffic.py run --workload $W --ops gpurun_out/full_ops_$W.json > gpurun_out/full_$W.log 2>&1
tail -3 gpurun_out/full_$W.log
ncu -i /tmp/full_$W.ncu-rep --page raw --csv > gpurun_out/full_${W}_raw.csv 2>/dev/null
ncu -i /tmp/full_$W.ncu-rep --page details --csv > gpurun_out/full_${W}_details.csv 2>/dev/null
ls -la /tmp/full_$W.ncu-rep gpurun_out/full_${W}_*.csv
sz=$(stat -c %s /tmp/full_$W.ncu-rep)
if [ "$sz" -lt 40000000 ]; then cp /tmp/full_$W.ncu-rep gpurun_out/; fi
