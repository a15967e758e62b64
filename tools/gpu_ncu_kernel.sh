# ncu --set full of the first launches of one kernel (regex) in an eager AlexNet step; exports
# raw + source CSVs to gpurun_out/k_<tag>_*.   usage: bash tools/gpu_ncu_kernel.sh TAG REGEX COUNT [WORKLOAD]
T=$1; R=$2; C=${3:-1}; W=${4:-alexnet}
PSG_EAGER=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$R" -c $C \
  -o /tmp/k_$T -f python tools/op_traffic.py run --workload $W --ops /tmp/ops.json > gpurun_out/k_$T.log 2>&1
echo "ncu $T rc $?"
ncu -i /tmp/k_$T.ncu-rep --page details --csv > gpurun_out/k_${T}_details.csv 2>/dev/null
for i in $(seq 0 $(($C - 1))); do
  ncu -i /tmp/k_$T.ncu-rep --page source --csv --launch-skip $i --launch-count 1 --print-source sass > gpurun_out/k_${T}_src$i.csv 2>/dev/null
done
gzip -f gpurun_out/k_${T}_src*.csv
