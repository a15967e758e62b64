# ncu --set full (source-level) of AlexNet's conv GEMMs: conv1-3 fprop and conv2 wgrad/dgrad
# of the first eager training step.  Exports raw + source pages as CSV (gpurun_out/full_*).
set -x
mkdir -p gpurun_out
for spec in "fwd 0 3" "c2bwd 20 2"; do
  set -- $spec
  PSG_EAGER=1 timeout 1200 ncu --set full --import-source on --clock-control none \
    -k regex:tc_gemm_kernel -s $2 -c $3 -o /tmp/full_$1 -f \
    python tools/op_traffic.py run --workload alexnet --ops /tmp/ops.json > gpurun_out/full_$1.log 2>&1
  echo ncu $1 rc $?
  ncu -i /tmp/full_$1.ncu-rep --page raw --csv > gpurun_out/full_$1_raw.csv 2>/dev/null
  ncu -i /tmp/full_$1.ncu-rep --page details --csv > gpurun_out/full_$1_details.csv 2>/dev/null
  for i in $(seq 0 $(($3 - 1))); do
    ncu -i /tmp/full_$1.ncu-rep --page source --csv --launch-skip $i --launch-count 1 --print-source sass > gpurun_out/full_$1_src$i.csv 2>/dev/null
  done
done
gzip -f gpurun_out/full_*_src*.csv
ls -la gpurun_out/
