python tools/op_traffic.py run --workload alexnet --ops /tmp/o.json > /dev/null 2>&1 && \
PSG_EAGER=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 16 -c 3 -o /tmp/w -f python tools/op_traffic.py run --workload alexnet --ops /tmp/ops.json > gpurun_out/w.log 2>&1; echo rc $?
ncu -i /tmp/w.ncu-rep --page details --csv > gpurun_out/w_details.csv 2>/dev/null
for i in 0 1 2; do ncu -i /tmp/w.ncu-rep --page source --csv --launch-skip $i --launch-count 1 --print-source sass > gpurun_out/w_src$i.csv 2>/dev/null; done
gzip -f gpurun_out/w_src*.csv
