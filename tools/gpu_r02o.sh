#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/tc python tools/ncu_tc.py > gpurun_out/ncu_tc.txt 2>&1
python tools/ncu_summary.py full gpurun_out/tc.ncu-rep gpurun_out/r02_ncu_tc.md gpurun_out/tc.json > /dev/null 2>&1
ncu -i gpurun_out/tc.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k,x in zip(h,v):
    if any(s in k for s in ['pipe_tensor','tensor_op','gpu__time_duration.sum','dram__bytes','lts__t_bytes.sum','sm__throughput.avg.pct']): print(k, x)
" > gpurun_out/tc_metrics.txt
rm -f gpurun_out/tc.ncu-rep
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_gpu.txt; head -30 gpurun_out/tc_metrics.txt; cut -c1-300 gpurun_out/bench.json
