#!/bin/bash
# ncu --set full of two tensor-core shapes: 1x1 64->256 @32 with shortcut, 3x3 128->128 @16
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for spec in 64,256,1,1,32,res 128,128,3,1,16; do
  tag=$(echo $spec | tr ',' '_')
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/tc_$tag python tools/ncu_tc.py $spec > gpurun_out/ncu_tc_$tag.txt 2>&1
  python tools/ncu_summary.py full gpurun_out/tc_$tag.ncu-rep gpurun_out/r02_ncu_tc_$tag.md gpurun_out/tc.json > /dev/null 2>&1
  ncu -i gpurun_out/tc_$tag.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/tc_raw_$tag.csv
  ncu -i gpurun_out/tc_$tag.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/tc_src_$tag.csv.gz
  rm -f gpurun_out/tc_$tag.ncu-rep
done
head -50 gpurun_out/r02_ncu_tc_*.md
