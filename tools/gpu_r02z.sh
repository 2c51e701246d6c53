#!/bin/bash
# ncu of the ResNet-50 fp32 1x1 + shortcut convs on the sparse kernel (stage 1 and 2)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for spec in resnet50:fp32:s2b1.c3 resnet50:fp32:s2b1.c1 resnet50:fp32:s1b1.c3; do
  tag=$(echo $spec | tr ':.' '__')
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/$tag python tools/ncu_target.py $spec $tag > gpurun_out/ncu_$tag.txt 2>&1
  python tools/ncu_summary.py full gpurun_out/$tag.ncu-rep gpurun_out/r02_ncu_$tag.md gpurun_out/$tag.json > /dev/null 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/src_$tag.csv.gz
  rm -f gpurun_out/$tag.ncu-rep
  echo "== $tag"; sed -n 3,16p gpurun_out/r02_ncu_$tag.md; grep -A12 "stall reason" gpurun_out/r02_ncu_$tag.md
done
