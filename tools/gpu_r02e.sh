#!/bin/bash
# Round-2 GPU session E: dispatcher tuned states, ncu evidence (summarised on the box,
# reports deleted but the top kernel's), launch list.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export TUNED_OUT=gpurun_out
timeout 900 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet.jsonl 2> gpurun_out/disp.err
timeout 600 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg.jsonl 2>> gpurun_out/disp.err
NCU="ncu --set full --import-source on --clock-control none --profile-from-start off -c 1"
for spec in vgg16:fp32:9 vgg16:fp16:5 vgg16:cb4:5 vgg16:int8:5 resnet50:fp16:s0b0.c3 resnet50:fp16:s0b1.c1 resnet50:fp32:s0b0.c3; do
  tag=$(echo $spec | tr ':.' '__')
  timeout 600 $NCU -o gpurun_out/$tag python tools/ncu_target.py $spec $tag > gpurun_out/ncu_$tag.txt 2>&1
  python tools/ncu_summary.py full gpurun_out/$tag.ncu-rep gpurun_out/r02_ncu_$tag.md gpurun_out/$tag.json > /dev/null 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page source --csv > gpurun_out/src_$tag.csv 2>/dev/null
  [ "$tag" != "vgg16_fp32_9" ] && rm -f gpurun_out/$tag.ncu-rep
done
gzip -f gpurun_out/src_*.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cudnn --no-cfg1 > gpurun_out/bench_under_ncu.txt 2>&1
du -sh gpurun_out; ls -la gpurun_out | head -40
