#!/bin/bash
# ncu --set full of the newer tensor-core schedules + the sparse binary16 first layer
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for spec in 64,64,3,1,32 512,512,3,1,2 64,64,3,1,32,pool; do
  tag=tc_$(echo $spec | tr ',' '_')
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/$tag python tools/ncu_tc.py $spec > gpurun_out/ncu_$tag.txt 2>&1
  python tools/ncu_summary.py full gpurun_out/$tag.ncu-rep gpurun_out/r02_ncu_$tag.md gpurun_out/tc.json > /dev/null 2>&1
  rm -f gpurun_out/$tag.ncu-rep
done
tag=vgg16_fp16_0
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/$tag python tools/ncu_target.py vgg16:fp16:0 $tag > gpurun_out/ncu_$tag.txt 2>&1
python tools/ncu_summary.py full gpurun_out/$tag.ncu-rep gpurun_out/r02_ncu_$tag.md gpurun_out/$tag.json > /dev/null 2>&1
rm -f gpurun_out/$tag.ncu-rep
for f in gpurun_out/r02_ncu_tc_64_64_3_1_32.md gpurun_out/r02_ncu_tc_512_512_3_1_2.md gpurun_out/r02_ncu_tc_64_64_3_1_32_pool.md gpurun_out/r02_ncu_vgg16_fp16_0.md; do echo "== $f"; sed -n 1,12p $f; grep -A8 "derived" $f; done
