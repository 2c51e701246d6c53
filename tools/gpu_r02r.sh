#!/bin/bash
# re-search the binary16 dispatch states with the current tensor-core backend
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RETUNE_DISPATCH=1
timeout 1500 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet.jsonl 2> gpurun_out/disp.err
timeout 900 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg.jsonl 2>> gpurun_out/disp.err
cut -c1-400 gpurun_out/disp_resnet.jsonl gpurun_out/disp_vgg.jsonl; tail -3 gpurun_out/disp.err; ls gpurun_out/*dispatch*
