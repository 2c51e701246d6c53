#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python tools/bw_layer_probe.py fp32 1,3,5,8 > gpurun_out/bw_layers_fp32.jsonl 2> gpurun_out/bw_layers.err
timeout 300 python tools/bw_layer_probe.py fp16 5 > gpurun_out/bw_layers_fp16.jsonl 2>> gpurun_out/bw_layers.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bw -s 2 -c 1 -o gpurun_out/bw_l5 \
  python tools/ncu_cfg.py 5 kernel=3 window=1 pix_per_thread=4 rows_per_thread=1 ch_per_cta=48 threads=256 pixel_warps=2 samples_per_cta=64 stages=2 > gpurun_out/ncu_bw.txt 2>&1
cut -c1-600 gpurun_out/bw_layers_fp32.jsonl gpurun_out/bw_layers_fp16.jsonl; tail -3 gpurun_out/bw_layers.err; tail -3 gpurun_out/ncu_bw.txt
