#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export TUNED_OUT=gpurun_out RETUNE_DISPATCH=1
timeout 1200 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet.jsonl 2> gpurun_out/disp.err
timeout 900 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg.jsonl 2>> gpurun_out/disp.err
python - <<'PY'
import json
for f in ["gpurun_out/disp_resnet.jsonl", "gpurun_out/disp_vgg.jsonl"]:
    for l in open(f):
        d = json.loads(l); dd = d.get("dispatch", {})
        print(d["variant"], d["images_per_s"], "dispatch", dd.get("images_per_s"), dd.get("speedup_vs_cudnn"), dd.get("pick"), dd.get("search"), dd.get("backends"))
PY
tail -3 gpurun_out/disp.err
