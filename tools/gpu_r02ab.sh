#!/bin/bash
# one TMA box per row window (xrow) vs one per pixel: tests, per-shape probe, networks
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_tc.py tests/test_gpu_dispatch.py -q -x 2>&1 | tail -3
for x in 0 1; do
  if [ $x = 0 ]; then export USC_NO_XROW=1; else unset USC_NO_XROW; fi
  timeout 600 python tools/tc_cfg_probe.py > gpurun_out/tc_cfg_xrow$x.jsonl 2>&1
  timeout 900 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg_xrow$x.jsonl 2> gpurun_out/disp.err
  timeout 900 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet_xrow$x.jsonl 2>> gpurun_out/disp.err
done
python - <<'PY'
import json
for x in (0, 1):
    print("xrow", x)
    for l in open(f"gpurun_out/tc_cfg_xrow{x}.jsonl"):
        try:
            d = json.loads(l)
        except Exception:
            continue
        print("  ", d["layer"], d.get("0/0"), d.get("4/1"), d.get("2/1"))
    for f in (f"gpurun_out/disp_vgg_xrow{x}.jsonl", f"gpurun_out/disp_resnet_xrow{x}.jsonl"):
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print("  ", f, d["dispatch"]["images_per_s"], d["dispatch"]["ms_per_step"])
PY
