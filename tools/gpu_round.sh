#!/bin/bash
# One GPU session: tests, bench (autotuned tiles dumped), launch list, ncu of the top kernel.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python tools/check_tiles.py 64 2>&1 | tail -2 > gpurun_out/check.txt
timeout 600 python bench.py --retune --dump-configs gpurun_out/tuned.json > gpurun_out/bench.json 2> gpurun_out/bench.err
L=$(python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['roofline']['kernel'].split('layer ')[1].split(' ')[0])")
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --configs gpurun_out/tuned.json --no-cpu-baseline --no-cudnn > gpurun_out/bench_under_ncu.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bi -s 13 -c 1 -o gpurun_out/top_kernel \
    python tools/ncu_layer.py $L gpurun_out/tuned.json > gpurun_out/ncu_top.txt 2>&1
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:k_bi -o gpurun_out/traffic \
    python tools/ncu_traffic.py gpurun_out/tuned.json > gpurun_out/ncu_traffic.txt 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/check.txt; cat gpurun_out/bench.json | cut -c1-3000
