#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cudnn --no-cfg1 > gpurun_out/bench_under_ncu.txt 2>&1
timeout 2400 python tools/bench_variants.py --steps 30 > gpurun_out/variants.jsonl 2> gpurun_out/variants.err
cat gpurun_out/pytest_gpu.txt; cut -c1-300 gpurun_out/bench.json; echo; cut -c1-300 gpurun_out/bench_ref.json; echo; cut -c1-250 gpurun_out/variants.jsonl | head -8
