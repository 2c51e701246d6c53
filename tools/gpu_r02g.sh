#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
BENCH_SHARE_GPU=1 BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 20 --warmup 3 --no-cudnn --no-cfg1 > gpurun_out/bench_2rank_shared.json 2> gpurun_out/bench_2rank.err
BENCH_SHARE_GPU=1 BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --global-batch 512 --steps 20 --warmup 3 --no-cudnn --no-cfg1 > gpurun_out/bench_2rank_strong.json 2>> gpurun_out/bench_2rank.err
timeout 600 python tools/sweep_sharded.py --points r50-1x1-64x256-32@0.9,r50-3x3-256x8@0.9 > gpurun_out/sweep_sharded.jsonl 2> gpurun_out/sweep_sharded.err
cat gpurun_out/pytest_gpu.txt; cut -c1-400 gpurun_out/bench.json; echo; cut -c1-700 gpurun_out/bench_2rank_shared.json gpurun_out/bench_2rank_strong.json; tail -3 gpurun_out/bench_2rank.err; cat gpurun_out/sweep_sharded.jsonl; tail -3 gpurun_out/sweep_sharded.err
