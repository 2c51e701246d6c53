#!/bin/bash
# Round-2 GPU session B: register-window kernel correctness + probe, dispatcher tests.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "layer_configs or random_corpus_bitwise" 2>&1 | tail -25 > gpurun_out/pytest_tiles.txt
timeout 600 python -m pytest tests/test_gpu_dispatch.py -q 2>&1 | tail -40 > gpurun_out/pytest_dispatch.txt
timeout 900 python tools/bw_probe.py > gpurun_out/bw_probe.jsonl 2> gpurun_out/bw_probe.err
cat gpurun_out/pytest_tiles.txt gpurun_out/pytest_dispatch.txt; cut -c1-1500 gpurun_out/bw_probe.jsonl; tail -5 gpurun_out/bw_probe.err
