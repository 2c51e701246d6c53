#!/bin/bash
# round-end validation: full GPU suite, smoke, bench (+ reference arm), launch list, ncu of the
# dominant kernel, every variant with the committed states
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cudnn --no-cfg1 > gpurun_out/bench_under_ncu.txt 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/r02_launches.md > /dev/null 2>&1
tag=vgg16_fp32_5
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/$tag \
    python tools/ncu_target.py vgg16:fp32:5 $tag > gpurun_out/ncu_$tag.txt 2>&1
python tools/ncu_summary.py full gpurun_out/$tag.ncu-rep gpurun_out/r02_ncu_$tag.md gpurun_out/$tag.json > /dev/null 2>&1
rm -f gpurun_out/$tag.ncu-rep
timeout 2400 python tools/bench_variants.py --steps 30 > gpurun_out/variants.jsonl 2> gpurun_out/variants.err
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt; cut -c1-300 gpurun_out/bench.json; echo; cut -c1-300 gpurun_out/bench_ref.json; echo
head -12 gpurun_out/r02_launches.md; head -12 gpurun_out/r02_ncu_$tag.md
cut -c1-250 gpurun_out/variants.jsonl | head -8; tail -n 3 gpurun_out/variants.err; tail -n 3 gpurun_out/bench.err
