#!/bin/bash
# dev loop on the GPU box: parity tests then a bench line (no CPU baseline)
tag=${1:-dev}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$tag.log
python bench.py --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_$tag.err
python tools/bench_summary.py gpurun_out/bench_$tag.json
