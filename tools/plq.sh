tag=$1
python -m pytest tests -m gpu -x -q -k "frame or batch or ab_variants" 2>&1 | tail -1
python bench.py --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/${tag}.json; python tools/bench_summary.py gpurun_out/${tag}.json | head -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"label_pl" -s 2 -c 1 -o gpurun_out/${tag}_batch python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
