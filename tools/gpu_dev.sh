#!/bin/bash
# dev loop on the GPU box: parity tests, bench (no CPU baseline), optional ncu captures
tag=${1:-dev}; ncu_on=${2:-1}
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $out/${tag}_pytest.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc=$?"; tail -3 $out/${tag}_bench.err
python tools/bench_summary.py $out/${tag}_bench.json
if [ "$ncu_on" != "0" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"label_pl|label_batch" -s 2 -c 1 \
    -o $out/${tag}_batch python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/${tag}_ncu_batch.log 2>&1; echo "ncu batch rc=$?"
[ "$ncu_on" = "1" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:label_stream -s 5 -c 1 \
    -o $out/${tag}_stream python tools/sweep_stream.py > $out/${tag}_ncu_stream.log 2>&1; echo "ncu stream rc=$?"
fi
