#!/bin/bash
# Full evidence pass on the GPU box: parity tests, smoke, bench (both arms),
# ncu launch list of the bench command, ncu --set full of the two labeling
# kernels.  Everything lands in gpurun_out/<tag>_*.
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/${tag}_gpu.txt 2>&1
nproc > $out/${tag}_nproc.txt; lscpu | grep -E 'Model name|^CPU\(s\)|Thread' >> $out/${tag}_nproc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $out/${tag}_smoke.log
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc=$?"; tail -3 $out/${tag}_bench.err
python tools/bench_summary.py $out/${tag}_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err; echo "ref rc=$?"; cat $out/${tag}_bench_ref.json
# launch list (cold-cache, serialised): shares only
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv \
    python bench.py --quick --steps 3 --warmup 3 --no-cpu-baseline --no-cfg5 > $out/${tag}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
# full captures of the labeling kernels (tools/wm_ab.py child mode: the bench's inputs, P resident)
timeout 900 env WM_CHILD=1 OUT=/tmp/wm.npy ncu --set full --clock-control none --import-source on -k regex:"label_wm|label_pl" -s 2 -c 1 \
    -o $out/${tag}_batch python tools/wm_ab.py > $out/${tag}_ncu_batch.log 2>&1; echo "ncu batch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:label_stream -s 5 -c 1 \
    -o $out/${tag}_stream python tools/sweep_stream.py > $out/${tag}_ncu_stream.log 2>&1; echo "ncu stream rc=$?"
timeout 900 env WM_CHILD=1 CFG=5 OUT=/tmp/wm.npy ncu --set full --clock-control none --import-source on -k regex:"label_wm" -s 2 -c 1 \
    -o $out/${tag}_cfg5batch python tools/wm_ab.py > $out/${tag}_ncu_cfg5batch.log 2>&1; echo "ncu cfg5 batch rc=$?"
timeout 900 env WM_CHILD=1 CFG=5 SINGLE=1 OUT=/tmp/wm.npy ncu --set full --clock-control none --import-source on -k regex:"label_wm1|label_stream" -s 3 -c 1 \
    -o $out/${tag}_cfg5stream python tools/wm_ab.py > $out/${tag}_ncu_cfg5stream.log 2>&1; echo "ncu cfg5 stream rc=$?"
timeout 900 env WM_CHILD=1 CFG=5 LTLG_TC=1 LTLG_DEV_SO=paper_1810_02612_b200/_lib/libltlgrid_gpu_ab.so OUT=/tmp/wm.npy ncu --set full --clock-control none --import-source on -k regex:"label_tc" -s 1 -c 1 \
    -o $out/${tag}_cfg5tc python tools/wm_ab.py > $out/${tag}_ncu_cfg5tc.log 2>&1; echo "ncu cfg5 tc rc=$?"
ls -la $out
