"""Dev: per-rank device time of the bench step (config 4: 64 frames, 32 props,
512^2) on each of the N spatial edge-row shards (bench.spatial_shard: rows
sorted by median swept word, cut into N word-balanced parts) that N GPUs would
hold, N = 1, 2, 4, 8 -- the compute side of strong scaling, measured on one GPU
(P resident; the per-step NCCL broadcast of P is not included).  Prints the
max over the ranks (what bench.py's max-over-ranks timing sees) and the mean.

  python tools/shard_scaling.py            (NS="1 8" ROWS=113: ranks, word-major task rows)
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1810_02612_b200 import LabelEngine  # noqa: E402
from workload.synth import SyntheticPRM, props_words  # noqa: E402

depth, E, props, F = 18, 2_000_000, 32, 64
prm = SyntheticPRM(1, depth)
P = torch.from_numpy(props_words(1, depth, props, 0, F).view("int64")).cuda()
T = prm.words(0, E)
base = None
pbase = [None]
for n in [int(x) for x in os.environ.get("NS", "1 2 4 8").split()]:
    per, summ, pipe = [], [], []
    for r in range(n):
        ids, so, w, m = bench.spatial_shard(T.offsets, T.words, T.masks, r, n)
        eng = LabelEngine(devices=[0], profile=True, task_rows=int(os.environ.get("ROWS", "0")))
        eng.load_abstraction_words(len(ids), 1 << depth, so, w, m)
        ts, ss = [], []
        for it in range(10):
            eng.submit_grid_device(1 << depth, props, P.data_ptr(), F)
            eng.wait()
            if it >= 3:
                st = eng.stage_times(0, 0)
                ts.append(st[1] + st[2])
                ss.append(st[1])
        # pipelined steps (the summary of step k+1 during the labelling of step
        # k, as bench.py runs them): event time over 20 async submits
        st_ = torch.cuda.ExternalStream(eng.stream())
        rdy = torch.cuda.Event()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st_)
        rdy.record(st_)
        for it in range(20):
            eng.submit_grid_device(1 << depth, props, P.data_ptr(), F, ready_event=rdy.cuda_event)
        e1.record(st_)
        e1.synchronize()
        pipe.append(e0.elapsed_time(e1) / 20)
        eng.close()
        per.append(statistics.median(ts))
        summ.append(statistics.median(ss))
    mx = max(per)
    base = base or mx
    print(f"N={n} rows/rank={E // n} step_ms max={mx:.4f} mean={statistics.mean(per):.4f} "
          f"speedup(max)={base / mx:.2f} eff={base / mx / n:.2f} (summary kernel mean {statistics.mean(summ):.4f}); "
          f"pipelined step max={max(pipe):.4f} speedup={pbase[0] / max(pipe) if pbase[0] else 1:.2f}", flush=True)
    pbase[0] = pbase[0] or max(pipe)
