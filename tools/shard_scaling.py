"""Dev: per-rank device time of the bench step (config 4: 64 frames, 32 props,
512^2) on the edge-row shard one of N GPUs would hold (2M/N rows), N = 1, 2, 4,
8 -- the compute side of strong scaling, measured on one GPU (P resident; the
per-step NCCL broadcast of P is not included).

  python tools/shard_scaling.py
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02612_b200 import LabelEngine  # noqa: E402
from workload.synth import SyntheticPRM, props_words  # noqa: E402

depth, E, props, F = 18, 2_000_000, 32, 64
prm = SyntheticPRM(1, depth)
P = torch.from_numpy(props_words(4, depth, props, 0, F).view("int64")).cuda()
base = None
for n in [int(x) for x in os.environ.get("NS", "1 2 4 8").split()]:
    rows = E // n
    off = int(float(os.environ.get("OFF", "0")) * E) // n * n  # shard start (fraction of E)
    T = prm.words(off, off + rows)
    eng = LabelEngine(devices=[0], profile=True)
    eng.load_abstraction_words(rows, 1 << depth, T.offsets, T.words, T.masks)
    ts = []
    for it in range(10):
        eng.submit_grid_device(1 << depth, props, P.data_ptr(), F)
        eng.wait()
        if it >= 3:
            st = eng.stage_times(0, 0)
            ts.append(st[1] + st[2])
    med = statistics.median(ts)
    base = base or med
    print(f"N={n} rows/rank={rows} first_row={off} summary_ms={statistics.median(eng.stage_times(0, b)[1] for b in range(5)):.4f} "
          f"step_ms={med:.4f} speedup={base / med:.2f} eff={base / med / n:.2f}", flush=True)
    eng.close()
