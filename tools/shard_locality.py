"""Dev: config-4 step time of a 1/N shard whose rows are (a) a contiguous range
of the original order vs (b) the N-th part of the rows sorted by median swept
word (z-order), i.e. a spatial shard.  Tests whether the 8-GPU per-rank cost
is set by the locality density of the rows.

  NS="8" python tools/shard_locality.py
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02612_b200 import LabelEngine  # noqa: E402
from workload.synth import SyntheticPRM, props_words  # noqa: E402

depth, E, props, F = 18, 2_000_000, 32, 64
prm = SyntheticPRM(1, depth)
P = torch.from_numpy(props_words(4, depth, props, 0, F).view("int64")).cuda()
T = prm.words(0, E)
off = T.offsets.astype(np.int64)
med = T.words[off[:-1] + (off[1:] - off[:-1]) // 2]
order = np.argsort(med, kind="stable")


def subset(rows):
    cnt = off[rows + 1] - off[rows]
    so = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(cnt, out=so[1:])
    idx = np.repeat(off[rows] - so[:-1], cnt) + np.arange(so[-1])
    return so.astype(np.uint64), T.words[idx], T.masks[idx]


def step_ms(rows):
    so, w, m = subset(rows)
    eng = LabelEngine(devices=[0], profile=True)
    eng.load_abstraction_words(len(rows), 1 << depth, so, w, m)
    ts = []
    for it in range(10):
        eng.submit_grid_device(1 << depth, props, P.data_ptr(), F)
        eng.wait()
        if it >= 3:
            st = eng.stage_times(0, 0)
            ts.append(st[1] + st[2])
    eng.close()
    return statistics.median(ts)


for n in [int(x) for x in os.environ.get("NS", "8").split()]:
    k = E // n
    for part in (0, n // 2):
        a = step_ms(np.arange(part * k, (part + 1) * k))
        b = step_ms(np.sort(order[part * k:(part + 1) * k]))
        print(f"N={n} part={part}: contiguous rows {a:.4f} ms, z-sorted spatial shard {b:.4f} ms "
              f"(ideal {2.53 / n:.4f})", flush=True)
