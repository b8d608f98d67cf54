"""Dev: p50 single-frame latency (pinned host P -> labels in HBM, stage
events off) of BASELINE configs 1-3 (host clock, 150 frames after a warm-up),
plus the stage breakdown from a profiled pass.

  python tools/cfg_latency.py [1 2 3 5]     (5: the 1M-row per-GPU shard)
"""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1810_02612_b200 import LabelEngine
    from workload.synth import CONFIGS, SyntheticPRM, props_words

    for cfg in [int(x) for x in (sys.argv[1:] or ["1", "2", "3"])]:
        c = CONFIGS[cfg]
        depth, E, props = c["depth"], c["edges"], c["props"]
        if cfg == 5:
            E //= 8  # one GPU's shard of the 8-way row partition
        prm = SyntheticPRM(seed=1, depth=depth)
        T = prm.words(0, E)
        eng = LabelEngine(devices=[0], profile=False)
        eng.load_abstraction_words(E, 1 << depth, T.offsets, T.words, T.masks)
        nw = ((1 << depth) + 63) // 64
        frames = torch.from_numpy(props_words(3, depth, props, 0, 151).view(np.int64)).pin_memory()
        lat = []
        for q in range(151):
            t0 = time.perf_counter()
            eng.submit_grid(1 << depth, props, frames[q], 1)
            eng.wait()
            if q:
                lat.append((time.perf_counter() - t0) * 1e6)
        eng.set_profiling(True)
        st = []
        for q in range(31):
            eng.submit_grid(1 << depth, props, frames[q], 1)
            eng.wait()
            if q:
                st.append(eng.stage_times(0, 0))
        med = [statistics.median(x[i] for x in st) * 1e3 for i in range(3)]
        print(f"config {cfg}: E={E} depth={depth} props={props}: p50 {statistics.median(lat):.1f} us, "
              f"p99 {sorted(lat)[int(0.99 * (len(lat) - 1))]:.1f} us; stages (profiled) upload {med[0]:.1f} / "
              f"summary {med[1]:.1f} / label {med[2]:.1f} us")
        eng.close()


if __name__ == "__main__":
    main()
