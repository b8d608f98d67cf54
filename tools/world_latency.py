"""p50 single-frame latency from a world-frame perception grid (north_star
subsystem 2): pinned host world grid -> vehicle-frame P resampled on the GPU
(ltlg_submit_world_grid) -> labels resident in HBM, config 3 (2M edges,
512^2 vehicle grid, 16 props) with a 1024^2 world grid and a random pose per
frame.  Host clock, 150 frames after one warm-up.

  python tools/world_latency.py [--frames 150]
"""
import argparse
import json
import math
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=150)
    a = ap.parse_args()
    import torch

    from paper_1810_02612_b200 import LabelEngine
    from workload.synth import SyntheticPRM, props_words

    depth, E, props = 18, 2_000_000, 16
    prm = SyntheticPRM(seed=1, depth=depth)
    T = prm.words(0, E)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, T.offsets, T.words, T.masks)
    vehicle = (depth, -40.0, 40.0, -40.0, 40.0)
    wdepth = 20
    world = (wdepth, -100.0, 100.0, -100.0, 100.0)
    W = torch.from_numpy(props_words(9, wdepth, props, 0, 1)[0].view(np.int64)).pin_memory()
    rng = np.random.default_rng(1)
    lat = []
    for q in range(-1, a.frames):
        th = rng.uniform(-math.pi, math.pi)
        pose = [(rng.uniform(-30, 30), rng.uniform(-30, 30), math.cos(th), math.sin(th))]
        t0 = time.perf_counter()
        eng.submit_world_grid(vehicle, world, props, W, pose)
        eng.wait()
        if q >= 0:
            lat.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"what": "pinned host world grid (1024^2, 16 props) -> resample -> labels in HBM, config 3",
                      "p50_ms": statistics.median(lat), "p99_ms": sorted(lat)[int(0.99 * (len(lat) - 1))],
                      "frames": a.frames, "world_bytes": int(W.numel() * 8)}))


if __name__ == "__main__":
    main()
