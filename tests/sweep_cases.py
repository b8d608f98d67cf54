"""Trajectory inputs for the swept-volume parity tests (test input generators,
not an oracle): seeded straight / turning motions as State5 samples
(px, py, heading, speed, tau; abstraction.hpp:16-22), plus the reference
unit-test cases of test_abstraction.cpp:145-232."""
from __future__ import annotations

import numpy as np

FOOTPRINT = (4.6, 2.0, -1.4)  # FootprintSpec defaults (abstraction.hpp:58-62)


def random_motions(seed: int, edges: int, lo=(0.0, 0.0, 0.0), hi=(64.0, 64.0, 4.0), samples=41, step=0.0125,
                   margin=6.0, empty_every: int = 0):
    """Edges of `samples` states along constant-curvature arcs inside the box
    (shrunk by `margin`), tau advancing by `step`.  Every `empty_every`-th
    edge has no samples."""
    rng = np.random.default_rng(seed)
    rows = []
    for e in range(edges):
        if empty_every and e % empty_every == empty_every - 1:
            rows.append(np.zeros((0, 5)))
            continue
        n = samples
        x0 = rng.uniform(lo[0] + margin, hi[0] - margin)
        y0 = rng.uniform(lo[1] + margin, hi[1] - margin)
        h0 = rng.uniform(-np.pi, np.pi)
        v = rng.uniform(0.0, 8.0)
        k = rng.uniform(-0.3, 0.3)
        t0 = rng.uniform(lo[2], hi[2] - n * step - 1e-9)
        t = np.arange(n) * step
        h = h0 + k * v * t
        px = x0 + np.cumsum(np.r_[0.0, v * step * np.cos(h[:-1])])
        py = y0 + np.cumsum(np.r_[0.0, v * step * np.sin(h[:-1])])
        px = np.clip(px, lo[0] + margin, hi[0] - margin)
        py = np.clip(py, lo[1] + margin, hi[1] - margin)
        hw = (h + np.pi) % (2 * np.pi) - np.pi
        rows.append(np.stack([px, py, hw, np.full(n, v), t0 + t], axis=1))
    return flatten(rows)


def flatten(rows):
    off = np.zeros(len(rows) + 1, dtype=np.uint64)
    if rows:
        off[1:] = np.cumsum([r.shape[0] for r in rows])
    smp = np.concatenate(rows) if rows else np.zeros((0, 5))
    return off, np.ascontiguousarray(smp, dtype=np.float64).reshape(-1, 5)


def axis_aligned(seed: int, edges: int, depth: int, lo=(0.0, 0.0, 0.0), hi=(64.0, 64.0, 4.0)):
    """Headings 0 / +-pi/2 / pi and centres on cell faces: the SAT test's
    strict inequalities meet equality (shared faces must not count)."""
    rng = np.random.default_rng(seed)
    bits = [depth // 3 + (a < depth % 3) for a in range(3)]
    w = [(hi[a] - lo[a]) / (1 << bits[a]) for a in range(3)]
    rows = []
    for _ in range(edges):
        n = int(rng.integers(1, 12))
        cx = lo[0] + w[0] * rng.integers(8 / w[0] + 2, (hi[0] - 8) / w[0] - 2, size=n)
        cy = lo[1] + w[1] * rng.integers(8 / w[1] + 2, (hi[1] - 8) / w[1] - 2, size=n)
        h = rng.choice([0.0, np.pi / 2, -np.pi / 2, np.pi], size=n)
        tau = lo[2] + w[2] * rng.integers(0, (1 << bits[2]) - 1, size=n) + rng.choice([0.0, 0.5 * w[2]], size=n)
        rows.append(np.stack([cx, cy, h, np.zeros(n), tau], axis=1))
    return flatten(rows)
