"""Generate tests/golden/sweep_*.npz by running the UNMODIFIED reference core.

Run here (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_sweep_golden.py

Inputs: trajectories from the reference's own build_abstraction (Rect region)
with the configuration of test_label.cpp:212-235 ("swept_volume_matrix equals
per-edge sweep_voxelize rows": 64 x 64 m x 4 s grid, depth 12, seed 17, 50
edges), plus a denser 500-edge set on a depth-18 grid.  Expected outputs:
the reference's swept_volume_matrix (label.cpp:75-116), through
oracle/_ref/libltlgrid_ref.so.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefCore  # noqa: E402

FOOTPRINT = (4.6, 2.0, -1.4)  # FootprintSpec defaults (abstraction.hpp:58-62)
CASES = {
    # name: (abstraction kwargs, depth, lo, hi)
    "sweep_test_label": (dict(target_edges=50, seed=17), 12, (0.0, 0.0, 0.0), (64.0, 64.0, 4.0)),
    "sweep_d18": (dict(target_edges=500, seed=5), 18, (0.0, 0.0, 0.0), (64.0, 64.0, 4.0)),
}


def main():
    ref = RefCore()
    for name, (kw, depth, lo, hi) in CASES.items():
        off, smp = ref.abstraction(**kw)
        rows, cols = ref.swept_volume(depth, lo, hi, FOOTPRINT, off, smp, workers=2)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), sample_off=off, samples=smp, depth=depth,
                            lo=np.array(lo), hi=np.array(hi), footprint=np.array(FOOTPRINT), row_offsets=rows,
                            col_indices=cols)
        print(name, off.size - 1, "edges", smp.shape[0], "samples", cols.size, "nnz")


if __name__ == "__main__":
    main()
