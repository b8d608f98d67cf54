"""Parity of the labeling path under the current environment's A/B knobs
(LTLG_STREAM64, LTLG_BATCH64, LTLG_STREAM_CFG, LTLG_STREAM_TABLE, LTLG_PROPLANE,
LTLG_WORDMAJOR, LTLG_WM1, LTLG_TC): run by
tests/test_gpu_parity.py in subprocesses, since the knobs are read once per
process.  Exits 0 iff every case is bit-exact against the CPU oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402  (checker only)
from paper_1810_02612_b200 import LabelEngine, LabelMatrix  # noqa: E402
from workload.synth import SyntheticPRM, props_words  # noqa: E402

O = Oracle()
bad = 0
for depth, E, props, F in [(12, 9_000, 4, 3), (14, 20_000, 16, 2), (16, 30_000, 32, 3), (14, 12_000, 64, 2),
                           (14, 15_000, 20, 40), (13, 8_000, 7, 17), (20, 30_000, 64, 1), (20, 30_000, 40, 2)]:
    prm = SyntheticPRM(seed=depth + props, depth=depth)
    off, idx = prm.csr(0, E)
    t = prm.words(0, E)
    P = props_words(props, depth, props, 0, F)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    for frames in (1, F):
        eng.submit_grid(1 << depth, props, P[:frames], frames)
        for f in range(frames):
            want = O.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f])
            if not eng.get_labels(f) == LabelMatrix(E, props, want):
                print("MISMATCH", depth, E, props, frames, f)
                bad += 1
    eng.close()
print("ab-parity", {k: v for k, v in os.environ.items() if k.startswith("LTLG_")}, "bad", bad)
sys.exit(1 if bad else 0)
