"""Dev: single-frame and 8-frame kernel times on a config-5 per-GPU shard
(1M of the 8M edges = one of 8 GPUs, 1024^2 grid, PROPS props)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02612_b200 import LabelEngine  # noqa: E402
from workload.synth import SyntheticPRM, props_words  # noqa: E402

depth, E, props = 20, int(os.environ.get("ROWS", "1000000")), int(os.environ.get("PROPS", "64"))
prm = SyntheticPRM(1, depth)
T = prm.words(0, E)
P = props_words(4, depth, props, 0, 8)
eng = LabelEngine(devices=[0], profile=True)
eng.load_abstraction_words(E, 1 << depth, T.offsets, T.words, T.masks)
for frames in (1, 8):
    ts = []
    for it in range(15):
        eng.submit_grid(1 << depth, props, P[: frames] if frames > 1 else P[it % 8], frames)
        eng.wait()
        if it >= 3:
            ts.append(eng.stage_times(0, 0)[2])
    lb = 1 if props <= 8 else 2 if props <= 16 else 4 if props <= 32 else 8
    alg = 8 * int(eng.info().words) + 4 * (E + 1) + frames * ((1 << depth) * props // 8 + E * lb)
    med = statistics.median(ts)
    print(f"cfg5-shard rows={E} props={props} frames={frames} kernel_ms={med:.4f} "
          f"GB/s={alg / med / 1e6:.0f} frac={alg / med / 1e6 / 6450:.3f}")
