"""Dev sweep: single-frame labeling kernel time on config 3 (2M edges, 512^2,
16 props) for the current build/env knobs.  Prints median kernel ms."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02612_b200 import LabelEngine  # noqa: E402
from workload.synth import SyntheticPRM, props_words  # noqa: E402

depth, E, props = 18, 2_000_000, int(os.environ.get("PROPS", "16"))
prm = SyntheticPRM(1, depth)
T = prm.words(0, E)
P = props_words(4, depth, props, 0, 8)
eng = LabelEngine(devices=[0], profile=True)
eng.load_abstraction_words(E, 1 << depth, T.offsets, T.words, T.masks)
ts = []
for it in range(40):
    eng.submit_grid(1 << depth, props, P[it % 8], 1)
    eng.wait()
    if it >= 5:
        ts.append(eng.stage_times(0, 0)[2])
alg = 8 * int(eng.info().words) + 4 * (E + 1) + (1 << depth) * props // 8 + E * (2 if props <= 16 else 4)
med = statistics.median(ts)
print(f"{os.environ.get('TAG', '')} props={props} label_kernel_ms={med:.4f} min={min(ts):.4f} "
      f"GB/s={alg / med / 1e6:.0f} frac={alg / med / 1e6 / 6561.6:.3f}")
