"""Dev: labeling kernel time vs frames per submit (2M edges, 512^2, PROPS props)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02612_b200 import LabelEngine  # noqa: E402
from workload.synth import SyntheticPRM, props_words  # noqa: E402

depth, E, props = 18, 2_000_000, int(os.environ.get("PROPS", "16"))
prm = SyntheticPRM(1, depth)
T = prm.words(0, E)
FR = [int(x) for x in os.environ.get("FRAMES", "1 2 4 8 16 32 64").split()]
P = props_words(4, depth, props, 0, max(FR))
eng = LabelEngine(devices=[0], profile=True)
eng.load_abstraction_words(E, 1 << depth, T.offsets, T.words, T.masks)
for frames in FR:
    ts = []
    for it in range(8):
        eng.submit_grid(1 << depth, props, P[:frames], frames)
        eng.wait()
        if it >= 2:
            st = eng.stage_times(0, 0)
            ts.append(st[1] + st[2])
    med = statistics.median(ts)
    print(f"props={props} frames={frames} summary+label_ms={med:.4f} per_frame_ms={med / frames:.4f} "
          f"edge_labels_per_s={E * frames / med * 1e3:.3g}")
