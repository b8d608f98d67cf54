"""Dev A/B: config-4 batched step (2M edges x 64 frames, 512^2, 32 props, P
resident) with the word-major kernel at several task sizes vs the pair-major
prop-lane kernel (LTLG_WORDMAJOR=0).  Prints summary / label kernel ms (stage
events on the launching stream) and checks a row sample against the first
variant's labels.

  python tools/wm_ab.py            # all variants, one process each
  CFG=5 python tools/wm_ab.py      # config-5 shard (1M rows, 1024^2, 64 props)
  WM_CHILD=1 OUT=x.npy [CFG=5] [SINGLE=1] python tools/wm_ab.py   # one variant (profilers)
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one():
    import numpy as np
    import torch

    from paper_1810_02612_b200 import LabelEngine
    from workload.synth import SyntheticPRM, props_words

    cfg = int(os.environ.get("CFG", "4"))
    depth, E, props, F = (18, 2_000_000, 32, 64) if cfg == 4 else (20, 1_000_000, 64, 64)
    props = int(os.environ.get("PROPS", props))
    prm = SyntheticPRM(1, depth)
    P = torch.from_numpy(props_words(1, depth, props, 0, F).view("int64")).cuda()
    T = prm.words(0, E)
    eng = LabelEngine(devices=[0], profile=True, task_rows=int(os.environ.get("ROWS", "0")))
    eng.load_abstraction_words(E, 1 << depth, T.offsets, T.words, T.masks)
    ts, ss = [], []
    if os.environ.get("SINGLE"):  # single frames (the single-frame kernel; also for profilers)
        for it in range(40):
            eng.submit_grid_device(1 << depth, props, P[it % F].data_ptr(), 1)
            eng.wait()
            if it >= 8:
                st = eng.stage_times(0, 0)
                ss.append(st[1])
                ts.append(st[2])
        print(json.dumps({"summary_ms": statistics.median(ss), "label_ms": statistics.median(ts)}))
        eng.close()
        return
    for it in range(12):
        eng.submit_grid_device(1 << depth, props, P.data_ptr(), F)
        eng.wait()
        if it >= 4:
            st = eng.stage_times(0, 0)
            ss.append(st[1])
            ts.append(st[2])
    lab = eng.get_labels_packed()
    sample = lab[:: 997].copy()
    np.save(os.environ["OUT"], sample)
    print(json.dumps({"summary_ms": statistics.median(ss), "label_ms": statistics.median(ts)}))


if __name__ == "__main__":
    if os.environ.get("WM_CHILD"):
        run_one()
        sys.exit(0)
    import numpy as np

    from paper_1810_02612_b200._native import AB_SO  # (pl, tc: A/B build only)

    variants = [("wm128", {"ROWS": "128"}), ("pl", {"LTLG_WORDMAJOR": "0", "LTLG_DEV_SO": AB_SO}),
                ("tc", {"LTLG_TC": "1", "LTLG_DEV_SO": AB_SO})]
    if os.environ.get("VARIANTS"):
        variants = [v for v in variants if v[0] in os.environ["VARIANTS"].split(",")]
    ref = None
    for name, env in variants:
        out = f"/tmp/wm_ab_{name}.npy"
        e = dict(os.environ, WM_CHILD="1", OUT=out, **env)
        r = subprocess.run([sys.executable, __file__], env=e, capture_output=True, text=True)
        if r.returncode:
            print(name, "FAILED", r.stdout[-2000:], r.stderr[-3000:])
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        lab = np.load(out)
        same = None if ref is None else bool(np.array_equal(lab, ref))
        ref = lab if ref is None else ref
        print(name, res, "same_as_first:", same, flush=True)
