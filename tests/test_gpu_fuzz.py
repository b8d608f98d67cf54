"""Randomised end-to-end parity (GPU): random shapes, proposition counts,
frame counts across every dispatch path (single frame, per-frame, prop-lane
slices, > 64 frames), shard counts, row sorting, read-back blocks, task
sizes, word-major task rows, pageable or pinned P -- against the oracle."""
import random

import numpy as np
import pytest

from oracle.oracle import Oracle, SplitMix64, bits_to_words, random_rows, to_csr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chunk", range(5))
def test_randomised_engine_configs(chunk):
    run_chunk(chunk)


@pytest.mark.parametrize("chunk", range(5, 8))
def test_randomised_engine_configs_word_major_single_frame(chunk):
    # the same with every single frame on label_wm1_kernel (LTLG_WM1=1, read
    # once per process: a child process) -- the fuzz grids are small enough for
    # the stream64 kernel otherwise; task_rows 256 takes its 256-row label block
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    code = f"import sys; sys.path[:0] = [{os.path.dirname(here)!r}, {here!r}]; import test_gpu_fuzz as t; t.run_chunk({chunk})"
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LTLG_WM1="1"), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def run_chunk(chunk):
    import torch

    from paper_1810_02612_b200 import CsrBoolMatrix, LabelEngine, LabelMatrix

    O = Oracle()
    rnd = random.Random(1000 + chunk)
    for it in range(40):
        r = rnd.choice([0, 1, 7, 100, 513, 2000])
        c = rnd.choice([1, 63, 64, 65, 1000, 4097, 9000])
        props = rnd.choice([0, 1, 5, 16, 17, 31, 32, 33, 48, 64])
        frames = rnd.choice([1, 1, 2, 9, 10, 15, 16, 17, 40, 64, 65, 100])
        dens = rnd.choice([0.0, 0.001, 0.02, 0.2])
        rng = SplitMix64(chunk * 1000 + it)
        rows = random_rows(rng, r, c, dens) if r else np.zeros((0, c), bool)
        off, idx = to_csr(rows)
        P = np.zeros((frames, props, (c + 63) // 64), np.uint64)
        for f in range(frames):
            if props:
                P[f] = bits_to_words(random_rows(rng, props, c, rnd.choice([0.001, 0.05, 0.5, 0.97])))
        if props and frames > 2:
            P[::3, :, ::4] = np.uint64(0xFFFFFFFFFFFFFFFF)
        devs = rnd.choice([[0], [0], [0, 0], [0, 0, 0]])
        eng = LabelEngine(devices=devs, sort_rows=rnd.random() < 0.5, readback_chunks=rnd.choice([0, 1, 3, 8]),
                          stream_task_pairs=rnd.choice([0, 1, 50, 4096]), batch_task_pairs=rnd.choice([0, 1, 7, 300]),
                          task_rows=rnd.choice([0, 1, 5, 33, 128, 256]))
        eng.load_abstraction(CsrBoolMatrix(r, c, off, idx))
        src = P
        if rnd.random() < 0.4 and P.size:
            src = torch.from_numpy(P.view(np.int64).copy()).pin_memory()
        eng.submit_grid(c, props, src, frames)
        for f in range(frames):
            want = O.label_all(r, c, off, idx, c, props, P[f])
            assert eng.get_labels(f) == LabelMatrix(r, props, want), (it, r, c, props, frames, devs, f)
        eng.close()
