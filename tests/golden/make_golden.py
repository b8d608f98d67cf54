"""Generate tests/golden/* by running the UNMODIFIED reference core.

Run here (where /root/reference exists):  make -C oracle ref && python tests/golden/make_golden.py

Every expected output in these fixtures is produced by the reference's own
functions (ltlgrid::label_all, to_csr-equivalent CSR, CsrBoolMatrix::save,
LabelMatrix::save, save_bitset, z_index, validate) through
oracle/_ref/libltlgrid_ref.so.  Inputs follow the reference tests
(test_label.cpp, test_grid.cpp) with the same SplitMix64 seeds, plus a set of
seeded random scenes covering the edge cases label_all must honour (empty
rows, cells not a multiple of 64, 0/1/31/32/33/63/64 propositions).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import (RefCore, SplitMix64, bits_to_words, dense_label, labels_dense,  # noqa: E402
                           labels_to_words, random_rows, to_csr)


def save_case(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def label_case(ref, name, dense_rows, dense_cols, workers=0, **extra):
    rows, cells = dense_rows.shape
    props = dense_cols.shape[0]
    off, idx = to_csr(dense_rows)
    colw = bits_to_words(dense_cols) if props else np.zeros((0, (cells + 63) // 64), np.uint64)
    L = ref.label_all(rows, cells, off, idx, cells, props, colw, workers)
    # The reference's own dense triple loop (oracles.hpp:203-216) agrees.
    assert np.array_equal(labels_dense(L, rows, props), dense_label(dense_rows, dense_cols)), name
    save_case(name, rows=np.uint64(rows), cols=np.uint64(cells), offsets=off, indices=idx,
              props=np.int64(props), colwords=colw.reshape(-1), labels=L, **extra)
    return off, idx, colw, L


def main():
    ref = RefCore()

    # SplitMix64 / mix_seed stream (rng.hpp:10-34) from the reference itself.
    import ctypes as C
    n = 4096
    out = np.zeros(n, np.uint64)
    uni = np.zeros(n, np.float64)
    ref.lib.ref_splitmix_block.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
    ref.lib.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    ref.lib.ref_mix_seed.restype = C.c_uint64
    ref.lib.ref_splitmix_block(11, n, out.ctypes.data_as(C.POINTER(C.c_uint64)), uni.ctypes.data_as(C.POINTER(C.c_double)))
    mixes = np.array([ref.lib.ref_mix_seed(s, q) for s in (0, 1, 11, 2**63 + 5) for q in (0, 1, 2, 63, 1000)], np.uint64)
    assert np.array_equal(SplitMix64(11).next_block(n), out)
    assert np.array_equal(SplitMix64(11).uniform_block(n), uni)
    save_case("splitmix_seed11", next=out, uniform=uni, mix_seed=mixes)

    # test_label.cpp:13-27 / 58-66 / 87-109: the Eq. 13 worked example.
    ex = np.zeros((5, 5), dtype=bool)
    for r, cs in enumerate([[4], [1, 2], [0], [2, 3], [3]]):
        ex[r, cs] = True
    col4 = np.zeros((1, 5), dtype=bool)
    col4[0, 4] = True
    off, idx, _, L = label_case(ref, "eq13_col4", ex, col4)
    assert off.tolist() == [0, 1, 3, 4, 6, 7] and idx.tolist() == [4, 1, 2, 0, 2, 3, 3]
    assert labels_dense(L, 5, 1)[:, 0].tolist() == [True, False, False, False, False]
    label_case(ref, "eq13_allfalse", ex, np.zeros((2, 5), dtype=bool))

    # test_label.cpp:111-119: 1000x4096 @1e-3 x 3 props @0.5, seed 11.
    rng = SplitMix64(11)
    rows = random_rows(rng, 1000, 4096, 1e-3)
    cols = random_rows(rng, 3, 4096, 0.5)
    label_case(ref, "rand_seed11", rows, cols)

    # test_label.cpp:121-132: worker invariance, seed 77.
    rng = SplitMix64(77)
    rows = random_rows(rng, 333, 1024, 0.01)
    cols = random_rows(rng, 2, 1024, 0.4)
    off, idx, colw, L1 = label_case(ref, "workers_seed77", rows, cols, workers=1)
    for w in (2, 5):
        assert np.array_equal(ref.label_all(333, 1024, off, idx, 1024, 2, colw, w), L1)

    # test_label.cpp:134-146: monotone, seed 909.
    rng = SplitMix64(909)
    rows = random_rows(rng, 100, 512, 0.02)
    col = random_rows(rng, 1, 512, 0.05)
    grown = col.copy()
    for _ in range(30):
        grown[0, rng.below(512)] = True
    label_case(ref, "monotone_seed909_before", rows, col)
    label_case(ref, "monotone_seed909_after", rows, grown)

    # test_label.cpp:155-185: label_edge_counting.
    column = np.zeros((1, 16), dtype=bool)
    column[0, 3] = True
    cw = bits_to_words(column)[0]
    cnt = []
    for row in ([3, 7, 9], [1, 5, 7, 12], [1, 5, 3, 9]):
        hit, ex_ = ref.label_edge_counting(np.array(row, np.uint32), 16, cw)
        cnt.append([int(hit), ex_])
    assert cnt == [[1, 1], [0, 4], [1, 3]]
    rng = SplitMix64(4444)
    rows = random_rows(rng, 120, 512, 0.03)
    col = random_rows(rng, 1, 512, 0.2)
    off, idx, colw, L = label_case(ref, "counting_seed4444", rows, col)
    ex_counts = []
    for i in range(120):
        r = idx[off[i]:off[i + 1]]
        hit, e = ref.label_edge_counting(r, 512, colw[0])
        ex_counts.append([int(hit), e])
    save_case("counting_examples", fixed=np.array(cnt, np.uint64),
              seed4444=np.array(ex_counts, np.uint64))

    # Seeded random scenes: edge cases of shape, density and prop count.
    rng = SplitMix64(20260101)
    scenes = [
        (0, 64, 3, 0.1, 0.5), (7, 5, 1, 0.4, 0.5), (50, 100, 0, 0.05, 0.5),
        (64, 1000, 1, 0.01, 0.2), (200, 4096, 31, 0.003, 0.02), (200, 4096, 32, 0.003, 0.02),
        (150, 4096, 33, 0.003, 0.02), (100, 2048, 63, 0.004, 0.01), (100, 2048, 64, 0.004, 0.01),
        (300, 256, 4, 0.0, 0.5), (300, 256, 4, 1.0, 0.01), (257, 4096, 16, 0.005, 0.0),
        (257, 4096, 16, 0.005, 1.0), (1000, 4096, 8, 0.002, 0.03), (33, 33, 5, 0.3, 0.3),
        (500, 16384, 12, 0.001, 0.005), (129, 65, 64, 0.1, 0.05), (1, 1, 1, 1.0, 1.0),
        (2, 70, 2, 0.5, 0.0), (400, 8192, 24, 0.0015, 0.004),
    ]
    meta = []
    for s, (r, c, p, dr, dp) in enumerate(scenes):
        rows = random_rows(rng, r, c, dr)
        if r >= 4:
            rows[r // 3] = False  # an empty row
        cols = random_rows(rng, p, c, dp)
        label_case(ref, f"scene_{s:02d}", rows, cols)
        meta.append({"scene": s, "rows": r, "cells": c, "props": p, "row_density": dr, "prop_density": dp})
    with open(os.path.join(HERE, "scenes.json"), "w") as f:
        json.dump(meta, f, indent=1)

    # File formats written by the reference (label.cpp:251-326, grid.cpp:370-390).
    rng = SplitMix64(31337)
    rows = random_rows(rng, 64, 2048, 0.02)
    off, idx = to_csr(rows)
    ref.csr_save(os.path.join(HERE, "seed31337.csb1"), 64, 2048, off, idx)
    save_case("seed31337_csr", rows=np.uint64(64), cols=np.uint64(2048), offsets=off, indices=idx)
    lab = np.zeros((5, 3), dtype=bool)
    lab[0, 2] = lab[3, 0] = lab[3, 1] = True
    ref.label_save(os.path.join(HERE, "l5x3.lbm1"), 5, 3, labels_to_words(lab))
    rng = SplitMix64(10)
    bits = np.zeros((1, 256), dtype=bool)
    for _ in range(100):
        bits[0, rng.below(256)] = True
    ref.save_bitset(os.path.join(HERE, "seed10_d8.zobv"), 2, 8, bits_to_words(bits)[0])
    save_case("seed10_d8_bits", words=bits_to_words(bits)[0])

    # validate() messages (label.cpp:16-40) for malformed matrices.
    bad = [
        (2, 4, [0, 1], [1]), (2, 4, [0, 2, 1], [1]), (2, 4, [0, 1, 1], [9]),
        (2, 4, [1, 1, 1], [1]), (2, 4, [0, 1, 2], [1]), (1, 8, [0, 2], [3, 3]),
        (1, 8, [0, 2], [5, 2]), (2, 8, [0, 1, 2], [7, 0]),
    ]
    vmsg = []
    for r, c, o, i in bad:
        vmsg.append({"rows": r, "cols": c, "offsets": o, "indices": i,
                     "error": ref.validate_csr(r, c, np.array(o, np.uint64), np.array(i, np.uint32))})
    with open(os.path.join(HERE, "validate.json"), "w") as f:
        json.dump(vmsg, f, indent=1)

    # z-order (grid.cpp:85-117): test_grid.cpp:24-37 examples + seeded points.
    zs = {"examples": [
        {"k": 2, "depth": 2, "lo": [0, 0], "hi": [1, 1], "p": [0.1, 0.1]},
        {"k": 2, "depth": 2, "lo": [0, 0], "hi": [1, 1], "p": [0.9, 0.9]},
        {"k": 2, "depth": 4, "lo": [0, 0], "hi": [1, 1], "p": [0.6, 0.2]},
        {"k": 1, "depth": 1, "lo": [0], "hi": [1], "p": [0.5]},
    ]}
    for e in zs["examples"]:
        e["z"] = ref.z_index(e["k"], e["depth"], e["lo"], e["hi"], e["p"])
    assert [e["z"] for e in zs["examples"]] == [0, 3, 8, 1]
    rng = SplitMix64(42)
    pts = []
    for k in (2, 3):
        for d in (8, 12, 18, 20, 21):
            lo = [-3.0 + i for i in range(k)]
            hi = [7.0 + 2 * i for i in range(k)]
            for _ in range(100):
                p = [lo[i] + (hi[i] - lo[i]) * float(rng.uniform_block(1)[0]) for i in range(k)]
                pts.append({"k": k, "depth": d, "lo": lo, "hi": hi, "p": p,
                            "z": ref.z_index(k, d, lo, hi, p)})
    zs["random"] = pts
    with open(os.path.join(HERE, "zorder.json"), "w") as f:
        json.dump(zs, f)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
