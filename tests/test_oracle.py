"""Pin the CPU oracle (oracle/ltlg_oracle.c) against the reference's goldens.

The fixtures in tests/golden/ were produced by the unmodified reference core
(tests/golden/make_golden.py); these tests check the C restatement reproduces
every one of them bit-exactly, plus the reference's own known-answer tests
(test_label.cpp, test_grid.cpp).  CPU only.
"""
import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.oracle import (SplitMix64, bits_to_words, dense_label, labels_dense, mix_seed,
                           random_rows, to_csr)


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


LABEL_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                     if "labels" in np.load(p).files)


def test_golden_inventory():
    assert len(LABEL_CASES) >= 27
    assert "rand_seed11" in LABEL_CASES and "eq13_col4" in LABEL_CASES


@pytest.mark.parametrize("case", LABEL_CASES)
@pytest.mark.parametrize("workers", [1, 3, 0])
def test_oracle_label_all_matches_reference_golden(oracle, case, workers):
    g = load(case)
    rows, cols, props = int(g["rows"]), int(g["cols"]), int(g["props"])
    out = oracle.label_all(rows, cols, g["offsets"], g["indices"], cols, props, g["colwords"], workers)
    assert np.array_equal(out, g["labels"])


def test_splitmix_matches_reference_stream():
    g = load("splitmix_seed11")
    assert np.array_equal(SplitMix64(11).next_block(4096), g["next"])
    assert np.array_equal(SplitMix64(11).uniform_block(4096), g["uniform"])
    mixes = [mix_seed(s, q) for s in (0, 1, 11, 2**63 + 5) for q in (0, 1, 2, 63, 1000)]
    assert mixes == [int(x) for x in g["mix_seed"]]


def test_splitmix_known_answer():
    # Published splitmix64 vector: seed 0 -> 0xe220a8397b1dcdaf.
    assert SplitMix64(0).next() == 0xE220A8397B1DCDAF


def test_oracle_mix_seed_c_matches(oracle):
    for s in (0, 1, 11, 2**63 + 5):
        for q in (0, 1, 2, 63, 1000):
            assert oracle.mix_seed(s, q) == mix_seed(s, q)


def test_eq13_csr_and_label():
    # test_label.cpp:58-66 and :87-99
    ex = np.zeros((5, 5), dtype=bool)
    for r, cs in enumerate([[4], [1, 2], [0], [2, 3], [3]]):
        ex[r, cs] = True
    off, idx = to_csr(ex)
    assert off.tolist() == [0, 1, 3, 4, 6, 7]
    assert idx.tolist() == [4, 1, 2, 0, 2, 3, 3]
    g = load("eq13_col4")
    assert labels_dense(g["labels"], 5, 1)[:, 0].tolist() == [True, False, False, False, False]


def test_rand_seed11_regenerates_bit_exactly():
    # test_label.cpp:111-119 inputs regenerate from the seed.
    rng = SplitMix64(11)
    rows = random_rows(rng, 1000, 4096, 1e-3)
    cols = random_rows(rng, 3, 4096, 0.5)
    off, idx = to_csr(rows)
    g = load("rand_seed11")
    assert np.array_equal(off, g["offsets"]) and np.array_equal(idx, g["indices"])
    assert np.array_equal(bits_to_words(cols).reshape(-1), g["colwords"])
    assert np.array_equal(labels_dense(g["labels"], 1000, 3), dense_label(rows, cols))


def test_monotone_golden():
    a, b = load("monotone_seed909_before"), load("monotone_seed909_after")
    la, lb = labels_dense(a["labels"], 100, 1), labels_dense(b["labels"], 100, 1)
    assert np.all(lb[la])


def test_oracle_dimension_mismatch_message(oracle):
    from oracle.oracle import OracleError

    off = np.array([0, 1], np.uint64)
    idx = np.array([0], np.uint32)
    with pytest.raises(OracleError, match="dimension mismatch: matrix cols 5 vs proposition rows 8"):
        oracle.label_all(1, 5, off, idx, 8, 1, np.zeros(1, np.uint64))
    with pytest.raises(OracleError, match="at most 64 propositions"):
        oracle.label_all(1, 5, off, idx, 5, 65, np.zeros(65, np.uint64))


def test_oracle_validate_messages_match_reference():
    from oracle.oracle import Oracle

    o = Oracle()
    with open(os.path.join(GOLDEN, "validate.json")) as f:
        cases = json.load(f)
    for c in cases:
        got = o.validate_csr(c["rows"], c["cols"], np.array(c["offsets"], np.uint64),
                             np.array(c["indices"], np.uint32))
        assert got == c["error"], c


def test_oracle_edge_counting(oracle):
    g = load("counting_examples")
    column = np.zeros((1, 16), dtype=bool)
    column[0, 3] = True
    cw = bits_to_words(column)[0]
    got = [list(oracle.label_edge_counting(np.array(r, np.uint32), cw)) for r in
           ([3, 7, 9], [1, 5, 7, 12], [1, 5, 3, 9])]
    assert [[int(h), e] for h, e in got] == g["fixed"].tolist()
    c = load("counting_seed4444")
    off, idx, colw = c["offsets"], c["indices"], c["colwords"]
    for i in range(120):
        hit, e = oracle.label_edge_counting(idx[off[i]:off[i + 1]], colw)
        assert [int(hit), e] == g["seed4444"][i].tolist()


def test_zorder_goldens(oracle):
    with open(os.path.join(GOLDEN, "zorder.json")) as f:
        z = json.load(f)
    for e in z["examples"] + z["random"]:
        assert oracle.z_index(e["k"], e["depth"], e["lo"], e["hi"], e["p"]) == e["z"]
        assert oracle.z_index_tree_descent(e["k"], e["depth"], e["lo"], e["hi"], e["p"]) == e["z"]
    with pytest.raises(IndexError):
        oracle.z_index(2, 4, [0, 0], [1, 1], [1.0, 0.5])


def test_oracle_against_refcore_random(oracle, refcore):
    rng = SplitMix64(5150)
    for trial in range(10):
        r, c, p = 50 + 37 * trial, 64 * (1 + trial * 7) + trial, 1 + 6 * trial
        rows = random_rows(rng, r, c, 0.02)
        cols = random_rows(rng, p, c, 0.03)
        off, idx = to_csr(rows)
        cw = bits_to_words(cols)
        assert np.array_equal(oracle.label_all(r, c, off, idx, c, p, cw),
                              refcore.label_all(r, c, off, idx, c, p, cw))
