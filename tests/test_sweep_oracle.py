"""CPU tests of the swept-volume oracle (oracle_swept_volume, the C
restatement of swept_volume_matrix, label.cpp:75-116 + abstraction.cpp:
136-221): pinned against the golden fixtures made by the unmodified
reference, and against the reference core itself (oracle/_ref) on seeded
inputs, the reference's unit-test cases and its error paths."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from sweep_cases import FOOTPRINT, axis_aligned, flatten, random_motions


def _golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.mark.parametrize("name", ["sweep_test_label", "sweep_d18"])
def test_oracle_matches_golden(oracle, name):
    g = _golden(name)
    rows, cols = oracle.swept_volume(int(g["depth"]), g["lo"], g["hi"], g["footprint"], g["sample_off"], g["samples"])
    assert np.array_equal(rows, g["row_offsets"])
    assert np.array_equal(cols, g["col_indices"])


@pytest.mark.parametrize("depth", [3, 9, 12, 17, 21, 24, 30, 32])
def test_oracle_matches_reference_random(oracle, refcore, depth):
    off, smp = random_motions(depth, 60, empty_every=7)
    a = oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp)
    b = refcore.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("depth", [9, 15, 18])
def test_oracle_matches_reference_axis_aligned(oracle, refcore, depth):
    off, smp = axis_aligned(depth, 80, depth)
    a = oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), (4.0, 2.0, 0.0), off, smp)
    b = refcore.swept_volume(depth, (0, 0, 0), (64, 64, 4), (4.0, 2.0, 0.0), off, smp)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_oracle_reference_unit_cases(oracle, refcore):
    # test_abstraction.cpp:145-164: stationary sample covers one time slab
    off, smp = flatten([np.array([[8, 8, 0.2, 0, 1.3]], dtype=np.float64)])
    for args in [(9, (0, 0, 0), (16, 16, 4), (3.0, 1.5, 0.0))]:
        a = oracle.swept_volume(*args, off, smp)
        b = refcore.swept_volume(*args, off, smp)
        assert np.array_equal(a[1], b[1]) and a[1].size > 0


def test_oracle_errors_match_reference(oracle, refcore):
    from oracle.oracle import DomainError, OracleError

    # test_abstraction.cpp:221-232: leaving the workspace throws (position, then time)
    pos = flatten([np.array([[9.8, 5, 0, 0, 0.5]])])
    late = flatten([np.array([[5, 5, 0, 0, 1.5]])])
    for off, smp, msg in [(*pos, "trajectory exits workspace (position)"),
                          (*late, "trajectory exits workspace (time axis)")]:
        for impl in (oracle, refcore):
            with pytest.raises(DomainError, match=msg.replace("(", r"\(").replace(")", r"\)")):
                impl.swept_volume(9, (0, 0, 0), (10, 10, 1), (2.0, 1.0, 0.0), off, smp)
    ok = flatten([np.array([[5, 5, 0, 0, 0.5]])])
    for impl in (oracle, refcore):
        with pytest.raises(OracleError, match="footprint must be positive"):
            impl.swept_volume(9, (0, 0, 0), (10, 10, 1), (0.0, 1.0, 0.0), *ok)
        with pytest.raises(OracleError, match="supports depth <= 32"):
            impl.swept_volume(33, (0, 0, 0), (10, 10, 1), (2.0, 1.0, 0.0), *ok)
    # the first offending sample in (edge, sample) order decides
    mixed = flatten([np.array([[5, 5, 0, 0, 0.5], [5, 5, 0, 0, 1.5]]), np.array([[9.8, 5, 0, 0, 0.5]])])
    for impl in (oracle, refcore):
        with pytest.raises(DomainError, match="time axis"):
            impl.swept_volume(9, (0, 0, 0), (10, 10, 1), (2.0, 1.0, 0.0), *mixed)


def test_oracle_matches_reference_abstraction(oracle, refcore):
    off, smp = refcore.abstraction(target_edges=300, seed=23)
    for depth in (12, 18, 24):
        a = oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp)
        b = refcore.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp, workers=3)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
