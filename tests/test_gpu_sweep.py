"""GPU parity of the swept-volume matrix (ltlg_swept_volume)
against the golden fixtures made by the unmodified reference
(swept_volume_matrix, label.cpp:75-116) and against the oracle restatement
on seeded inputs: bit-exact CSR (row offsets and column indices)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from sweep_cases import FOOTPRINT, axis_aligned, flatten, random_motions

pytestmark = pytest.mark.gpu


def _gpu(off, smp, depth, lo=(0, 0, 0), hi=(64, 64, 4), fp=FOOTPRINT):
    from paper_1810_02612_b200 import FootprintSpec, swept_volume_matrix

    m = swept_volume_matrix((off, smp), FootprintSpec(*fp), tuple(zip(lo, hi)), depth)
    return m.row_offsets, m.col_indices


def _same(a, b):
    assert a[0].size == b[0].size and np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1])


@pytest.mark.parametrize("name", ["sweep_test_label", "sweep_d18"])
def test_sweep_golden(name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    got = _gpu(g["sample_off"], g["samples"], int(g["depth"]), g["lo"], g["hi"], tuple(g["footprint"]))
    _same(got, (g["row_offsets"], g["col_indices"]))


@pytest.mark.parametrize("depth", [3, 9, 12, 15, 17, 18, 21, 24, 27, 30, 32])
def test_sweep_random_vs_oracle(oracle, depth):
    off, smp = random_motions(100 + depth, 400, empty_every=9)
    _same(_gpu(off, smp, depth), oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp))


@pytest.mark.parametrize("depth", [9, 12, 15, 18, 24])
def test_sweep_axis_aligned_vs_oracle(oracle, depth):
    off, smp = axis_aligned(depth, 300, depth)
    fp = (4.0, 2.0, 0.0)
    _same(_gpu(off, smp, depth, fp=fp), oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), fp, off, smp))


def test_sweep_odd_bounds_vs_oracle(oracle):
    off, smp = random_motions(7, 300, lo=(-37.5, 12.25, 3.0), hi=(41.0, 80.0, 9.5))
    lo, hi = (-37.5, 12.25, 3.0), (41.0, 80.0, 9.5)
    for depth in (10, 19, 29):
        _same(_gpu(off, smp, depth, lo, hi), oracle.swept_volume(depth, lo, hi, FOOTPRINT, off, smp))


def test_sweep_overflow_rows_vs_oracle(oracle):
    # a 30 m x 12 m footprint on 0.25 m cells: > kSweepCap (2048) distinct
    # cells per row -> the global-memory sets; 60 m x 40 m -> their retry
    for fp, depth in [((30.0, 12.0, 0.0), 24), ((60.0, 40.0, 0.0), 24)]:
        off, smp = random_motions(3, 12, lo=(0, 0, 0), hi=(128, 128, 4), margin=40.0, samples=9)
        lo, hi = (0, 0, 0), (128, 128, 4)
        want = oracle.swept_volume(depth, lo, hi, fp, off, smp)
        assert np.diff(want[0].astype(np.int64)).max() > 2048
        _same(_gpu(off, smp, depth, lo, hi, fp), want)


@pytest.mark.parametrize("stage", ["0", "5000"])
def test_sweep_staging_shortfall_vs_oracle(oracle, monkeypatch, stage):
    """A staging buffer too small for the rows: the rows are rasterized again
    straight into place (MODE 1); overflow rows still take the global sets."""
    monkeypatch.setenv("LTLG_SWEEP_STAGE", stage)
    off, smp = random_motions(41, 300, empty_every=5)
    for depth in (15, 24):
        _same(_gpu(off, smp, depth), oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp))


def test_sweep_empty_inputs():
    off, smp = flatten([])
    rows, cols = _gpu(off, smp, 12)
    assert rows.tolist() == [0] and cols.size == 0
    off, smp = flatten([np.zeros((0, 5))] * 5)
    rows, cols = _gpu(off, smp, 12)
    assert rows.tolist() == [0] * 6 and cols.size == 0


def test_sweep_errors_match_reference():
    from paper_1810_02612_b200 import DomainError

    pos = flatten([np.array([[9.8, 5, 0, 0, 0.5]])])
    late = flatten([np.array([[5, 5, 0, 0, 1.5]])])
    ok = flatten([np.array([[5, 5, 0, 0, 0.5]])])
    b = ((0, 0, 0), (10, 10, 1))
    with pytest.raises(DomainError, match=r"trajectory exits workspace \(position\)"):
        _gpu(*pos, 9, *b, fp=(2.0, 1.0, 0.0))
    with pytest.raises(DomainError, match=r"trajectory exits workspace \(time axis\)"):
        _gpu(*late, 9, *b, fp=(2.0, 1.0, 0.0))
    with pytest.raises(ValueError, match="footprint must be positive"):
        _gpu(*ok, 9, *b, fp=(2.0, -1.0, 0.0))
    with pytest.raises(ValueError, match="supports depth <= 32"):
        _gpu(*ok, 33, *b, fp=(2.0, 1.0, 0.0))
    mixed = flatten([np.array([[5, 5, 0, 0, 0.5], [5, 5, 0, 0, 1.5]]), np.array([[9.8, 5, 0, 0, 0.5]])])
    with pytest.raises(DomainError, match="time axis"):
        _gpu(*mixed, 9, *b, fp=(2.0, 1.0, 0.0))
    from paper_1810_02612_b200 import swept_volume_matrix

    with pytest.raises(ValueError, match="requires a 3-d"):
        swept_volume_matrix(ok, None, ((0, 10), (0, 10)), 8)


def test_sweep_loads_into_engine(oracle):
    """GPU-built T -> engine (ltlg_load_csr) -> labels == label_all on the oracle CSR."""
    from paper_1810_02612_b200 import FootprintSpec, LabelEngine, swept_volume

    depth = 15
    off, smp = random_motions(11, 500)
    rows, cols = oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp)
    sv = swept_volume((off, smp), FootprintSpec(*FOOTPRINT), ((0, 64), (0, 64), (0, 4)), depth)
    cells = 1 << depth
    rng = np.random.default_rng(5)
    props = 6
    P = rng.integers(0, 2**63, size=(props, (cells + 63) // 64), dtype=np.uint64) & \
        rng.integers(0, 2**63, size=(props, (cells + 63) // 64), dtype=np.uint64)
    eng = LabelEngine()
    eng.load_swept_volume(sv)
    eng.submit_grid(cells, props, P)
    got = eng.get_labels(0)
    want = oracle.label_all(off.size - 1, cells, rows, cols, cells, props, P)
    assert np.array_equal(got.bits.reshape(-1), np.asarray(want).reshape(-1))
    sv.close()


def test_sweep_reference_abstraction(refcore, oracle):
    off, smp = refcore.abstraction(target_edges=2000, seed=29)
    for depth in (12, 18, 24):
        _same(_gpu(off, smp, depth), oracle.swept_volume(depth, (0, 0, 0), (64, 64, 4), FOOTPRINT, off, smp))


def test_sweep_saved_as_csb1_like_the_reference(refcore, tmp_path):
    """ltlg_csr_save: the GPU-built matrix as CSB1, byte-identical to the
    reference's CsrBoolMatrix::save of the same rows; and it loads back."""
    from paper_1810_02612_b200 import FootprintSpec, LabelEngine, swept_volume

    off, smp = refcore.abstraction(target_edges=400, seed=9)
    sv = swept_volume((off, smp), FootprintSpec(*FOOTPRINT), ((0, 64), (0, 64), (0, 4)), 15)
    m = sv.to_csr()
    ours, theirs = tmp_path / "gpu.csb1", tmp_path / "ref.csb1"
    sv.save(str(ours))
    refcore.csr_save(str(theirs), m.rows, m.cols, m.row_offsets, m.col_indices)
    assert ours.read_bytes() == theirs.read_bytes()
    eng = LabelEngine()
    eng.load_abstraction_file(str(ours))
    assert eng.info().rows == m.rows
    eng.close()
    sv.close()
    with pytest.raises(RuntimeError, match="cannot open for writing"):
        sv2 = swept_volume((off, smp), FootprintSpec(*FOOTPRINT), ((0, 64), (0, 64), (0, 4)), 15)
        sv2.save(str(tmp_path / "no" / "such" / "dir.csb1"))
