"""GPU parity: the sm_100a labeling path through the C ABI vs the CPU oracle.

Bit-exact (LabelMatrix::operator==, label.hpp:79) on
  * every golden fixture produced by the unmodified reference (tests/golden),
  * >= 100 seeded random scenes (SPEC.md:616 acceptance), single and batched,
  * the synthetic BASELINE configs 1-3 in full and config 4 on sampled frames,
  * the world->vehicle resample (vs oracle_resample),
and the reference's error behaviour (messages of label.cpp:124-154, 16-40, 271-298).
"""
import glob
import math
import os
import zlib

import numpy as np
import pytest

from conftest import GOLDEN, has_gpu
from oracle.oracle import (Oracle, SplitMix64, bits_to_words, dense_label, labels_dense, random_rows, to_csr,
                           words_to_bits)

pytestmark = pytest.mark.gpu

if not has_gpu():  # pragma: no cover - collected on CPU-only hosts
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1810_02612_b200 import (CsrBoolMatrix, DensePropMatrix, LabelEngine, LabelMatrix,  # noqa: E402
                                   LtlgError, label_all)
from workload.synth import CONFIGS, SyntheticPRM, props_words  # noqa: E402

ORACLE = Oracle()
LABEL_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                     if "labels" in np.load(p).files)
ENGINE_VARIANTS = [
    dict(),
    dict(sort_rows=False),
    dict(stream_task_pairs=1, batch_task_pairs=1),
    dict(stream_task_pairs=37, batch_task_pairs=5, sort_rows=False),
    dict(readback_chunks=3),
    dict(readback_chunks=7, stream_task_pairs=37, batch_task_pairs=5),
]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


@pytest.fixture(scope="module", params=range(len(ENGINE_VARIANTS)))
def engine(request):
    e = LabelEngine(devices=[0], **ENGINE_VARIANTS[request.param])
    yield e
    e.close()


@pytest.mark.parametrize("case", LABEL_CASES)
def test_golden_single_frame(engine, case):
    g = load(case)
    rows, cols, props = int(g["rows"]), int(g["cols"]), int(g["props"])
    engine.load_abstraction(CsrBoolMatrix(rows, cols, g["offsets"], g["indices"]))
    engine.submit_grid(cols, props, g["colwords"], 1)
    got = engine.get_labels(0)
    assert got == LabelMatrix(rows, props, g["labels"])


@pytest.mark.parametrize("case", LABEL_CASES)
def test_golden_batched_frames(engine, case):
    g = load(case)
    rows, cols, props = int(g["rows"]), int(g["cols"]), int(g["props"])
    nw = (cols + 63) // 64
    rng = SplitMix64(zlib.crc32(case.encode()))
    frames = 3
    P = np.zeros((frames, props, nw), np.uint64)
    P[0] = g["colwords"].reshape(props, nw)
    for f in range(1, frames):
        if props:
            P[f] = bits_to_words(random_rows(rng, props, cols, 0.05 * f))
    engine.load_abstraction(CsrBoolMatrix(rows, cols, g["offsets"], g["indices"]))
    engine.submit_grid(cols, props, P, frames)
    assert engine.get_labels(0) == LabelMatrix(rows, props, g["labels"])
    for f in range(1, frames):
        want = ORACLE.label_all(rows, cols, g["offsets"], g["indices"], cols, props, P[f])
        assert engine.get_labels(f) == LabelMatrix(rows, props, want)


@pytest.mark.parametrize("case", ["eq13_col4", "rand_seed11", "scene_04", "scene_08"])
@pytest.mark.parametrize("workers", [0, 1, 2, 5])
def test_label_all_drop_in(case, workers):
    g = load(case)
    rows, cols, props = int(g["rows"]), int(g["cols"]), int(g["props"])
    m = CsrBoolMatrix(rows, cols, g["offsets"], g["indices"])
    p = DensePropMatrix.from_words(cols, g["colwords"].reshape(props, -1))
    assert label_all(m, p, workers) == LabelMatrix(rows, props, g["labels"])


def _scene(seed):
    rng = SplitMix64(seed)
    r = int(rng.below(600))
    c = int(1 + rng.below(5000))
    props = int(rng.below(65))
    frames = [1, 1, 2, 3, 5, 31, 33, 64, 65][int(rng.below(9))]
    dr = [0.0, 0.001, 0.01, 0.05, 0.3][int(rng.below(5))]
    rows = random_rows(rng, r, c, dr) if r else np.zeros((0, c), bool)
    P = np.zeros((frames, props, (c + 63) // 64), np.uint64)
    for f in range(frames):
        for j in range(props):
            kind = int(rng.below(4))
            if kind == 0:
                col = random_rows(rng, 1, c, [0.001, 0.01, 0.1, 0.5][int(rng.below(4))])[0]
            elif kind == 1:  # contiguous run -> full words
                a = int(rng.below(c))
                col = np.zeros(c, bool)
                col[a:a + int(rng.below(c - a + 1))] = True
            elif kind == 2:
                col = np.ones(c, bool)
            else:
                col = np.zeros(c, bool)
            P[f, j] = bits_to_words(col[None, :])[0]
    return rows, P, frames, props, c


@pytest.mark.parametrize("seed", range(120))
def test_random_scenes(seed):
    rows, P, frames, props, c = _scene(1000 + seed)
    r = rows.shape[0]
    off, idx = to_csr(rows)
    eng = LabelEngine(devices=[0], stream_task_pairs=int(1 + seed % 97), batch_task_pairs=int(1 + seed % 13),
                      sort_rows=bool(seed % 2))
    eng.load_abstraction(CsrBoolMatrix(r, c, off, idx))
    eng.submit_grid(c, props, P, frames)
    packed = eng.get_labels_packed() if props else None
    for f in range(frames):
        want = ORACLE.label_all(r, c, off, idx, c, props, P[f])
        if props and r * c <= 2_000_000:  # the oracle itself vs the dense triple loop
            assert np.array_equal(labels_dense(want, r, props), dense_label(rows, words_to_bits(P[f], c)))
        got = eng.get_labels(f)
        assert got == LabelMatrix(r, props, want), f"frame {f}"
        if props:
            assert np.array_equal(packed[:, f].astype(np.uint64), want.reshape(r, -1)[:, 0])
    eng.close()


@pytest.mark.parametrize("props", [5, 20, 40, 64])
@pytest.mark.parametrize("frames", [65, 130])
def test_many_frames_in_slices(props, frames):
    """> 64 frames: the prop-lane kernel in balanced frame slices (two or
    three passes), each writing its columns of the edge-major labels."""
    rng = SplitMix64(props * 1000 + frames)
    r, c = 700, 3001
    rows = random_rows(rng, r, c, 0.01)
    off, idx = to_csr(rows)
    P = np.zeros((frames, props, (c + 63) // 64), np.uint64)
    for f in range(frames):
        P[f] = bits_to_words(random_rows(rng, props, c, [0.002, 0.05, 0.6][f % 3]))
    P[::7, :, ::5] = np.uint64(0xFFFFFFFFFFFFFFFF)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(r, c, off, idx))
    eng.submit_grid(c, props, P, frames)
    packed = eng.get_labels_packed()
    for f in range(frames):
        want = ORACLE.label_all(r, c, off, idx, c, props, P[f])
        assert np.array_equal(packed[:, f].astype(np.uint64), want.reshape(r, -1)[:, 0]), f"frame {f}"
    eng.close()


@pytest.mark.parametrize("props", [1, 7, 16, 17, 32, 33, 64])
def test_pinned_single_frame_fused_upload(props):
    """One frame from pinned host memory: the summary kernel reads P through
    the host mapping and writes the device copy (no cudaMemcpyAsync).  The
    random P makes most words carry > 2 partial props, so the labeling kernel
    also reads that device copy."""
    import torch

    rng = np.random.default_rng(props)
    r, c = 3000, 64 * 97 + 13
    rows = rng.random((r, c)) < 0.004
    off, idx = to_csr(rows)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(r, c, off, idx))
    nw = (c + 63) // 64
    for trial in range(3):
        P = rng.integers(0, 2**63, size=(1, props, nw), dtype=np.uint64)
        if trial == 2:  # whole words set / clear too
            P[:, :, ::3] = np.uint64(0xFFFFFFFFFFFFFFFF)
            P[:, :, 1::5] = 0
        pinned = torch.from_numpy(P.view(np.int64).copy()).pin_memory()
        eng.submit_grid(c, props, pinned, 1)
        eng.wait()
        want = ORACLE.label_all(r, c, off, idx, c, props, P[0])
        assert eng.get_labels(0) == LabelMatrix(r, props, want), f"trial {trial}"
        # the same frame from pageable memory (copy-engine upload) agrees
        eng.submit_grid(c, props, P, 1)
        assert eng.get_labels(0) == LabelMatrix(r, props, want)
    eng.close()


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_synthetic_configs_full(cfg):
    c = CONFIGS[cfg]
    depth, E, props = c["depth"], c["edges"], c["props"]
    prm = SyntheticPRM(seed=1, depth=depth)
    t = prm.words(0, E)
    off, idx = prm.csr(0, E)
    P = props_words(1, depth, props, 0, 1)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    eng.submit_grid(1 << depth, props, P, 1)
    got = eng.get_labels(0)
    want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[0])
    assert got == LabelMatrix(E, props, want)
    hit = labels_dense(want[: min(E, 20000)], min(E, 20000), props).mean()
    assert 0.02 < hit < 0.6  # parity is non-trivial
    # the CSR path packs to the same device image and labels identically
    if cfg < 3:
        eng.load_abstraction(CsrBoolMatrix(E, 1 << depth, off, idx))
        eng.submit_grid(1 << depth, props, P, 1)
        assert eng.get_labels(0) == got
    eng.close()


def _sampled_csr(prm, row_ids, chunk=100_000):
    """Reference CSR arrays of the given (sorted) rows only, generated chunk by
    chunk (row i of the synthetic PRM depends only on (seed, i))."""
    row_ids = np.asarray(row_ids, dtype=np.int64)
    offs, idxs, base = [np.zeros(1, np.uint64)], [], 0
    for c0 in range(0, int(row_ids[-1]) + 1, chunk):
        sel = row_ids[(row_ids >= c0) & (row_ids < c0 + chunk)] - c0
        if not sel.size:
            continue
        off, idx = prm.csr(c0, min(c0 + chunk, int(row_ids[-1]) + 1))
        cnt = (off[sel + 1] - off[sel]).astype(np.int64)
        take = np.concatenate([np.arange(int(off[i]), int(off[i + 1])) for i in sel]) if cnt.sum() else np.zeros(0, int)
        idxs.append(idx[take])
        offs.append(base + np.cumsum(cnt).astype(np.uint64))
        base += int(cnt.sum())
    return np.concatenate(offs), (np.concatenate(idxs) if idxs else np.zeros(0, np.uint32))


def test_config4_batched_frames():
    """BASELINE config 4 (the bench's `value` workload: 2M edges x 64 frames,
    512^2, 32 props) through the prop-lane kernel, against the oracle:
    every one of the 64 frames on a row sample (every 97th row), plus three
    frames on all 2M rows."""
    c = CONFIGS[4]
    depth, E, props, F = c["depth"], c["edges"], c["props"], c["frames"]
    prm = SyntheticPRM(seed=1, depth=depth)
    t = prm.words(0, E)
    P = props_words(1, depth, props, 0, F)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    eng.submit_grid(1 << depth, props, P, F)
    packed = eng.get_labels_packed()
    eng.close()
    assert packed.shape == (E, F) and packed.dtype == np.uint32
    sample = np.arange(0, E, 97)
    soff, sidx = _sampled_csr(prm, sample)
    hits = 0
    for f in range(F):  # all 64 frames, row-sampled
        want = ORACLE.label_all(len(sample), 1 << depth, soff, sidx, 1 << depth, props, P[f])
        assert np.array_equal(packed[sample, f].astype(np.uint64), want), f"frame {f}"
        hits += int(np.count_nonzero(want))
    assert hits > len(sample) * F // 10  # non-trivial labels
    off, idx = prm.csr(0, E)
    for f in (0, 17, 63):  # full oracle parity on all rows
        want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f])
        assert np.array_equal(packed[:, f].astype(np.uint64), want), f"frame {f} (all rows)"


def test_config5_shard_single_frame_full():
    """BASELINE config 5 (8M edges, 1024^2, 64 props) on one per-GPU shard of
    the 8-way row partition: rows [0, 1M), all of them, one frame, through
    label_stream64_kernel<64, u64, ...> (64-bit labels, the L1 table path).
    The oracle runs in 125k-row chunks to bound host memory."""
    c = CONFIGS[5]
    depth, props, E = c["depth"], c["props"], c["edges"] // 8
    prm = SyntheticPRM(seed=1, depth=depth)
    t = prm.words(0, E)
    P = props_words(1, depth, props, 0, 1)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    del t
    eng.submit_grid(1 << depth, props, P[0], 1)
    got = eng.get_labels(0).bits
    eng.close()
    step = 125_000
    for r0 in range(0, E, step):
        off, idx = prm.csr(r0, r0 + step)
        want = ORACLE.label_all(step, 1 << depth, off, idx, 1 << depth, props, P[0])
        assert np.array_equal(got[r0:r0 + step], want), f"rows {r0}..{r0 + step}"


def test_config5_shard_64_frames():
    """Config 5 shard (rows [0, 1M) of the 8M-edge T, 1024^2, 64 props) x a
    64-frame batch: label_pl_kernel<u64, 2> (two props per lane) and
    pl_build_kernel<6>. Every frame on a row sample (every 61st row), two
    frames on all rows."""
    c = CONFIGS[5]
    depth, props, E, F = c["depth"], c["props"], c["edges"] // 8, 64
    prm = SyntheticPRM(seed=1, depth=depth)
    t = prm.words(0, E)
    P = props_words(1, depth, props, 0, F)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    del t
    eng.submit_grid(1 << depth, props, P, F)
    packed = eng.get_labels_packed()
    eng.close()
    assert packed.shape == (E, F) and packed.dtype == np.uint64
    sample = np.arange(0, E, 61)
    soff, sidx = _sampled_csr(prm, sample)
    for f in range(F):
        want = ORACLE.label_all(len(sample), 1 << depth, soff, sidx, 1 << depth, props, P[f])
        assert np.array_equal(packed[sample, f], want), f"frame {f}"
    del soff, sidx
    step = 250_000
    for f in (5, 62):
        for r0 in range(0, E, step):
            off, idx = prm.csr(r0, r0 + step)
            want = ORACLE.label_all(step, 1 << depth, off, idx, 1 << depth, props, P[f])
            assert np.array_equal(packed[r0:r0 + step, f], want), f"frame {f} rows {r0}.."


def test_monotone_in_proposition_bits():
    # test_label.cpp:134-146 at driving-PRM scale
    depth, E = 16, 200_000
    prm = SyntheticPRM(seed=3, depth=depth)
    t = prm.words(0, E)
    P = props_words(7, depth, 8, 0, 1)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    eng.submit_grid(1 << depth, 8, P, 1)
    before = eng.get_labels(0).bits
    grown = P.copy()
    rng = SplitMix64(99)
    for _ in range(2000):
        z = rng.below(1 << depth)
        j = rng.below(8)
        grown[0, j, z >> 6] |= np.uint64(1 << (z & 63))
    eng.submit_grid(1 << depth, 8, grown, 1)
    after = eng.get_labels(0).bits
    assert np.all((before & ~after) == 0) and np.any(after != before)
    eng.close()


def test_errors_mirror_reference():
    g = load("eq13_col4")
    eng = LabelEngine(devices=[0])
    with pytest.raises(LtlgError, match="no abstraction loaded"):
        eng.submit_grid(5, 1, g["colwords"], 1)
    eng.load_abstraction(CsrBoolMatrix(5, 5, g["offsets"], g["indices"]))
    # label.cpp:151-154
    with pytest.raises(ValueError, match="^dimension mismatch: matrix cols 5 vs proposition rows 8$"):
        eng.submit_grid(8, 1, np.zeros(1, np.uint64), 1)
    # label.cpp:124
    with pytest.raises(ValueError, match="^at most 64 propositions$"):
        eng.submit_grid(5, 65, np.zeros(65, np.uint64), 1)
    # validate(), label.cpp:16-40
    with pytest.raises(ValueError, match="^column index out of range$"):
        eng.load_abstraction(CsrBoolMatrix(2, 4, [0, 1, 1], [9]))
    with pytest.raises(ValueError, match="^row_offsets must be nondecreasing$"):
        eng.load_abstraction(CsrBoolMatrix(2, 4, [0, 2, 1], [1]))
    with pytest.raises(ValueError, match="^column indices must be strictly ascending per row$"):
        eng.load_abstraction(CsrBoolMatrix(1, 8, [0, 2], [5, 2]))
    with pytest.raises(ValueError, match="dimension mismatch"):
        label_all(CsrBoolMatrix(5, 5, g["offsets"], g["indices"]), DensePropMatrix.from_words(8, np.zeros((1, 1))))
    eng.close()


def test_csb1_file_loader(tmp_path):
    g = load("seed31337_csr")
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_file(os.path.join(GOLDEN, "seed31337.csb1"))  # written by the reference
    rng = SplitMix64(5)
    P = bits_to_words(random_rows(rng, 3, 2048, 0.02))
    eng.submit_grid(2048, 3, P, 1)
    want = ORACLE.label_all(64, 2048, g["offsets"], g["indices"], 2048, 3, P)
    assert eng.get_labels(0) == LabelMatrix(64, 3, want)
    bad = tmp_path / "bad.csb1"
    bad.write_bytes(b"XXXX0000")
    with pytest.raises(RuntimeError, match="^not a CSR file: "):
        eng.load_abstraction_file(str(bad))
    trunc = tmp_path / "trunc.csb1"
    trunc.write_bytes(open(os.path.join(GOLDEN, "seed31337.csb1"), "rb").read()[:100])
    with pytest.raises(RuntimeError, match="^truncated CSR file: "):
        eng.load_abstraction_file(str(trunc))
    with pytest.raises(RuntimeError, match="^cannot open: "):
        eng.load_abstraction_file(str(tmp_path / "missing.csb1"))
    eng.close()


@pytest.mark.parametrize("pose", [(0.0, 0.0, 0.0), (3.7, -2.1, 0.0), (0.0, 0.0, 0.4), (-5.5, 8.25, 2.9),
                                  (60.0, 0.0, -1.2)])
@pytest.mark.parametrize("outside", [0, 1])
def test_world_resample_then_label(pose, outside):
    vdepth, wdepth, props = 12, 14, 5
    vgrid = (vdepth, 0.0, 102.4, 0.0, 102.4)
    wgrid = (wdepth, -50.0, 150.0, -40.0, 160.0)
    world = props_words(11, wdepth, props, 0, 1)[0]
    dx, dy, th = pose
    ps = (dx, dy, math.cos(th), math.sin(th))
    want_P = ORACLE.resample(vgrid, wgrid, ps, props, world, outside)
    prm = SyntheticPRM(seed=2, depth=vdepth)
    t = prm.words(0, 5000)
    off, idx = prm.csr(0, 5000)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(5000, 1 << vdepth, t.offsets, t.words, t.masks)
    eng.submit_world_grid(vgrid, wgrid, props, world, [ps], outside=outside)
    want = ORACLE.label_all(5000, 1 << vdepth, off, idx, 1 << vdepth, props, want_P)
    assert eng.get_labels(0) == LabelMatrix(5000, props, want)
    eng.close()


def test_world_resample_batched_poses():
    vdepth, wdepth, props = 12, 12, 3
    vgrid = (vdepth, 0.0, 102.4, 0.0, 102.4)
    wgrid = (wdepth, 0.0, 102.4, 0.0, 102.4)
    world = props_words(4, wdepth, props, 0, 1)[0]
    poses = [(1.5 * k, -0.7 * k, math.cos(0.1 * k), math.sin(0.1 * k)) for k in range(6)]
    prm = SyntheticPRM(seed=2, depth=vdepth)
    t = prm.words(0, 3000)
    off, idx = prm.csr(0, 3000)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(3000, 1 << vdepth, t.offsets, t.words, t.masks)
    eng.submit_world_grid(vgrid, wgrid, props, world, poses)
    for f, ps in enumerate(poses):
        want = ORACLE.label_all(3000, 1 << vdepth, off, idx, 1 << vdepth, props,
                                ORACLE.resample(vgrid, wgrid, ps, props, world, 0))
        assert eng.get_labels(f) == LabelMatrix(3000, props, want)
    eng.close()


@pytest.mark.parametrize("frames", [1, 3])
def test_pinned_submit_then_world_grid_and_boxes(frames):
    """A fused pinned single-frame submit_grid leaves no host mapping behind:
    the next world-grid / boxes submit labels with the P it just produced
    (a stale P_host used to be re-read, or read past its end)."""
    import torch

    vdepth, props = 12, 5
    vgrid = (vdepth, 0.0, 102.4, 0.0, 102.4)
    wgrid = (vdepth, -10.0, 112.4, -10.0, 112.4)
    world = props_words(23, vdepth, props, 0, 1)[0]
    prm = SyntheticPRM(seed=3, depth=vdepth)
    E = 4000
    t = prm.words(0, E)
    off, idx = prm.csr(0, E)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << vdepth, t.offsets, t.words, t.masks)
    cells = 1 << vdepth

    def pinned_submit(seed):
        P = props_words(seed, vdepth, props, 0, 1)
        pin = torch.from_numpy(P.view(np.int64).copy()).pin_memory()
        eng.submit_grid(cells, props, pin, 1)
        assert eng.get_labels(0) == LabelMatrix(E, props, ORACLE.label_all(E, cells, off, idx, cells, props, P[0]))
        pin.fill_(-1)  # the caller reuses its buffer after the labels are back
        return pin

    keep = pinned_submit(7)
    poses = [(1.0 * k, -0.5 * k, math.cos(0.2 * k), math.sin(0.2 * k)) for k in range(frames)]
    eng.submit_world_grid(vgrid, wgrid, props, world, poses)
    for f, ps in enumerate(poses):
        want_P = ORACLE.resample(vgrid, wgrid, ps, props, world, 0)
        assert eng.get_labels(f) == LabelMatrix(E, props, ORACLE.label_all(E, cells, off, idx, cells, props, want_P))
    del keep
    keep = pinned_submit(8)
    from oracle.oracle import RefCore

    if RefCore.available():
        ref = RefCore()
        lo, hi = [0.0, 0.0], [102.4, 102.4]
        rng = np.random.default_rng(frames)
        columns = []
        for _ in range(frames * props):
            c = rng.uniform(0, 102.4, size=(3, 2))
            columns.append([((x - 4).tolist(), (x + 5).tolist()) for x in c])
        eng.submit_boxes(2, vdepth, lo, hi, columns, props, frames)
        for f in range(frames):
            P = np.stack([ref.rasterize_union(2, vdepth, lo, hi, np.array([b[0] for b in columns[f * props + j]]),
                                              np.array([b[1] for b in columns[f * props + j]])) for j in range(props)])
            want = ORACLE.label_all(E, cells, off, idx, cells, props, P)
            assert eng.get_labels(f) == LabelMatrix(E, props, want), f
    del keep
    eng.close()


def test_empty_and_degenerate():
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(0, 64, [0], []))
    eng.submit_grid(64, 3, np.zeros(3, np.uint64), 1)
    assert eng.get_labels(0) == LabelMatrix(0, 3)
    eng.load_abstraction(CsrBoolMatrix(4, 64, [0, 0, 0, 0, 0], []))
    eng.submit_grid(64, 2, np.full(2, ~np.uint64(0)), 1)
    assert eng.get_labels(0) == LabelMatrix(4, 2)  # all-false rows never hit (test_label.cpp:68-73)
    eng.submit_grid(64, 0, np.zeros(0, np.uint64), 2)
    assert eng.get_labels(1) == LabelMatrix(4, 0)
    eng.close()


@pytest.mark.parametrize("chunks", [2, 8])
@pytest.mark.parametrize("devices", [[0], [0, 0, 0]])
def test_chunked_readback(devices, chunks):
    # readback_chunks: rows z-sorted within blocks, one launch per block, the
    # label copy of block c overlapping the labelling of later blocks
    depth, E, props, F = 16, 60_001, 20, 6
    prm = SyntheticPRM(seed=21, depth=depth)
    t = prm.words(0, E)
    off, idx = prm.csr(0, E)
    P = props_words(23, depth, props, 0, F)
    eng = LabelEngine(devices=devices, readback_chunks=chunks)
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    for rep in range(2):  # twice: the per-block task counters are reset per submit
        eng.submit_grid(1 << depth, props, P, F)
        packed = eng.get_labels_packed()
        for f in range(F):
            want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f])
            assert np.array_equal(packed[:, f].astype(np.uint64), want), (rep, f)
    eng.submit_grid(1 << depth, props, P[4], 1)
    want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[4])
    assert np.array_equal(eng.get_labels_packed()[:, 0].astype(np.uint64), want)
    assert eng.get_labels(0) == LabelMatrix(E, props, want)
    # device-resident P declared for read-back (ltlg_submit_grid_device_ex)
    import torch

    Pd = torch.from_numpy(P.view(np.int64)).cuda()
    eng.submit_grid_device(1 << depth, props, Pd.data_ptr(), F, readback=True)
    packed = eng.get_labels_packed()
    for f in range(F):
        want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f])
        assert np.array_equal(packed[:, f].astype(np.uint64), want), f
    eng.close()


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0, 0, 0, 0, 0]])
def test_sharded_engine_on_one_device(devices):
    # several shards on one GPU exercise the multi-device code path (row
    # sharding, P broadcast, per-shard labels, assembly) without NCCL.
    depth, E, props, F = 14, 30_000, 12, 5
    prm = SyntheticPRM(seed=9, depth=depth)
    t = prm.words(0, E)
    off, idx = prm.csr(0, E)
    P = props_words(13, depth, props, 0, F)
    eng = LabelEngine(devices=devices)
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    eng.submit_grid(1 << depth, props, P, F)
    packed = eng.get_labels_packed()
    spans = [eng.device_labels(s)[1:3] for s in range(len(devices))]
    assert spans[0][0] == 0 and spans[-1][1] == E
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    for f in range(F):
        want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f])
        assert eng.get_labels(f) == LabelMatrix(E, props, want)
        assert np.array_equal(packed[:, f].astype(np.uint64), want)
    eng.submit_grid(1 << depth, props, P[2], 1)  # single-frame kernel on every shard
    want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[2])
    assert eng.get_labels(0) == LabelMatrix(E, props, want)
    eng.close()


def test_bench_two_ranks_on_one_gpu(tmp_path):
    """bench.py's N > 1 path (rank shards, P broadcast each step, max-over-ranks
    timing, teardown) under torchrun with two ranks sharing cuda:0 over gloo
    (NCCL refuses two ranks on one device): it must finish cleanly and rank 0
    must print one JSON line with n_gpus = 2."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(GOLDEN))
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", BENCH_FORCE_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29633", "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--quick", "--no-cpu-baseline",
                        "--dump-labels", os.path.join(str(tmp_path), "two")],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0
    assert lines[0]["e2e"]["value"] > 0
    # the two rank shards (double-buffered P broadcast overlapped with the
    # labelling) label exactly like one rank over all edges
    r1 = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--quick", "--no-cpu-baseline",
                         "--no-e2e", "--dump-labels", os.path.join(str(tmp_path), "one")],
                        cwd=root, capture_output=True, text=True, timeout=900)
    assert r1.returncode == 0, r1.stderr[-3000:]
    one = np.load(os.path.join(str(tmp_path), "one_rank0.npz"))
    pos = {int(x): i for i, x in enumerate(one["rows"])}
    checked = 0
    for rank in (0, 1):
        d = np.load(os.path.join(str(tmp_path), f"two_rank{rank}.npz"))
        for row, lab in zip(d["rows"], d["labels"]):
            if int(row) in pos:
                assert np.array_equal(lab, one["labels"][pos[int(row)]]), (rank, int(row))
                checked += 1
    assert checked > 100


def test_cpp_drop_in_parity():
    # the reference core and include/ltlgrid_gpu.hpp compiled into one binary
    import subprocess

    exe = os.path.join(os.path.dirname(GOLDEN), "..", "oracle", "_ref", "cpp_parity")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/cpp_parity not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout


def test_zobv_ingest_and_lbm1_dump(tmp_path):
    # ZOBV proposition columns in (load_bitset, grid.cpp:375-405),
    # LBM1 labels out (LabelMatrix::save, label.cpp:300-309), both byte-compatible
    # with the reference's own writers.
    from oracle.oracle import RefCore

    if not RefCore.available():
        pytest.skip("oracle/_ref not built")
    ref = RefCore()
    depth, E, props, F = 12, 7_001, 5, 2
    prm = SyntheticPRM(seed=31, depth=depth)
    off, idx = prm.csr(0, E)
    P = props_words(37, depth, props, 0, F)
    paths = []
    for f in range(F):
        for j in range(props):
            p = tmp_path / f"f{f}_p{j}.zobv"
            ref.save_bitset(str(p), 2, depth, P[f, j])
            paths.append(str(p))
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(E, 1 << depth, off, idx))
    eng.submit_grid_files(paths, props, F)
    for f in range(F):
        want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f])
        assert eng.get_labels(f) == LabelMatrix(E, props, want)
        ours, theirs = tmp_path / f"ours{f}.lbm", tmp_path / f"ref{f}.lbm"
        eng.save_labels(str(ours), f)
        ref.label_save(str(theirs), E, props, want)
        assert ours.read_bytes() == theirs.read_bytes()
    with pytest.raises(ValueError, match="column length mismatch"):
        small = tmp_path / "small.zobv"
        ref.save_bitset(str(small), 2, depth - 2, P[0, 0][: (1 << (depth - 2)) // 64])
        eng.submit_grid_files([str(small)], 1, 1)
    with pytest.raises(RuntimeError, match="cannot open"):
        eng.submit_grid_files([str(tmp_path / "nope.zobv")], 1, 1)
    eng.close()


def test_csb1_streaming_load_large(tmp_path):
    # the streaming CSB1 loader on a file with > 2^24 indices (several read
    # chunks) labels exactly like the in-memory CSR path
    from oracle.oracle import RefCore

    if not RefCore.available():
        pytest.skip("oracle/_ref not built")
    depth, E, props = 16, 120_000, 9
    prm = SyntheticPRM(seed=77, depth=depth)
    off, idx = prm.csr(0, E)
    assert idx.size > (1 << 24)
    p = tmp_path / "big.csb1"
    RefCore().csr_save(str(p), E, 1 << depth, off, idx)
    P = props_words(3, depth, props, 0, 1)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_file(str(p))
    eng.submit_grid(1 << depth, props, P[0], 1)
    want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[0])
    assert eng.get_labels(0) == LabelMatrix(E, props, want)
    eng.close()


RASTER_GRIDS = [(1, 9), (2, 6), (2, 7), (2, 12), (2, 13), (3, 9), (3, 14), (3, 21)]


@pytest.mark.parametrize("k,depth", RASTER_GRIDS)
def test_rasterize_boxes_vs_reference(k, depth):
    # GPU rasterize_box == the reference's rasterize_box (grid.cpp:260-344),
    # unions per column; boxes partly outside, degenerate (lo == hi), inverted, tiny.
    from oracle.oracle import RefCore

    if not RefCore.available():
        pytest.skip("oracle/_ref not built")
    from paper_1810_02612_b200 import rasterize_boxes

    ref = RefCore()
    rng = np.random.default_rng(1000 * k + depth)
    lo = rng.uniform(-50, 0, size=k)
    hi = lo + rng.uniform(10, 80, size=k)
    columns = []
    for c in range(7):
        boxes = []
        for _ in range(int(rng.integers(0, 6))):
            a = rng.uniform(lo - 5, hi + 5)
            b = a + rng.uniform(-2, 0.6, size=k) * (hi - lo)
            kind = rng.integers(0, 4)
            if kind == 0:
                b = a.copy()  # degenerate: zero measure
            boxes.append((a.tolist(), b.tolist()))
        columns.append(boxes)
    got = rasterize_boxes(k, depth, lo, hi, columns)
    for c, boxes in enumerate(columns):
        blo = np.array([b[0] for b in boxes]).reshape(-1, k) if boxes else np.zeros((0, k))
        bhi = np.array([b[1] for b in boxes]).reshape(-1, k) if boxes else np.zeros((0, k))
        want = ref.rasterize_union(k, depth, lo, hi, blo, bhi)
        assert np.array_equal(got[c], want), (c, boxes)


def test_submit_boxes_labels_and_errors():
    from oracle.oracle import RefCore

    if not RefCore.available():
        pytest.skip("oracle/_ref not built")
    ref = RefCore()
    depth, E, props, F = 14, 20_000, 6, 3
    prm = SyntheticPRM(seed=5, depth=depth)
    off, idx = prm.csr(0, E)
    lo, hi = [0.0, 0.0], [102.4, 102.4]
    rng = np.random.default_rng(9)
    columns = []
    for _ in range(F * props):
        boxes = []
        for _ in range(int(rng.integers(1, 7))):
            c = rng.uniform(0, 102.4, size=2)
            boxes.append(((c - 3).tolist(), (c + rng.uniform(0.1, 9, size=2)).tolist()))
        columns.append(boxes)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(E, 1 << depth, off, idx))
    eng.submit_boxes(2, depth, lo, hi, columns, props, F)
    for f in range(F):
        P = np.stack([ref.rasterize_union(2, depth, lo, hi, np.array([b[0] for b in columns[f * props + j]]),
                                          np.array([b[1] for b in columns[f * props + j]])) for j in range(props)])
        want = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P)
        assert eng.get_labels(f) == LabelMatrix(E, props, want)
    with pytest.raises(ValueError, match="dimension mismatch"):
        eng.submit_boxes(2, depth + 2, lo, hi, columns[:1], 1, 1)
    with pytest.raises(ValueError, match="grid bounds must satisfy lo < hi"):
        eng.submit_boxes(2, depth, [0.0, 5.0], [1.0, 5.0], columns[:1], 1, 1)
    with pytest.raises(ValueError, match=r"grid depth must be in \[k, 63\]"):
        eng.submit_boxes(3, 2, [0.0] * 3, [1.0] * 3, columns[:1], 1, 1)
    eng.close()


@pytest.mark.parametrize("props", [0, 5, 16, 32, 40])
def test_guard_consumer_vs_reference(props):
    # admitted-guard masks over the resident labels ==
    # TransitionGuard::admits (buchi.hpp:20-22) of the oracle's labels.
    from oracle.oracle import RefCore

    if not RefCore.available():
        pytest.skip("oracle/_ref not built")
    ref = RefCore()
    depth, E, F = 12, 9_000, 3
    prm = SyntheticPRM(seed=19, depth=depth)
    off, idx = prm.csr(0, E)
    P = props_words(41, depth, props, 0, F) if props else np.zeros((F, 0, (1 << depth) // 64), np.uint64)
    rng = np.random.default_rng(props)
    ng = 64 if props == 16 else 13
    pos = np.zeros(ng, dtype=np.uint64)
    neg = np.zeros(ng, dtype=np.uint64)
    for t in range(ng):  # guards over props 0..props+3 (some need props the labels do not carry)
        for j in rng.choice(props + 4, size=int(rng.integers(0, 4)), replace=False):
            if rng.integers(0, 2):
                pos[t] |= np.uint64(1) << np.uint64(j)
            else:
                neg[t] |= np.uint64(1) << np.uint64(j)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(E, 1 << depth, off, idx))
    eng.set_guards(pos, neg)
    for frames in (1, F):  # single-frame and multi-frame kernels
        eng.submit_grid(1 << depth, props, P[:frames], frames)
        for f in range(frames):
            labels = (ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f]) if props
                      else np.zeros(E, dtype=np.uint64))
            want = ref.guard_admits(labels.reshape(E, -1)[:, 0], pos, neg)
            assert np.array_equal(eng.get_admitted(f), want), (frames, f)
    eng.close()


def test_config5_dense_grid_slice():
    # BASELINE config 5 (1024^2 grid, 64 props) on a 300k-row slice of the 8M-edge
    # abstraction: the 64-prop entry format, the L1 (not shared-memory) summary path
    # of the single-frame kernel and the 64-prop multi-frame kernel.
    c = CONFIGS[5]
    depth, props, E = c["depth"], c["props"], 300_000
    prm = SyntheticPRM(seed=1, depth=depth)
    t = prm.words(0, E)
    off, idx = prm.csr(0, E)
    P = props_words(1, depth, props, 0, 3)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction_words(E, 1 << depth, t.offsets, t.words, t.masks)
    eng.submit_grid(1 << depth, props, P[0], 1)
    want0 = ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[0])
    assert eng.get_labels(0) == LabelMatrix(E, props, want0)
    eng.submit_grid(1 << depth, props, P, 3)
    for f in range(3):
        want = want0 if f == 0 else ORACLE.label_all(E, 1 << depth, off, idx, 1 << depth, props, P[f])
        assert eng.get_labels(f) == LabelMatrix(E, props, want)
    eng.close()


@pytest.mark.parametrize("knobs", [
    {"LTLG_STREAM64": "0", "LTLG_BATCH64": "0"},                            # 32-cell kernels
    {"LTLG_STREAM64": "0", "LTLG_STREAM_CFG": "2"},                         # double-buffered 32-cell
    {"LTLG_STREAM64": "0", "LTLG_STREAM_CFG": "4"},                         # TMA-ring 32-cell
    {"LTLG_STREAM_TABLE": "0"},                                             # summary through L1
    {"LTLG_NT64": "512"},                                                   # 64-prop kernel, 16 warps
    {"LTLG_NT64": "1024"},                                                  # 64-prop kernel, 32 warps
    {"LTLG_PROPLANE": "0"},                                                 # frame-per-lane 64-cell kernel
    {"LTLG_WORDMAJOR": "0"},                                                # pair-major prop-lane kernel
    {"LTLG_WM1": "1"},                                                      # word-major single frame everywhere
    {"LTLG_WM1": "0"},                                                      # stream64 single frame everywhere
    {"LTLG_TC": "1"},                                                       # tcgen05 kind::i8 multi-frame
])
def test_ab_variants_parity(knobs):
    # the A/B kernel variants (env knobs, read once per process) stay bit-exact;
    # they run on the A/B build of the library (the product one leaves them out)
    import subprocess
    import sys

    from paper_1810_02612_b200._native import AB_SO

    env = dict(os.environ, LTLG_DEV_SO=AB_SO, **knobs)
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(GOLDEN), "..", "tools", "ab_parity.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("knobs", [{"LTLG_TC": "1"}, {"LTLG_WORDMAJOR": "0"}, {"LTLG_STREAM64": "0"}])
def test_product_library_ignores_ab_knobs(knobs):
    # the product library has no A/B kernels: their knobs leave the default
    # dispatch in place (and the labels bit-exact)
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k != "LTLG_DEV_SO"}
    env.update(knobs)
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(GOLDEN), "..", "tools", "ab_parity.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_edge_counting_vs_golden_and_oracle():
    """ltlg_edge_counting == label_edge_counting (label.cpp:140-148) for every
    edge: the reference-generated seed-4444 fixture (test_label.cpp:155-185),
    then seeded scenes (empty rows, cells not a multiple of 64, several props and
    frames, sorted and unsorted engines, several shards) against the oracle."""
    g = load("counting_examples")
    c = load("counting_seed4444")
    r, cols = int(c["rows"]), int(c["cols"])
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(r, cols, c["offsets"], c["indices"]))
    eng.submit_grid(cols, 1, c["colwords"].reshape(1, 1, -1), 1)
    hit, ex = eng.edge_counting(0, 0)
    assert np.array_equal(np.stack([hit.astype(np.uint64), ex], 1), g["seed4444"])
    eng.close()
    for seed, devs, sort in ((1, [0], True), (2, [0], False), (3, [0, 0, 0], True)):
        rng = SplitMix64(300 + seed)
        r, cols, props, F = 1500, 64 * 40 + 17, 3, 4
        rows = random_rows(rng, r, cols, 0.01)
        rows[::13] = False  # empty rows
        off, idx = to_csr(rows)
        P = np.stack([bits_to_words(random_rows(rng, props, cols, d)) for d in (0.002, 0.02, 0.3, 0.9)])
        eng = LabelEngine(devices=devs, sort_rows=sort)
        eng.load_abstraction(CsrBoolMatrix(r, cols, off, idx))
        eng.submit_grid(cols, props, P, F)
        for f in range(F):
            for j in range(props):
                hit, ex = eng.edge_counting(f, j)
                for i in range(r):
                    h, e = ORACLE.label_edge_counting(idx[off[i]:off[i + 1]], P[f, j])
                    assert (bool(hit[i]), int(ex[i])) == (h, e), (seed, f, j, i)
        with pytest.raises(ValueError, match="prop out of range"):
            eng.edge_counting(0, props)
        eng.close()


@pytest.mark.parametrize("props", [0, 3, 64])
def test_apply_labels_vs_reference(props):
    """ltlg_apply_labels == apply_labels (label.cpp:191-210): per-edge
    AlphabetSymbol bits, and the reference's two checks in its order."""
    rng = SplitMix64(900 + props)
    r, cols = 700, 1000
    rows = random_rows(rng, r, cols, 0.01)
    off, idx = to_csr(rows)
    P = bits_to_words(random_rows(rng, props, cols, 0.02)) if props else np.zeros((0, 16), np.uint64)
    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(r, cols, off, idx))
    eng.submit_grid(cols, props, P.reshape(1, props, 16), 1)
    el = eng.apply_labels(r, props)
    want = ORACLE.label_all(r, cols, off, idx, cols, props, P) if props else np.zeros(r, np.uint64)
    assert el.alphabet_size == props and np.array_equal(el.labels, want.reshape(r, -1)[:, 0] if props else want)
    with pytest.raises(ValueError, match=f"^label matrix rows {r} vs edges {r + 1}$"):
        eng.apply_labels(r + 1, props + 1)  # rows are checked first
    with pytest.raises(ValueError, match=f"^label matrix props {props} vs alphabet size {props + 1}$"):
        eng.apply_labels(r, props + 1)
    eng.close()


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_double_buffered_P_bursts(devices):
    """P is double-buffered per shard (rotate_P): a submit's upload /
    broadcast runs on the comm stream while the previous submit labels, gated
    by the read_done event of the buffer it refills; an async device submit
    builds its summary on the comm stream after the caller's event.  Bursts of
    submits without a wait in between (pageable, pinned, device and async
    device P, several frame counts) must leave exactly the last submit's
    labels."""
    import torch

    rng = np.random.default_rng(len(devices))
    r, c = 4000, 64 * 70 + 5
    rows = rng.random((r, c)) < 0.01
    off, idx = to_csr(rows)
    eng = LabelEngine(devices=devices)
    eng.load_abstraction(CsrBoolMatrix(r, c, off, idx))
    nw = (c + 63) // 64
    for burst in range(6):
        props = int(rng.choice([3, 17, 40]))
        Ps = []
        for k in range(int(rng.integers(2, 5))):
            frames = int(rng.choice([1, 3, 20]))
            P = rng.integers(0, 2**63, size=(frames, props, nw), dtype=np.uint64)
            P[:, :, ::4] &= np.uint64(0x0101010101010101)
            P[:, :, 1::7] = np.uint64(0xFFFFFFFFFFFFFFFF)
            kind = (burst + k) % 4
            if kind == 0:
                eng.submit_grid(c, props, P, frames)
            elif kind == 1:
                eng.submit_grid(c, props, torch.from_numpy(P.view(np.int64).copy()).pin_memory(), frames)
            elif kind == 2:
                dev = torch.from_numpy(P.view(np.int64).copy()).cuda()
                eng.submit_grid_device(c, props, dev.data_ptr(), frames)
                Ps.append(dev)  # (kept alive until the labels are read)
            else:  # async: P written on a side stream, ready when its event completes
                side = torch.cuda.Stream()
                with torch.cuda.stream(side):
                    dev = torch.empty((frames, props, nw), dtype=torch.int64, device="cuda")
                    dev.copy_(torch.from_numpy(P.view(np.int64).copy()).pin_memory(), non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(side)
                eng.submit_grid_device(c, props, dev.data_ptr(), frames, ready_event=ev.cuda_event)
                Ps.extend([dev, ev, side])
            Ps.append(P)
        P = [q for q in Ps if isinstance(q, np.ndarray)][-1]
        for f in range(P.shape[0]):
            want = ORACLE.label_all(r, c, off, idx, c, props, P[f])
            assert eng.get_labels(f) == LabelMatrix(r, props, want), (burst, f)
    eng.close()
