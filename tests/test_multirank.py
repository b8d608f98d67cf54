"""Multi-rank host logic of the N>1 bench path, on CPU with gloo (world size 2).

bench.py under torchrun gives each rank a spatially compact, word-balanced
part of the abstraction's edge rows (bench.spatial_shard: rows sorted by median
swept word, cut into contiguous parts of that order), receives each frame's P by
a broadcast from rank 0 and labels its shard; the timing is the max over ranks.  Here the CPU oracle stands in for
the per-rank GPU engine so the sharding / broadcast / reassembly logic is
checked end to end against a single-process labeling.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _csr_rows(off, idx, rows):
    """The CSR arrays of the given rows (in that order)."""
    off = off.astype(np.int64)
    cnt = off[rows + 1] - off[rows]
    so = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(cnt, out=so[1:])
    return so.astype(np.uint64), idx[np.repeat(off[rows] - so[:-1], cnt) + np.arange(so[-1])]


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle.oracle import Oracle
    from workload.synth import SyntheticPRM, props_words

    E, depth, props, F = 9_001, 12, 6, 3
    cells = 1 << depth
    nw = (cells + 63) // 64
    prm = SyntheticPRM(seed=5, depth=depth)
    T = prm.words(0, E)
    ids = bench.spatial_shard(T.offsets, T.words, T.masks, rank, world)[0]
    off, idx = _csr_rows(*prm.csr(0, E), ids)
    P = torch.zeros((F, props, nw), dtype=torch.int64)
    if rank == 0:
        props_words(3, depth, props, 0, F, out=P)
    dist.broadcast(P, src=0)
    o = Oracle()
    labels = np.stack([o.label_all(len(ids), cells, off, idx, cells, props, P[f].numpy().view(np.uint64))
                       for f in range(F)], axis=1)  # edge-major like get_labels_packed
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sizes = [None] * world
    dist.all_gather_object(sizes, (ids, labels))
    if rank == 0:
        full = np.zeros((E, F), np.uint64)
        seen = np.zeros(E, np.int64)
        for rows, lab in sizes:
            full[rows] = lab
            seen[rows] += 1
        assert (seen == 1).all()  # the parts partition the rows
        np.save(os.path.join(out_dir, "sharded.npy"), full)
        np.save(os.path.join(out_dir, "tmax.npy"), t.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_labels_equal_single_process(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from oracle.oracle import Oracle
    from workload.synth import SyntheticPRM, props_words

    E, depth, props, F = 9_001, 12, 6, 3
    cells = 1 << depth
    off, idx = SyntheticPRM(seed=5, depth=depth).csr(0, E)
    P = props_words(3, depth, props, 0, F)
    want = np.stack([Oracle().label_all(E, cells, off, idx, cells, props, P[f]) for f in range(F)], axis=1)
    got = np.load(tmp_path / "sharded.npy")
    assert np.array_equal(got, want)
    assert float(np.load(tmp_path / "tmax.npy")[0]) == world  # max over ranks


def test_shard_rows_partition():
    import bench

    for E in (0, 1, 7, 2_000_000):
        for world in (1, 2, 3, 8):
            spans = [bench.shard_rows(E, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == E
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_spatial_shard_partition():
    import bench
    from workload.synth import SyntheticPRM

    T = SyntheticPRM(seed=5, depth=14).words(0, 20_000)
    off = T.offsets.astype(np.int64)
    med = T.words[off[:-1] + (off[1:] - off[:-1]) // 2]
    for world in (1, 2, 3, 8):
        parts = [bench.spatial_shard(T.offsets, T.words, T.masks, r, world) for r in range(world)]
        ids = np.concatenate([p[0] for p in parts])
        assert np.array_equal(np.sort(ids), np.arange(20_000))  # every row exactly once
        nwords = [int(p[1][-1]) for p in parts]
        assert sum(nwords) == len(T.words)
        assert max(nwords) - min(nwords) <= 2 * int((off[1:] - off[:-1]).max())  # word-balanced
        for i, (rows, so, w, m) in enumerate(parts):  # each part's arrays are its rows' own
            for k in (0, len(rows) // 2, len(rows) - 1):
                r = rows[k]
                assert np.array_equal(w[so[k]:so[k + 1]], T.words[off[r]:off[r + 1]])
                assert np.array_equal(m[so[k]:so[k + 1]], T.masks[off[r]:off[r + 1]])
            if i:  # contiguous ranges of the median-word order
                assert med[parts[i - 1][0]].max() <= med[rows].min()


def test_spatial_shard_empty_rows():
    # empty rows (including a trailing one, whose offset is len(words)) sort as
    # word 0 and still land in exactly one part
    import bench

    off = np.array([0, 2, 2, 5, 5, 6, 6], np.uint64)
    words = np.array([9, 40, 3, 4, 5, 70], np.uint32)
    masks = np.arange(1, 7, dtype=np.uint32)
    for world in (1, 2, 3):
        parts = [bench.spatial_shard(off, words, masks, r, world) for r in range(world)]
        ids = np.concatenate([p[0] for p in parts])
        assert np.array_equal(np.sort(ids), np.arange(6))
        assert sum(int(p[1][-1]) for p in parts) == len(words)


def test_synthetic_rows_are_row_addressable():
    from workload.synth import SyntheticPRM

    prm = SyntheticPRM(seed=5, depth=14)
    whole = prm.words(0, 3000)
    part = prm.words(1000, 2000)
    o0, o1 = whole.offsets[1000], whole.offsets[2000]
    assert np.array_equal(part.words, whole.words[o0:o1])
    assert np.array_equal(part.masks, whole.masks[o0:o1])
    off, idx = prm.csr(1000, 2000)
    # the cell CSR expands the same words (mask bits = z-order cells)
    cells = [(int(w) << 5) | b for w, m in zip(part.words, part.masks) for b in range(32) if (int(m) >> b) & 1]
    assert np.array_equal(idx, np.array(cells, np.uint32))
