"""Python access to the CPU oracle (TEST INFRASTRUCTURE ONLY).

Imported only by tests/, __graft_entry__.smoke() (as the checker) and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product package
(paper_1810_02612_b200) never imports this module.

Two backends:
  * ``Oracle``  -- oracle/liboracle.so, the C restatement (ltlg_oracle.c) of
    the reference labeling path, each function citing the reference file:line.
  * ``RefCore`` -- oracle/_ref/libltlgrid_ref.so, the UNMODIFIED reference core
    compiled from /root/reference by oracle/Makefile, behind ref_shim.cpp.

Plus numpy restatements of the reference test-input generators
(SplitMix64 ``random_rows`` of test_label.cpp:29-40, ``to_csr`` of
label.cpp:42-57) so fixtures can be regenerated bit-exactly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libltlgrid_ref.so")

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


# ---------------------------------------------------------------------------
# SplitMix64 (rng.hpp:10-34), vectorised
# ---------------------------------------------------------------------------

class SplitMix64:
    """Stateful SplitMix64 identical to ltlgrid::SplitMix64 (rng.hpp:10-29)."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next_block(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            k = np.arange(1, n + 1, dtype=np.uint64)
            z = self.state + k * _GOLDEN
            self.state = np.uint64(self.state + np.uint64(n) * _GOLDEN)
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            return z ^ (z >> np.uint64(31))

    def next(self) -> int:
        return int(self.next_block(1)[0])

    def uniform_block(self, n: int) -> np.ndarray:
        """SplitMix64::uniform (rng.hpp:21): (next >> 11) * 2^-53."""
        return (self.next_block(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def below(self, n: int) -> int:
        return self.next() % n if n else 0


def mix_seed(seed: int, stream: int) -> int:
    """mix_seed, rng.hpp:31-34."""
    with np.errstate(over="ignore"):
        s = np.uint64(seed) ^ (np.uint64(stream) * _GOLDEN + np.uint64(0x2545F4914F6CDD1D))
    return SplitMix64(int(s)).next()


def random_rows(rng: SplitMix64, rows: int, cols: int, density: float) -> np.ndarray:
    """random_rows of test_label.cpp:29-40: row-major Bernoulli(density)."""
    return (rng.uniform_block(rows * cols) < density).reshape(rows, cols)


def to_csr(dense: np.ndarray):
    """to_csr, label.cpp:42-57 (ascending set bits per row via collect)."""
    dense = np.asarray(dense, dtype=bool)
    rows = dense.shape[0]
    counts = dense.sum(axis=1).astype(np.uint64)
    offsets = np.zeros(rows + 1, dtype=np.uint64)
    np.cumsum(counts, out=offsets[1:])
    indices = np.nonzero(dense)[1].astype(np.uint32)
    return offsets, indices


def bits_to_words(bits: np.ndarray) -> np.ndarray:
    """Bool [n, cells] -> u64 words [n, ceil(cells/64)], LE bit i = cell i
    (OccupancyBitset layout, grid.hpp:93-125)."""
    bits = np.atleast_2d(np.asarray(bits, dtype=bool))
    n, cells = bits.shape
    nw = (cells + 63) // 64
    padded = np.zeros((n, nw * 64), dtype=bool)
    padded[:, :cells] = bits
    by = np.packbits(padded.reshape(n, nw * 8, 8), axis=2, bitorder="little").reshape(n, nw * 8)
    return np.ascontiguousarray(by).view(np.uint64).reshape(n, nw)


def words_to_bits(words: np.ndarray, cells: int) -> np.ndarray:
    words = np.atleast_2d(np.ascontiguousarray(words, dtype=np.uint64))
    by = words.view(np.uint8)
    return np.unpackbits(by, axis=1, bitorder="little")[:, :cells].astype(bool)


def labels_dense(words: np.ndarray, rows: int, props: int) -> np.ndarray:
    """LabelMatrix words (label.hpp:61-92) -> bool [rows, props]."""
    if props == 0:
        return np.zeros((rows, 0), dtype=bool)
    wpr = (props + 63) // 64
    w = np.asarray(words, dtype=np.uint64).reshape(rows, wpr)
    return words_to_bits(w, wpr * 64)[:, :props]


def dense_label(dense_rows: np.ndarray, dense_cols: np.ndarray) -> np.ndarray:
    """oracles::label_triple_loop (tests/support/oracles.hpp:203-216) as a
    boolean matrix product."""
    m = np.asarray(dense_rows, dtype=np.int64)
    p = np.asarray(dense_cols, dtype=np.int64)
    if p.shape[0] == 0:
        return np.zeros((m.shape[0], 0), dtype=bool)
    return (m @ p.T) > 0


def labels_to_words(dense: np.ndarray) -> np.ndarray:
    rows, props = dense.shape
    wpr = (props + 63) // 64
    if wpr == 0:
        return np.zeros(0, dtype=np.uint64)
    padded = np.zeros((rows, wpr * 64), dtype=bool)
    padded[:, :props] = dense
    return bits_to_words(padded).reshape(-1)


# ---------------------------------------------------------------------------
# ctypes backends
# ---------------------------------------------------------------------------

def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


class OracleError(ValueError):
    pass


class Oracle:
    """oracle/liboracle.so -- the C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = C.CDLL(path)
        u64, u32, i32 = C.c_uint64, C.c_uint32, C.c_int
        P64, P32 = C.POINTER(u64), C.POINTER(u32)
        L.oracle_label_all.argtypes = [u64, u64, P64, P32, u64, i32, P64, i32, P64, C.c_char_p, C.c_size_t]
        L.oracle_label_all.restype = i32
        L.oracle_validate_csr.argtypes = [u64, u64, P64, u64, P32, u64, C.c_char_p, C.c_size_t]
        L.oracle_validate_csr.restype = i32
        L.oracle_label_edge_counting.argtypes = [P32, u64, P64, P64]
        L.oracle_label_edge_counting.restype = i32
        L.oracle_z_index_of_cells.argtypes = [i32, i32, P64]
        L.oracle_z_index_of_cells.restype = u64
        L.oracle_z_index.argtypes = [i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.oracle_z_index.restype = u64
        L.oracle_z_index_tree_descent.argtypes = L.oracle_z_index.argtypes
        L.oracle_z_index_tree_descent.restype = u64
        L.oracle_mix_seed.argtypes = [u64, u64]
        L.oracle_mix_seed.restype = u64
        L.oracle_effective_workers.argtypes = [i32, u64]
        L.oracle_effective_workers.restype = i32
        d = C.c_double
        L.oracle_resample.argtypes = [i32, d, d, d, d, i32, d, d, d, d, d, d, d, d, i32, P64, i32, P64]
        L.oracle_resample.restype = None
        self.lib = L

    def label_all(self, rows, cols, offsets, indices, cells, props, colwords, workers=0):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint32)
        colwords = np.ascontiguousarray(colwords, dtype=np.uint64).reshape(-1)
        if colwords.size == 0:
            colwords = np.zeros(1, dtype=np.uint64)
        if indices.size == 0:
            indices = np.zeros(1, dtype=np.uint32)
        wpr = (props + 63) // 64 if 0 <= props <= 64 else 1
        out = np.zeros(max(rows * wpr, 1), dtype=np.uint64)
        err = C.create_string_buffer(256)
        rc = self.lib.oracle_label_all(rows, cols, _p(offsets, C.c_uint64), _p(indices, C.c_uint32),
                                       cells, props, _p(colwords, C.c_uint64), workers,
                                       _p(out, C.c_uint64), err, 256)
        if rc:
            raise OracleError(err.value.decode())
        return out[: rows * wpr]

    def validate_csr(self, rows, cols, offsets, indices):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint32)
        err = C.create_string_buffer(256)
        rc = self.lib.oracle_validate_csr(rows, cols, _p(offsets, C.c_uint64), offsets.size,
                                          _p(indices, C.c_uint32), indices.size, err, 256)
        return None if rc == 0 else err.value.decode()

    def label_edge_counting(self, row, column_words):
        row = np.ascontiguousarray(row, dtype=np.uint32)
        col = np.ascontiguousarray(column_words, dtype=np.uint64)
        ex = C.c_uint64(0)
        hit = self.lib.oracle_label_edge_counting(_p(row, C.c_uint32), row.size, _p(col, C.c_uint64), C.byref(ex))
        return bool(hit), ex.value

    def z_index_of_cells(self, k, depth, cells):
        c = np.ascontiguousarray(cells, dtype=np.uint64)
        return self.lib.oracle_z_index_of_cells(k, depth, _p(c, C.c_uint64))

    def _zcall(self, fn, k, depth, lo, hi, p):
        a = [np.ascontiguousarray(x, dtype=np.float64) for x in (lo, hi, p)]
        r = fn(k, depth, *[_p(x, C.c_double) for x in a])
        if r == 0xFFFFFFFFFFFFFFFF:
            raise IndexError("point outside workspace bounds")
        return r

    def z_index(self, k, depth, lo, hi, p):
        return self._zcall(self.lib.oracle_z_index, k, depth, lo, hi, p)

    def z_index_tree_descent(self, k, depth, lo, hi, p):
        return self._zcall(self.lib.oracle_z_index_tree_descent, k, depth, lo, hi, p)

    def mix_seed(self, seed, stream):
        return self.lib.oracle_mix_seed(seed, stream)

    def effective_workers(self, workers, items):
        return self.lib.oracle_effective_workers(workers, items)

    def resample(self, vgrid, wgrid, pose, props, world_cols, outside=0):
        """vgrid/wgrid = (depth, lo0, hi0, lo1, hi1); pose = (dx, dy, cos, sin)."""
        dv = vgrid[0]
        vwords = ((1 << dv) + 63) // 64
        out = np.zeros(max(vwords * props, 1), dtype=np.uint64)
        wc = np.ascontiguousarray(world_cols, dtype=np.uint64).reshape(-1)
        self.lib.oracle_resample(*vgrid, *wgrid, *pose, props, _p(wc, C.c_uint64), int(outside),
                                 _p(out, C.c_uint64))
        return out[: vwords * props]

    def swept_volume(self, depth, lo, hi, footprint, sample_off, samples):
        """swept_volume_matrix restatement (oracle_swept_volume): returns
        (row_offsets u64, cols u32); raises OracleError / DomainError."""
        L = self.lib
        d = C.c_double
        L.oracle_swept_volume.argtypes = [C.c_int, C.POINTER(d), C.POINTER(d), d, d, d, C.c_uint64,
                                          C.POINTER(C.c_uint64), C.POINTER(d), C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint32), C.c_uint64, C.c_char_p, C.c_size_t]
        L.oracle_swept_volume.restype = C.c_int
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        off = np.ascontiguousarray(sample_off, dtype=np.uint64)
        smp = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1)
        edges = off.size - 1
        rows = np.zeros(edges + 1, dtype=np.uint64)
        err = C.create_string_buffer(256)
        args = (depth, _p(lo, d), _p(hi, d), *map(float, footprint), edges, _p(off, C.c_uint64), _p(smp, d),
                _p(rows, C.c_uint64))
        rc = L.oracle_swept_volume(*args, None, 0, err, 256)
        if rc == 0:
            cols = np.zeros(max(int(rows[-1]), 1), dtype=np.uint32)
            rc = L.oracle_swept_volume(*args, _p(cols, C.c_uint32), cols.size, err, 256)
        if rc == 3:
            raise DomainError(err.value.decode())
        if rc != 0:
            raise OracleError(err.value.decode())
        return rows, cols[: int(rows[-1])]


class DomainError(ArithmeticError):
    """The reference's std::domain_error."""


class RefCore:
    """oracle/_ref/libltlgrid_ref.so -- the unmodified reference core."""

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        L = C.CDLL(path)
        u64, u32, i32 = C.c_uint64, C.c_uint32, C.c_int
        P64, P32 = C.POINTER(u64), C.POINTER(u32)
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_concurrency.restype = i32
        L.ref_csr_create.argtypes = [u64, u64, P64, P32]
        L.ref_csr_create.restype = C.c_void_p
        L.ref_csr_free.argtypes = [C.c_void_p]
        L.ref_props_create.argtypes = [u64, i32, P64]
        L.ref_props_create.restype = C.c_void_p
        L.ref_props_free.argtypes = [C.c_void_p]
        L.ref_time_label_ms.argtypes = [C.c_void_p, C.c_void_p, i32, i32, P64]
        L.ref_time_label_ms.restype = C.c_double
        L.ref_label_all.argtypes = [u64, u64, P64, P32, u64, i32, P64, i32, P64]
        L.ref_label_all.restype = i32
        L.ref_csr_validate.argtypes = [u64, u64, P64, u64, P32, u64]
        L.ref_csr_validate.restype = i32
        L.ref_label_edge_counting.argtypes = [P32, u64, u64, P64, P64]
        L.ref_label_edge_counting.restype = i32
        L.ref_csr_save.argtypes = [C.c_char_p, u64, u64, P64, P32]
        L.ref_csr_save.restype = i32
        L.ref_csr_load.argtypes = [C.c_char_p, P64, P64, P64, P32]
        L.ref_csr_load.restype = C.c_int64
        L.ref_label_save.argtypes = [C.c_char_p, u64, i32, P64]
        L.ref_label_save.restype = i32
        L.ref_z_index.argtypes = [i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_z_index.restype = u64
        L.ref_rasterize_union.argtypes = [i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double), u64,
                                          C.POINTER(C.c_double), C.POINTER(C.c_double), P64]
        L.ref_rasterize_union.restype = i32
        L.ref_guard_admits.argtypes = [u64, P64, i32, P64, P64, P64]
        L.ref_guard_admits.restype = None
        L.ref_save_bitset.argtypes = [C.c_char_p, i32, i32, P64]
        L.ref_save_bitset.restype = i32
        L.ref_label_load.argtypes = [C.c_char_p, P64, C.POINTER(i32), P64, u64]
        L.ref_label_load.restype = i32
        L.ref_label_to_csv.argtypes = [u64, i32, P64, C.c_char_p, C.c_char_p, u64]
        L.ref_label_to_csv.restype = C.c_int64
        L.ref_to_csr.argtypes = [u64, u64, P64, P64, P32, u64]
        L.ref_to_csr.restype = C.c_int64
        self.lib = L

    def label_load(self, path):
        """LabelMatrix::load (label.cpp:311-326) -> (rows, props, words) or raises RuntimeError/ValueError."""
        rows, props = C.c_uint64(0), C.c_int(0)
        if self.lib.ref_label_load(str(path).encode(), C.byref(rows), C.byref(props), None, 0):
            raise RuntimeError(self.error())
        n = rows.value * ((props.value + 63) // 64)
        out = np.zeros(max(n, 1), np.uint64)
        self.lib.ref_label_load(str(path).encode(), C.byref(rows), C.byref(props), _p(out, C.c_uint64), out.size)
        return rows.value, props.value, out[:n]

    def label_to_csv(self, rows, props, words, names):
        """LabelMatrix::to_csv (label.cpp:328-344) with Alphabet(names)."""
        w = np.ascontiguousarray(words, dtype=np.uint64)
        if w.size == 0:
            w = np.zeros(1, np.uint64)
        nm = "".join(n + "\n" for n in names).encode()
        n = self.lib.ref_label_to_csv(rows, props, _p(w, C.c_uint64), nm, None, 0)
        if n < 0:
            raise ValueError(self.error())
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_label_to_csv(rows, props, _p(w, C.c_uint64), nm, buf, n + 1)
        return buf.raw[:n].decode()

    def to_csr(self, rows, cols, words):
        """to_csr (label.cpp:42-57) of dense bitset rows (ceil(cols/64) u64 words each)."""
        w = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)
        if w.size == 0:
            w = np.zeros(1, np.uint64)
        off = np.zeros(rows + 1, np.uint64)
        n = self.lib.ref_to_csr(rows, cols, _p(w, C.c_uint64), _p(off, C.c_uint64), None, 0)
        if n < 0:
            raise ValueError(self.error())
        idx = np.zeros(max(n, 1), np.uint32)
        self.lib.ref_to_csr(rows, cols, _p(w, C.c_uint64), _p(off, C.c_uint64), _p(idx, C.c_uint32), idx.size)
        return off, idx[:n]

    def error(self) -> str:
        return self.lib.ref_last_error().decode()

    def hardware_concurrency(self) -> int:
        return self.lib.ref_hardware_concurrency()

    def label_all(self, rows, cols, offsets, indices, cells, props, colwords, workers=0):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint32)
        if indices.size == 0:
            indices = np.zeros(1, dtype=np.uint32)
        colwords = np.ascontiguousarray(colwords, dtype=np.uint64).reshape(-1)
        if colwords.size == 0:
            colwords = np.zeros(1, dtype=np.uint64)
        wpr = (props + 63) // 64 if 0 <= props <= 64 else 1
        out = np.zeros(max(rows * wpr, 1), dtype=np.uint64)
        rc = self.lib.ref_label_all(rows, cols, _p(offsets, C.c_uint64), _p(indices, C.c_uint32), cells,
                                    props, _p(colwords, C.c_uint64), workers, _p(out, C.c_uint64))
        if rc:
            raise OracleError(self.error())
        return out[: rows * wpr]

    def validate_csr(self, rows, cols, offsets, indices):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint32)
        ind = indices if indices.size else np.zeros(1, dtype=np.uint32)
        rc = self.lib.ref_csr_validate(rows, cols, _p(offsets, C.c_uint64), offsets.size,
                                       _p(ind, C.c_uint32), indices.size)
        return None if rc == 0 else self.error()

    def label_edge_counting(self, row, cells, column_words):
        row = np.ascontiguousarray(row, dtype=np.uint32)
        col = np.ascontiguousarray(column_words, dtype=np.uint64)
        ex = C.c_uint64(0)
        hit = self.lib.ref_label_edge_counting(_p(row, C.c_uint32), row.size, cells, _p(col, C.c_uint64), C.byref(ex))
        return bool(hit), ex.value

    def z_index(self, k, depth, lo, hi, p):
        a = [np.ascontiguousarray(x, dtype=np.float64) for x in (lo, hi, p)]
        r = self.lib.ref_z_index(k, depth, *[_p(x, C.c_double) for x in a])
        if r == 0xFFFFFFFFFFFFFFFF:
            raise IndexError(self.error())
        return r

    def csr_save(self, path, rows, cols, offsets, indices):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint32)
        if indices.size == 0:
            indices = np.zeros(1, dtype=np.uint32)
        if self.lib.ref_csr_save(path.encode(), rows, cols, _p(offsets, C.c_uint64), _p(indices, C.c_uint32)):
            raise OracleError(self.error())

    def csr_load_shape(self, path):
        """CsrBoolMatrix::load (label.cpp:271-298) -> (rows, cols, nnz); raises
        OracleError with the reference's what() text."""
        rows, cols = C.c_uint64(), C.c_uint64()
        n = self.lib.ref_csr_load(path.encode(), C.byref(rows), C.byref(cols), None, None)
        if n < 0:
            raise OracleError(self.error())
        return rows.value, cols.value, n

    def rasterize_union(self, k, depth, lo, hi, box_lo, box_hi):
        """OR of the reference's rasterize_box (grid.cpp:331-335) over boxes
        (box_lo/box_hi: nboxes x k) of GridSpec(bounds, depth)."""
        D = C.POINTER(C.c_double)
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        blo = np.ascontiguousarray(box_lo, dtype=np.float64).reshape(-1)
        bhi = np.ascontiguousarray(box_hi, dtype=np.float64).reshape(-1)
        n = blo.size // k
        if n == 0:
            blo = bhi = np.zeros(1, dtype=np.float64)
        out = np.zeros(((1 << depth) + 63) // 64, dtype=np.uint64)
        if self.lib.ref_rasterize_union(k, depth, lo.ctypes.data_as(D), hi.ctypes.data_as(D), n,
                                        blo.ctypes.data_as(D), bhi.ctypes.data_as(D), _p(out, C.c_uint64)):
            raise OracleError(self.error())
        return out

    def guard_admits(self, labels, positive, negative):
        """TransitionGuard::admits (buchi.hpp:20-22): bit t of out[i] = guard t
        admits labels[i]."""
        labels = np.ascontiguousarray(labels, dtype=np.uint64).reshape(-1)
        pos = np.ascontiguousarray(positive, dtype=np.uint64)
        neg = np.ascontiguousarray(negative, dtype=np.uint64)
        out = np.zeros(max(1, labels.size), dtype=np.uint64)
        lab = labels if labels.size else np.zeros(1, dtype=np.uint64)
        g = max(1, pos.size)
        self.lib.ref_guard_admits(labels.size, _p(lab, C.c_uint64), pos.size,
                                  _p(pos if pos.size else np.zeros(g, np.uint64), C.c_uint64),
                                  _p(neg if neg.size else np.zeros(g, np.uint64), C.c_uint64), _p(out, C.c_uint64))
        return out[: labels.size]

    def label_save(self, path, rows, props, words):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if words.size == 0:
            words = np.zeros(1, dtype=np.uint64)
        if self.lib.ref_label_save(path.encode(), rows, props, _p(words, C.c_uint64)):
            raise OracleError(self.error())

    def save_bitset(self, path, k, depth, words):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if self.lib.ref_save_bitset(path.encode(), k, depth, _p(words, C.c_uint64)):
            raise OracleError(self.error())

    # timing handles (bench cpu_baseline / --impl reference)
    def csr_handle(self, rows, cols, offsets, indices):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint32)
        if indices.size == 0:
            indices = np.zeros(1, dtype=np.uint32)
        return self.lib.ref_csr_create(rows, cols, _p(offsets, C.c_uint64), _p(indices, C.c_uint32))

    def props_handle(self, cells, props, colwords):
        colwords = np.ascontiguousarray(colwords, dtype=np.uint64).reshape(-1)
        h = self.lib.ref_props_create(cells, props, _p(colwords, C.c_uint64))
        if not h:
            raise OracleError(self.error())
        return h

    def time_label_ms(self, m, p, workers=0, repeats=2, out=None):
        return self.lib.ref_time_label_ms(m, p, workers, repeats, _p(out, C.c_uint64) if out is not None else None)

    def abstraction(self, x=(0.0, 64.0), y=(0.0, 64.0), speed=(4.0, 8.0), tau=(0.2, 2.5), tau_limit=3.9,
                    target_edges=50, seed=17):
        """build_abstraction (Rect region) -> (sample_off u64, samples (n, 5) f64)."""
        L = self.lib
        d, u64 = C.c_double, C.c_uint64
        L.ref_abstraction_create.argtypes = [d] * 9 + [u64, u64]
        L.ref_abstraction_create.restype = C.c_void_p
        L.ref_abstraction_sizes.argtypes = [C.c_void_p, C.POINTER(u64), C.POINTER(u64)]
        L.ref_abstraction_export.argtypes = [C.c_void_p, C.POINTER(u64), C.POINTER(d)]
        L.ref_abstraction_free.argtypes = [C.c_void_p]
        h = L.ref_abstraction_create(*x, *y, *speed, *tau, tau_limit, target_edges, seed)
        if not h:
            raise RuntimeError(self.error())
        try:
            e, n = u64(0), u64(0)
            L.ref_abstraction_sizes(h, C.byref(e), C.byref(n))
            off = np.zeros(e.value + 1, dtype=np.uint64)
            smp = np.zeros((max(n.value, 1), 5), dtype=np.float64)
            L.ref_abstraction_export(h, _p(off, u64), _p(smp, d))
            return off, smp[: n.value]
        finally:
            L.ref_abstraction_free(h)

    def loop_abstraction(self, depth, target_edges, seed=1):
        """The reference benchmark roadmap (loop_abstraction_config + build_abstraction)
        -> (sample_off u64, samples (n, 5) f64)."""
        L = self.lib
        u64, d = C.c_uint64, C.c_double
        L.ref_loop_abstraction_create.argtypes = [C.c_int, u64, u64]
        L.ref_loop_abstraction_create.restype = C.c_void_p
        L.ref_abstraction_sizes.argtypes = [C.c_void_p, C.POINTER(u64), C.POINTER(u64)]
        L.ref_abstraction_export.argtypes = [C.c_void_p, C.POINTER(u64), C.POINTER(d)]
        L.ref_abstraction_free.argtypes = [C.c_void_p]
        h = L.ref_loop_abstraction_create(depth, target_edges, seed)
        if not h:
            raise RuntimeError(self.error())
        try:
            e, n = u64(0), u64(0)
            L.ref_abstraction_sizes(h, C.byref(e), C.byref(n))
            off = np.zeros(e.value + 1, dtype=np.uint64)
            smp = np.zeros((max(n.value, 1), 5), dtype=np.float64)
            L.ref_abstraction_export(h, _p(off, u64), _p(smp, d))
            return off, smp[: n.value]
        finally:
            L.ref_abstraction_free(h)

    def swept_volume(self, depth, lo, hi, footprint, sample_off, samples, workers=0):
        """The reference swept_volume_matrix -> (row_offsets u64, cols u32)."""
        L = self.lib
        d, u64 = C.c_double, C.c_uint64
        L.ref_swept_volume.argtypes = [C.c_int, C.POINTER(d), C.POINTER(d), d, d, d, u64, C.POINTER(u64),
                                       C.POINTER(d), C.c_int, C.POINTER(u64), C.POINTER(C.c_uint32), u64]
        L.ref_swept_volume.restype = C.c_int64
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        off = np.ascontiguousarray(sample_off, dtype=np.uint64)
        smp = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1)
        edges = off.size - 1
        rows = np.zeros(edges + 1, dtype=np.uint64)
        args = (depth, _p(lo, d), _p(hi, d), *map(float, footprint), edges, _p(off, u64), _p(smp, d), workers,
                _p(rows, u64))
        nnz = L.ref_swept_volume(*args, None, 0)
        if nnz >= 0:
            cols = np.zeros(max(nnz, 1), dtype=np.uint32)
            nnz = L.ref_swept_volume(*args, _p(cols, C.c_uint32), cols.size)
        if nnz < 0:
            msg = self.error()
            if msg.startswith("domain_error: "):
                raise DomainError(msg[len("domain_error: "):])
            raise OracleError(msg.split(": ", 1)[-1])
        return rows, cols[:nnz]

    def generate_scenario(self, cfg, agent_count, seed, lo, hi, depth, query_index):
        """generate_scenario -> (moving_vehicle words, not_nominal_lane words)."""
        L = self.lib
        d = C.c_double
        L.ref_generate_scenario.argtypes = [C.POINTER(d), C.c_int, C.c_uint64, C.POINTER(d), C.POINTER(d), C.c_int,
                                            C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_generate_scenario.restype = C.c_int
        c = np.ascontiguousarray(cfg, dtype=np.float64)
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        nw = ((1 << depth) + 63) // 64
        out = np.zeros(2 * nw, dtype=np.uint64)
        rc = L.ref_generate_scenario(_p(c, d), agent_count, seed, _p(lo, d), _p(hi, d), depth, query_index,
                                     _p(out, C.c_uint64))
        if rc:
            msg = self.error()
            if msg.startswith("domain_error: "):
                raise DomainError(msg[len("domain_error: "):])
            raise OracleError(msg)
        return out[:nw], out[nw:]

    def free(self, m=None, p=None):
        if m:
            self.lib.ref_csr_free(m)
        if p:
            self.lib.ref_props_free(p)
