"""Host-side mirror of the reference labeling interface, backed by the B200 engine.

Names, argument meaning and error behaviour follow
proj/core/include/ltlgrid/label.hpp (+ grid.hpp for OccupancyBitset):

  reference (C++)                          here (Python)
  ---------------------------------------  --------------------------------------
  CsrBoolMatrix         label.hpp:18-35    CsrBoolMatrix (numpy arrays)
  to_csr                label.hpp:38       to_csr
  OccupancyBitset       grid.hpp:93-125    OccupancyBitset
  DensePropMatrix       label.hpp:47-58    DensePropMatrix
  LabelMatrix           label.hpp:61-92    LabelMatrix (== compares like the reference)
  label_all             label.hpp:94-98    label_all  -> libltlgrid_gpu.so (sm_100a)
  std::invalid_argument                    ValueError
  std::runtime_error                       RuntimeError

The compute path is the C ABI of include/ltlgrid_gpu.h; there is no CPU
fallback (a missing library or device raises).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native as N


# ---------------------------------------------------------------------------
# Errors
# ---------------------------------------------------------------------------

class LtlgError(RuntimeError):
    """CUDA / NCCL / state errors of the engine."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class DomainError(ArithmeticError):
    """The reference's std::domain_error (e.g. a trajectory leaving the workspace)."""


def _raise(status: int, msg: str):
    if status == N.LTLG_EINVAL:
        raise ValueError(msg)
    if status == N.LTLG_EDOMAIN:
        raise DomainError(msg)
    if status in (N.LTLG_EFORMAT, N.LTLG_EIO):
        raise RuntimeError(msg)
    if status == N.LTLG_ENOMEM:
        raise MemoryError(msg)
    raise LtlgError(status, msg)


def _ptr(a) -> Optional[int]:
    """Raw address of a numpy array / torch tensor / int (None for empty)."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr() or None
    return a.ctypes.data if a.size else None


# ---------------------------------------------------------------------------
# OccupancyBitset / CsrBoolMatrix / DensePropMatrix / LabelMatrix
# ---------------------------------------------------------------------------

class OccupancyBitset:
    """Fixed-length bit vector over 2^depth cells (grid.hpp:93-125): u64
    little-endian words, bit i = cell i."""

    def __init__(self, size_bits: int):
        self.size_bits = int(size_bits)
        self.words = np.zeros((self.size_bits + 63) // 64, dtype=np.uint64)

    @classmethod
    def from_words(cls, size_bits: int, words) -> "OccupancyBitset":
        w = np.array(words, dtype=np.uint64).reshape(-1)
        if w.size != (size_bits + 63) // 64:
            raise ValueError("word count does not match bit length")
        b = cls.__new__(cls)
        b.size_bits = int(size_bits)
        if size_bits & 63:
            w[-1] &= np.uint64((1 << (size_bits & 63)) - 1)
        b.words = w
        return b

    def test(self, i: int) -> bool:
        return bool((int(self.words[i >> 6]) >> (i & 63)) & 1)

    def set(self, i: int) -> None:
        self.words[i >> 6] |= np.uint64(1 << (i & 63))

    def count(self) -> int:
        return int(np.unpackbits(self.words.view(np.uint8)).sum())

    def collect(self) -> np.ndarray:
        bits = np.unpackbits(self.words.view(np.uint8), bitorder="little")[: self.size_bits]
        return np.nonzero(bits)[0].astype(np.uint64)

    def __eq__(self, o) -> bool:
        return isinstance(o, OccupancyBitset) and self.size_bits == o.size_bits and np.array_equal(self.words, o.words)


class CsrBoolMatrix:
    """T: row i's set columns are col_indices[row_offsets[i]:row_offsets[i+1]],
    strictly ascending (label.hpp:18-35)."""

    def __init__(self, rows: int = 0, cols: int = 0, row_offsets=None, col_indices=None):
        self.rows = int(rows)
        self.cols = int(cols)
        self.row_offsets = np.ascontiguousarray(row_offsets if row_offsets is not None else [0], dtype=np.uint64)
        self.col_indices = np.ascontiguousarray(col_indices if col_indices is not None else [], dtype=np.uint32)

    def nnz(self) -> int:
        return int(self.col_indices.size)

    def row(self, i: int) -> np.ndarray:
        return self.col_indices[int(self.row_offsets[i]):int(self.row_offsets[i + 1])]

    def validate(self) -> None:
        """CsrBoolMatrix::validate (label.cpp:16-40): same checks, order, messages."""
        o, ix = self.row_offsets, self.col_indices
        if o.size != self.rows + 1:
            raise ValueError("row_offsets must have rows+1 entries")
        if o.size and o[0] != 0:
            raise ValueError("row_offsets must start at 0")
        if o.size > 1 and np.any(o[:-1] > o[1:]):
            raise ValueError("row_offsets must be nondecreasing")
        if o.size and int(o[-1]) != ix.size:
            raise ValueError("row_offsets must end at nnz")
        if ix.size == 0:
            return
        row_of = np.repeat(np.arange(self.rows), np.diff(o).astype(np.int64))
        bad_range = ix.astype(np.uint64) >= np.uint64(self.cols)
        same_row = np.zeros(ix.size, dtype=bool)
        same_row[1:] = row_of[1:] == row_of[:-1]
        bad_order = np.zeros(ix.size, dtype=bool)
        bad_order[1:] = same_row[1:] & (ix[:-1] >= ix[1:])
        bad = bad_range | bad_order
        if bad.any():
            k = int(np.argmax(bad))
            raise ValueError("column index out of range" if bad_range[k] else
                             "column indices must be strictly ascending per row")

    # CSB1, label.cpp:251-298
    def save(self, path: str) -> None:
        wide = self.cols > 0xFFFFFFFF or self.nnz() > 0xFFFFFFFF
        try:
            f = open(path, "wb")
        except OSError:
            raise RuntimeError("cannot open for writing: " + str(path))
        with f:
            f.write(b"CSB1")
            f.write(np.array([1 if wide else 0], "<u4").tobytes())
            f.write(np.array([self.rows, self.cols, self.nnz()], "<u8").tobytes())
            f.write(self.row_offsets.astype("<u8" if wide else "<u4").tobytes())
            f.write(self.col_indices.astype("<u8" if wide else "<u4").tobytes())

    @staticmethod
    def load(path: str) -> "CsrBoolMatrix":
        try:
            data = open(path, "rb").read()
        except OSError:
            raise RuntimeError("cannot open: " + str(path))
        if data[:4] != b"CSB1":
            raise RuntimeError("not a CSR file: " + str(path))
        if len(data) < 32:
            raise RuntimeError("truncated CSR file: " + str(path))
        flags = int(np.frombuffer(data, "<u4", 1, 4)[0])
        rows, cols, nnz = (int(x) for x in np.frombuffer(data, "<u8", 3, 8))
        if cols > 0xFFFFFFFF:
            raise RuntimeError("CSR column space too large for this build")
        wide = flags & 1
        dt, sz = ("<u8", 8) if wide else ("<u4", 4)
        need = 32 + (rows + 1) * sz + nnz * sz
        if len(data) < need:
            raise RuntimeError("truncated CSR file: " + str(path))
        off = np.frombuffer(data, dt, rows + 1, 32).astype(np.uint64)
        idx = np.frombuffer(data, dt, nnz, 32 + (rows + 1) * sz).astype(np.uint32)
        m = CsrBoolMatrix(rows, cols, off, idx)
        m.validate()
        return m


def to_csr(rows: Sequence[OccupancyBitset]) -> CsrBoolMatrix:
    """to_csr, label.cpp:42-57."""
    cols = rows[0].size_bits if len(rows) else 0
    off = [0]
    idx = []
    for r in rows:
        if r.size_bits != cols:
            raise ValueError("row length mismatch")
        c = r.collect()
        idx.append(c.astype(np.uint32))
        off.append(off[-1] + c.size)
    return CsrBoolMatrix(len(rows), cols, np.array(off, np.uint64),
                         np.concatenate(idx) if idx else np.zeros(0, np.uint32))


class DensePropMatrix:
    """P, column-major: one bitset per proposition (label.hpp:47-58)."""

    def __init__(self, cells: int, columns: Iterable[OccupancyBitset]):
        cols = list(columns)
        if len(cols) > 64:
            raise ValueError("at most 64 propositions")
        for c in cols:
            if c.size_bits != cells:
                raise ValueError("column length mismatch")
        self._cells = int(cells)
        self._columns = cols

    @classmethod
    def from_words(cls, cells: int, words: np.ndarray) -> "DensePropMatrix":
        w = np.asarray(words, dtype=np.uint64).reshape(-1, (int(cells) + 63) // 64)
        return cls(cells, [OccupancyBitset.from_words(cells, r) for r in w])

    def cells(self) -> int:
        return self._cells

    def num_props(self) -> int:
        return len(self._columns)

    def column(self, j: int) -> OccupancyBitset:
        return self._columns[j]

    def column_words(self) -> np.ndarray:
        nw = (self._cells + 63) // 64
        if not self._columns:
            return np.zeros((0, nw), np.uint64)
        return np.ascontiguousarray(np.stack([c.words for c in self._columns]))


class LabelMatrix:
    """Edge-by-proposition bits, ceil(props/64) u64 words per row (label.hpp:61-92)."""

    def __init__(self, rows: int = 0, props: int = 0, words=None):
        if props < 0 or props > 64:
            raise ValueError("props must be in [0, 64]")
        self._rows = int(rows)
        self._props = int(props)
        self._wpr = (props + 63) // 64
        n = self._rows * self._wpr
        self.bits = (np.zeros(n, np.uint64) if words is None
                     else np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)[:n].copy())

    def rows(self) -> int:
        return self._rows

    def props(self) -> int:
        return self._props

    def get(self, i: int, j: int) -> bool:
        bit = i * self._wpr * 64 + j
        return bool((int(self.bits[bit >> 6]) >> (bit & 63)) & 1)

    def set(self, i: int, j: int) -> None:
        bit = i * self._wpr * 64 + j
        self.bits[bit >> 6] |= np.uint64(1 << (bit & 63))

    def __eq__(self, o) -> bool:  # operator== (label.hpp:79): rows, props, words_per_row, bits
        return (isinstance(o, LabelMatrix) and self._rows == o._rows and self._props == o._props
                and self._wpr == o._wpr and np.array_equal(self.bits, o.bits))

    # LBM1, label.cpp:300-326
    def save(self, path: str) -> None:
        try:
            f = open(path, "wb")
        except OSError:
            raise RuntimeError("cannot open for writing: " + str(path))
        with f:
            f.write(b"LBM1")
            f.write(np.array([1], "<u4").tobytes())
            f.write(np.array([self._rows], "<u8").tobytes())
            f.write(np.array([self._props], "<u4").tobytes())
            f.write(self.bits.astype("<u8").tobytes())

    @staticmethod
    def load(path: str) -> "LabelMatrix":
        try:
            data = open(path, "rb").read()
        except OSError:
            raise RuntimeError("cannot open: " + str(path))
        if data[:4] != b"LBM1":
            raise RuntimeError("not a label matrix file: " + str(path))
        if len(data) < 8 or int(np.frombuffer(data, "<u4", 1, 4)[0]) != 1:
            raise RuntimeError("unsupported label matrix version")
        if len(data) < 20:
            raise RuntimeError("truncated label matrix file: " + str(path))
        rows = int(np.frombuffer(data, "<u8", 1, 8)[0])
        props = int(np.frombuffer(data, "<u4", 1, 16)[0])
        l = LabelMatrix(rows, props)
        n = l.bits.size
        if len(data) < 20 + 8 * n:
            raise RuntimeError("truncated label matrix file: " + str(path))
        l.bits[:] = np.frombuffer(data, "<u8", n, 20)
        return l

    def to_csv(self, names: Sequence[str]) -> str:
        """LabelMatrix::to_csv (label.cpp:328-344) given the alphabet's prop names."""
        if len(names) != self._props:
            raise ValueError("alphabet size mismatch")
        out = ["edge,propositions\n"]
        for i in range(self._rows):
            out.append(f"{i}," + " ".join(names[j] for j in range(self._props) if self.get(i, j)) + "\n")
        return "".join(out)


# ---------------------------------------------------------------------------
# The engine (load abstraction -> submit grid -> get labels)
# ---------------------------------------------------------------------------

@dataclass
class EdgeLabeling:
    """label.hpp:107-110: per-edge label sets (AlphabetSymbol::bits, one u64
    per edge, bit j = proposition j)."""
    alphabet_size: int
    labels: np.ndarray


class LabelEngine:
    """One ltlg_ctx: T resident in HBM (sharded over `devices`), per-frame P
    submissions, labels resident per shard (include/ltlgrid_gpu.h)."""

    def __init__(self, devices: Optional[Sequence[int]] = None, sort_rows: bool = True,
                 stream_task_pairs: int = 0, batch_task_pairs: int = 0, profile: bool = False,
                 readback_chunks: int = 0, task_rows: int = 0):
        self._L = N.lib()
        opts = N.Options()
        opts.sort_rows = 1 if sort_rows else 0
        opts.stream_task_pairs = stream_task_pairs
        opts.batch_task_pairs = batch_task_pairs
        opts.profile = 1 if profile else 0
        opts.readback_chunks = readback_chunks
        opts.task_rows = task_rows
        h = C.c_void_p()
        if devices is None:
            st = self._L.ltlg_create_ex(None, 1, C.byref(opts), C.byref(h))
        else:
            arr = (C.c_int * len(devices))(*devices)
            st = self._L.ltlg_create_ex(arr, len(devices), C.byref(opts), C.byref(h))
        if st:
            _raise(st, self._L.ltlg_last_error(None).decode())
        self._h = h
        self.n_devices = 1 if devices is None else len(devices)

    def close(self):
        if getattr(self, "_h", None):
            self._L.ltlg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, st: int):
        if st:
            _raise(st, self._L.ltlg_last_error(self._h).decode())

    # -- load abstraction ---------------------------------------------------
    def submit_scenario(self, cfg: Optional["ScenarioConfig"] = None, bounds=None, depth: int = 21,
                        query_index0: int = 0, frames: int = 1) -> None:
        """ltlg_submit_scenario: `frames` generate_scenario queries straight into P
        (prop 0 = moving_vehicle, prop 1 = not_nominal_lane), then labelling."""
        bounds = bounds or DEFAULT_BENCH_BOUNDS
        c = (cfg or ScenarioConfig())._c()
        g = _gridk(len(bounds), depth, [b[0] for b in bounds], [b[1] for b in bounds])
        self._ck(self._L.ltlg_submit_scenario(self._h, C.byref(c), C.byref(g), int(query_index0), frames))

    def load_swept_volume(self, sv: "SweptVolume") -> None:
        """ltlg_load_csr: the GPU-built swept-volume matrix as this engine's T."""
        self._ck(self._L.ltlg_load_csr(self._h, sv._h))

    def load_abstraction(self, m: CsrBoolMatrix) -> None:
        off = np.ascontiguousarray(m.row_offsets, dtype=np.uint64)
        idx = np.ascontiguousarray(m.col_indices, dtype=np.uint32)
        self._ck(self._L.ltlg_load_abstraction(self._h, m.rows, m.cols, _ptr(off), _ptr(idx)))

    def load_abstraction_file(self, path: str) -> None:
        self._ck(self._L.ltlg_load_abstraction_file(self._h, os.fsencode(path)))

    def load_abstraction_words(self, rows: int, cols: int, offsets, words, masks) -> None:
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        w = np.ascontiguousarray(words, dtype=np.uint32)
        mk = np.ascontiguousarray(masks, dtype=np.uint32)
        self._ck(self._L.ltlg_load_abstraction_words(self._h, rows, cols, _ptr(off), _ptr(w), _ptr(mk)))

    # -- submit grid --------------------------------------------------------
    def submit_grid(self, cells: int, num_props: int, column_words, frames: int = 1) -> None:
        """column_words: numpy (host) or a pinned torch tensor; frames x props x ceil(cells/64) u64."""
        if isinstance(column_words, np.ndarray):
            column_words = np.ascontiguousarray(column_words, dtype=np.uint64)
        self._ck(self._L.ltlg_submit_grid(self._h, cells, num_props, _ptr(column_words), frames))

    def submit_props(self, p: DensePropMatrix) -> None:
        self.submit_grid(p.cells(), p.num_props(), p.column_words(), 1)

    def submit_grid_files(self, paths: Sequence[str], num_props: int, frames: int = 1) -> None:
        """ZOBV proposition columns (paths[f * num_props + j]) -> labels
        (load_bitset grid.cpp:375-405 + DensePropMatrix + label_all)."""
        arr = (C.c_char_p * max(1, len(paths)))(*[os.fsencode(p) for p in paths])
        self._ck(self._L.ltlg_submit_grid_files(self._h, arr, num_props, frames))

    def submit_boxes(self, dims: int, depth: int, lo, hi, columns, num_props: int, frames: int = 1) -> None:
        """Rasterize boxes into P on the GPU (column f * num_props + j = union
        of columns[...] boxes) and label."""
        g = _gridk(dims, depth, lo, hi)
        off, blo, bhi = _boxes(columns)
        self._ck(self._L.ltlg_submit_boxes(self._h, C.byref(g), num_props, frames, off.ctypes.data, blo.ctypes.data,
                                           bhi.ctypes.data))

    def set_guards(self, positive, negative) -> None:
        """Monitor transition guards (TransitionGuard, buchi.hpp:16-26) whose
        admitted-masks are computed over the resident labels after every
        submit.  Empty lists turn the consumer off."""
        pos = np.ascontiguousarray(positive, dtype=np.uint64)
        neg = np.ascontiguousarray(negative, dtype=np.uint64)
        if pos.shape != neg.shape:
            raise ValueError("positive and negative guard lists differ in length")
        self._ck(self._L.ltlg_set_guards(self._h, int(pos.size), pos.ctypes.data if pos.size else None,
                                         neg.ctypes.data if neg.size else None))

    def get_admitted(self, frame: int = 0) -> np.ndarray:
        """u64 per edge: bit t = guard t admits the edge's label in `frame`."""
        out = np.zeros(max(1, self.info().rows), dtype=np.uint64)
        self._ck(self._L.ltlg_get_admitted(self._h, frame, out.ctypes.data))
        return out[: self.info().rows]

    def save_labels(self, path: str, frame: int = 0) -> None:
        """LBM1 file of one frame's labels (LabelMatrix::save, label.cpp:300-309)."""
        self._ck(self._L.ltlg_save_labels(self._h, frame, os.fsencode(path)))

    def submit_grid_device(self, cells: int, num_props: int, device_words, frames: int = 1,
                           readback: bool = False, ready_event=None) -> None:
        """P already in HBM; readback=True declares a following host read of
        the labels (block-wise labelling overlapped with the copy).
        ready_event (a recorded CUDA event handle, e.g. torch.cuda.Event's
        `cuda_event`): P is ready when it completes (ltlg_submit_grid_device_async),
        so the multi-frame summary overlaps the previous submit's labelling."""
        if ready_event is None:
            self._ck(self._L.ltlg_submit_grid_device_ex(self._h, cells, num_props, _ptr(device_words), frames,
                                                        1 if readback else 0))
        else:
            self._ck(self._L.ltlg_submit_grid_device_async(self._h, cells, num_props, _ptr(device_words), frames,
                                                           1 if readback else 0, C.c_void_p(int(ready_event))))

    def submit_world_grid(self, vehicle, world, num_props: int, world_words, poses, outside: int = 0,
                          words_on_device: bool = False) -> None:
        """vehicle/world = (depth, lo0, hi0, lo1, hi1); poses = [(dx, dy, cos, sin), ...]."""
        vg, wg = N.Grid2(*vehicle), N.Grid2(*world)
        arr = (N.Pose2 * len(poses))(*[N.Pose2(*p) for p in poses])
        if isinstance(world_words, np.ndarray):
            world_words = np.ascontiguousarray(world_words, dtype=np.uint64)
        self._ck(self._L.ltlg_submit_world_grid(self._h, C.byref(vg), C.byref(wg), num_props, _ptr(world_words),
                                                1 if words_on_device else 0, C.cast(arr, C.c_void_p), len(poses),
                                                int(outside)))

    def wait(self) -> None:
        self._ck(self._L.ltlg_wait(self._h))

    # -- get labels ---------------------------------------------------------
    def info(self) -> N.Info:
        i = N.Info()
        self._ck(self._L.ltlg_get_info(self._h, C.byref(i)))
        return i

    def get_labels(self, frame: int = 0) -> LabelMatrix:
        i = self.info()
        l = LabelMatrix(i.rows, i.props)
        buf = l.bits if l.bits.size else None
        self._ck(self._L.ltlg_get_labels(self._h, frame, _ptr(buf)))
        return l

    def apply_labels(self, num_edges: int, alphabet_size: int, frame: int = 0) -> "EdgeLabeling":
        """ltlg_apply_labels: apply_labels (label.cpp:191-210) -- one frame's
        labels as per-edge AlphabetSymbol bits, with the reference's row /
        alphabet-size checks and messages (ValueError)."""
        out = np.zeros(max(int(num_edges), 1), np.uint64)
        self._ck(self._L.ltlg_apply_labels(self._h, frame, int(num_edges), int(alphabet_size), _ptr(out)))
        return EdgeLabeling(int(alphabet_size), out[: int(num_edges)])

    def edge_counting(self, frame: int = 0, prop: int = 0):
        """ltlg_edge_counting: label_edge_counting (label.cpp:140-148) of every
        edge against column `prop` of frame `frame`, on the device.  Returns
        (hit bool[rows], examined uint64[rows])."""
        i = self.info()
        hit = np.zeros(max(i.rows, 1), np.uint8)
        ex = np.zeros(max(i.rows, 1), np.uint64)
        self._ck(self._L.ltlg_edge_counting(self._h, frame, prop, _ptr(hit), _ptr(ex)))
        return hit[: i.rows].astype(bool), ex[: i.rows]

    def get_labels_packed(self, out=None):
        """All frames, edge-major [rows, frames] of the packed label word
        (uint8/16/32/64 by prop count).  `out` may be a pinned torch tensor."""
        i = self.info()
        dt = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[i.label_bytes or 8]
        if out is None:
            out = np.zeros((i.rows, i.frames), dtype=dt)
        nbytes = out.nbytes if isinstance(out, np.ndarray) else out.numel() * out.element_size()
        self._ck(self._L.ltlg_get_labels_packed(self._h, _ptr(out), nbytes))
        return out

    def device_labels(self, shard: int = 0):
        p, b, e, d = C.c_void_p(), C.c_uint64(), C.c_uint64(), C.c_int()
        self._ck(self._L.ltlg_device_labels(self._h, shard, C.byref(p), C.byref(b), C.byref(e), C.byref(d)))
        return p.value, b.value, e.value, d.value

    def stream(self, shard: int = 0) -> int:
        s = C.c_void_p()
        self._ck(self._L.ltlg_stream(self._h, shard, C.byref(s)))
        return s.value or 0

    def set_profiling(self, on: bool) -> None:
        """Per-submit stage events on/off (ltlg_set_profiling)."""
        self._ck(self._L.ltlg_set_profiling(self._h, 1 if on else 0))

    def stage_times(self, shard: int = 0, back: int = 0):
        """(upload_ms, summary_ms, label_ms) of the submit `back` submits ago."""
        a, b, c = C.c_float(), C.c_float(), C.c_float()
        self._ck(self._L.ltlg_stage_times(self._h, shard, back, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value


def _gridk(dims: int, depth: int, lo, hi) -> "N.GridK":
    g = N.GridK()
    g.dims, g.depth = dims, depth
    for a in range(min(dims, 4)):
        g.lo[a], g.hi[a] = float(lo[a]), float(hi[a])
    return g


def _boxes(columns):
    """[[(lo, hi), ...] per column] -> (offsets u64, lo f64 flat, hi f64 flat)."""
    off = np.zeros(len(columns) + 1, dtype=np.uint64)
    lo, hi = [], []
    for c, boxes in enumerate(columns):
        for b_lo, b_hi in boxes:
            lo.extend(b_lo)
            hi.extend(b_hi)
        off[c + 1] = off[c] + len(boxes)
    lo = np.asarray(lo if lo else [0.0], dtype=np.float64)
    hi = np.asarray(hi if hi else [0.0], dtype=np.float64)
    return off, lo, hi


def rasterize_boxes(dims: int, depth: int, lo, hi, columns, device: int = 0) -> np.ndarray:
    """GPU rasterize_box (grid.cpp:260-344): column c = union of its boxes
    [(box_lo, box_hi), ...] on the k-D z-order grid GridSpec(bounds, depth).
    Returns [len(columns), ceil(2^depth/64)] u64 column words."""
    L = N.lib()
    g = _gridk(dims, depth, lo, hi)
    off, blo, bhi = _boxes(columns)
    out = np.zeros((max(1, len(columns)), ((1 << depth) + 63) // 64), dtype=np.uint64)
    st = L.ltlg_rasterize_boxes(C.byref(g), len(columns), off.ctypes.data, blo.ctypes.data, bhi.ctypes.data, device,
                                out.ctypes.data)
    if st:
        _raise(st, L.ltlg_last_error(None).decode())
    return out[: len(columns)]


class ScenarioConfig:
    """The reference benchmark scenario (ScenarioConfig, scenario.hpp:18-31); defaults are the reference's."""

    def __init__(self, loop_cx=36.0, loop_cy=36.0, loop_radius=24.0, lane_width=4.2, agent_count=3,
                 agent_speed_min=8.0, agent_speed_max=14.0, agent_length=4.6, agent_width=2.0, lateral_spread=3.5,
                 horizon=7.2, seed=1):
        self.loop_cx, self.loop_cy, self.loop_radius, self.lane_width = loop_cx, loop_cy, loop_radius, lane_width
        self.agent_count = agent_count
        self.agent_speed_min, self.agent_speed_max = agent_speed_min, agent_speed_max
        self.agent_length, self.agent_width, self.lateral_spread = agent_length, agent_width, lateral_spread
        self.horizon, self.seed = horizon, seed

    def _c(self):
        return N.Scenario(float(self.loop_cx), float(self.loop_cy), float(self.loop_radius), float(self.lane_width),
                          int(self.agent_count), float(self.agent_speed_min), float(self.agent_speed_max),
                          float(self.agent_length), float(self.agent_width), float(self.lateral_spread),
                          float(self.horizon), int(self.seed))


DEFAULT_BENCH_BOUNDS = ((0.0, 72.0), (0.0, 72.0), (0.0, 7.2))  # default_bench_grid (scenario.cpp:20-22)


def generate_scenario(cfg: Optional[ScenarioConfig] = None, bounds=DEFAULT_BENCH_BOUNDS, depth: int = 21,
                      query_index: int = 0, device: int = 0):
    """GPU generate_scenario (scenario.cpp:52-128): (moving_vehicle, not_nominal_lane)
    as OccupancyBitsets of the (x, y, tau) grid GridSpec(bounds, depth)."""
    L = N.lib()
    c = (cfg or ScenarioConfig())._c()
    g = _gridk(len(bounds), depth, [b[0] for b in bounds], [b[1] for b in bounds])
    nw = ((1 << depth) + 63) // 64
    out = np.zeros(2 * nw, dtype=np.uint64)
    st = L.ltlg_generate_scenario(C.byref(c), C.byref(g), int(query_index), device, out.ctypes.data)
    if st:
        _raise(st, L.ltlg_last_error(None).decode())
    return (OccupancyBitset.from_words(1 << depth, out[:nw]), OccupancyBitset.from_words(1 << depth, out[nw:]))


class FootprintSpec:
    """Rectangular footprint (abstraction.hpp:58-62); defaults are the reference's."""

    def __init__(self, length: float = 4.6, width: float = 2.0, ref_offset: float = -1.4):
        self.length, self.width, self.ref_offset = float(length), float(width), float(ref_offset)


def _trajectories(trajectories):
    """(sample_offsets u64 [E+1], samples f64 [S, 5]) from either that pair or
    a sequence of per-edge [n_i, 5] State5 arrays (px, py, heading, speed, tau)."""
    if isinstance(trajectories, tuple) and len(trajectories) == 2:
        off, smp = (np.asarray(x) for x in trajectories)
        if off.ndim == 1 and smp.ndim == 2 and smp.shape[1] == 5:
            return (np.ascontiguousarray(off, dtype=np.uint64),
                    np.ascontiguousarray(smp, dtype=np.float64))
    rows = [np.asarray(t, dtype=np.float64).reshape(-1, 5) for t in trajectories]
    off = np.zeros(len(rows) + 1, dtype=np.uint64)
    if rows:
        off[1:] = np.cumsum([r.shape[0] for r in rows])
    smp = np.ascontiguousarray(np.concatenate(rows) if rows else np.zeros((0, 5)), dtype=np.float64)
    return off, smp


class SweptVolume:
    """Device-resident swept-volume matrix built by ltlg_swept_volume."""

    def __init__(self, handle, lib):
        self._h, self._L = handle, lib
        self.rows = int(lib.ltlg_csr_rows(handle))
        self.cols = int(lib.ltlg_csr_cols(handle))
        self.nnz = int(lib.ltlg_csr_nnz(handle))
        self.build_ms = float(lib.ltlg_csr_build_ms(handle))

    def to_csr(self) -> CsrBoolMatrix:
        off = np.zeros(self.rows + 1, dtype=np.uint64)
        idx = np.zeros(max(self.nnz, 1), dtype=np.uint32)
        st = self._L.ltlg_csr_copy(self._h, off.ctypes.data, idx.ctypes.data)
        if st:
            _raise(st, self._L.ltlg_last_error(None).decode())
        return CsrBoolMatrix(self.rows, self.cols, off, idx[: self.nnz])

    def save(self, path: str) -> None:
        """CsrBoolMatrix::save (CSB1), byte-identical to the reference's file."""
        st = self._L.ltlg_csr_save(self._h, os.fsencode(path))
        if st:
            _raise(st, self._L.ltlg_last_error(None).decode())

    def close(self):
        if self._h:
            self._L.ltlg_csr_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def swept_volume(trajectories, footprint: Optional[FootprintSpec] = None, bounds=((0.0, 72.0), (0.0, 72.0), (0.0, 7.2)),
                 depth: int = 18, device: int = 0) -> SweptVolume:
    """GPU swept_volume_matrix (label.cpp:75-116), result left on the device."""
    L = N.lib()
    f = footprint or FootprintSpec()
    lo = [b[0] for b in bounds]
    hi = [b[1] for b in bounds]
    g = _gridk(len(bounds), depth, lo, hi) if len(bounds) <= 4 else None
    if g is None:
        raise ValueError("at most 4 grid axes in this build")
    off, smp = _trajectories(trajectories)
    fp = N.Footprint(f.length, f.width, f.ref_offset)
    h = C.c_void_p()
    st = L.ltlg_swept_volume(C.byref(g), C.byref(fp), off.size - 1, off.ctypes.data, smp.ctypes.data if smp.size else None,
                             device, C.byref(h))
    if st:
        _raise(st, L.ltlg_last_error(None).decode())
    return SweptVolume(h.value, L)


def swept_volume_matrix(trajectories, footprint: Optional[FootprintSpec] = None,
                        bounds=((0.0, 72.0), (0.0, 72.0), (0.0, 7.2)), depth: int = 18, workers: int = 0,
                        device: int = 0) -> CsrBoolMatrix:
    """Drop-in for ltlgrid::swept_volume_matrix (label.cpp:75-116): one CSR row
    per edge trajectory, the sorted z-order cells its footprint sweeps on the
    (x, y, tau) grid GridSpec(bounds, depth).  Built on the B200; `workers`
    is accepted for signature parity."""
    del workers
    sv = swept_volume(trajectories, footprint, bounds, depth, device)
    try:
        return sv.to_csr()
    finally:
        sv.close()


def read_csb1_shape(path: str):
    """Host-only streaming CSB1 read + validate + pack (the loader of
    ltlg_load_abstraction_file): (rows, cols, nnz, W32 words).  Raises like
    CsrBoolMatrix::load (label.cpp:271-298)."""
    L = N.lib()
    r, c, n, w = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    st = L.ltlg_read_csb1_words(os.fsencode(path), C.byref(r), C.byref(c), C.byref(n), C.byref(w))
    if st:
        _raise(st, L.ltlg_last_error(None).decode())
    return r.value, c.value, n.value, w.value


def read_zobv(path: str, cells: int) -> OccupancyBitset:
    """One ZOBV column of `cells` bits (load_bitset, grid.cpp:375-405)."""
    L = N.lib()
    words = np.zeros((cells + 63) // 64, dtype=np.uint64)
    st = L.ltlg_read_zobv(os.fsencode(path), cells, words.ctypes.data)
    if st:
        _raise(st, L.ltlg_last_error(None).decode())
    return OccupancyBitset.from_words(cells, words)


def label_all(m: CsrBoolMatrix, p: DensePropMatrix, workers: int = 0) -> LabelMatrix:
    """Drop-in for ltlgrid::label_all (label.cpp:150-189): L(i,j) = OR_k M(i,k) AND P(k,j),
    computed on the B200 through ltlg_label_all.  `workers` is accepted for
    signature parity; the result is identical for any value."""
    L = N.lib()
    if p.num_props() > 64:
        raise ValueError("at most 64 propositions")
    out = LabelMatrix(m.rows, p.num_props())
    off = np.ascontiguousarray(m.row_offsets, dtype=np.uint64)
    idx = np.ascontiguousarray(m.col_indices, dtype=np.uint32)
    cw = p.column_words()
    st = L.ltlg_label_all(m.rows, m.cols, _ptr(off), _ptr(idx), p.cells(), p.num_props(), _ptr(cw),
                          int(workers), _ptr(out.bits) if out.bits.size else None)
    if st:
        _raise(st, L.ltlg_last_error(None).decode())
    return out
