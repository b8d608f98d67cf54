"""Synthetic workloads (workload/libltlgrid_synth.so): the BASELINE configs' T and P.

Neither product nor checker: the input generator that the GPU engine, the CPU
oracle and the reference core all consume, so every arm sees identical T and
P.  See synth.cpp for the generator definitions.
Row i of the synthetic PRM depends only on (seed, i), so any row range can be
regenerated bit-identically -- the CPU oracle / reference time a bounded row
sample of exactly the rows the GPU labels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import ctypes as C
import os

SYNTH_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libltlgrid_synth.so")
_synth = None


def use_library(path: str) -> None:
    """Take the generator from another library that links synth.cpp (the
    reference arm uses oracle/_ref/libltlgrid_ref.so, so it loads nothing else
    of the repo).  Call before the first use."""
    global _synth, SYNTH_SO
    _synth = None
    SYNTH_SO = path


def _lib() -> C.CDLL:
    global _synth
    if _synth is not None:
        return _synth
    if not os.path.exists(SYNTH_SO):
        raise RuntimeError(f"{SYNTH_SO} is not built; run __graft_entry__.build()")
    S = C.CDLL(SYNTH_SO)
    u64, i32, vp = C.c_uint64, C.c_int, C.c_void_p
    S.synth_prm_create.argtypes = [u64, i32, C.c_double, i32]
    S.synth_prm_create.restype = vp
    S.synth_prm_free.argtypes = [vp]
    S.synth_prm_row_words.argtypes = [vp, u64, u64, vp]
    S.synth_prm_row_cells.argtypes = [vp, u64, u64, vp]
    S.synth_prm_fill_words.argtypes = [vp, u64, u64, vp, vp, vp]
    S.synth_prm_fill_cells.argtypes = [vp, u64, u64, vp, vp]
    S.synth_props.argtypes = [u64, i32, i32, u64, i32, vp]
    _synth = S
    return S

# BASELINE.json configs: k = 2 grids over 102.4 m x 102.4 m.
CONFIGS = {
    1: dict(name="cpu-oracle", edges=10_000, depth=12, props=4, frames=1),
    2: dict(name="driving-prm", edges=200_000, depth=16, props=8, frames=1),
    3: dict(name="large-abstraction", edges=2_000_000, depth=18, props=16, frames=1),
    4: dict(name="batched-frames", edges=2_000_000, depth=18, props=32, frames=64),
    5: dict(name="dense-grid-stress", edges=8_000_000, depth=20, props=64, frames=1),
}
EXTENT = 102.4
NPRIM = 2048


@dataclass
class WordT:
    rows: int
    cols: int
    offsets: np.ndarray  # u64 [rows+1]
    words: np.ndarray    # u32 [W]
    masks: np.ndarray    # u32 [W]


class SyntheticPRM:
    """Handle on the primitive library of one (seed, depth)."""

    def __init__(self, seed: int = 1, depth: int = 18, extent: float = EXTENT, nprim: int = NPRIM):
        self._S = _lib()
        self.depth = depth
        self.cells = 1 << depth
        self._h = self._S.synth_prm_create(seed, depth, extent, nprim)
        if not self._h:
            raise ValueError("unsupported synthetic grid depth (need 10..30)")

    def __del__(self):
        try:
            self._S.synth_prm_free(self._h)
        except Exception:
            pass

    def words(self, row_begin: int, row_end: int) -> WordT:
        n = row_end - row_begin
        cnt = np.zeros(n, np.uint64)
        self._S.synth_prm_row_words(self._h, row_begin, row_end, cnt.ctypes.data)
        off = np.zeros(n + 1, np.uint64)
        np.cumsum(cnt, out=off[1:])
        W = int(off[-1])
        w = np.zeros(max(W, 1), np.uint32)
        m = np.zeros(max(W, 1), np.uint32)
        self._S.synth_prm_fill_words(self._h, row_begin, row_end, off.ctypes.data, w.ctypes.data, m.ctypes.data)
        return WordT(n, self.cells, off, w[:W], m[:W])

    def csr(self, row_begin: int, row_end: int):
        """Reference CsrBoolMatrix arrays (offsets u64, indices u32) of the rows."""
        n = row_end - row_begin
        cnt = np.zeros(n, np.uint64)
        self._S.synth_prm_row_cells(self._h, row_begin, row_end, cnt.ctypes.data)
        off = np.zeros(n + 1, np.uint64)
        np.cumsum(cnt, out=off[1:])
        idx = np.zeros(max(int(off[-1]), 1), np.uint32)
        self._S.synth_prm_fill_cells(self._h, row_begin, row_end, off.ctypes.data, idx.ctypes.data)
        return off, idx[: int(off[-1])]


def props_words(seed: int, depth: int, props: int, frame0: int = 0, frames: int = 1, out=None) -> np.ndarray:
    """frames x props x ceil(2^depth/64) u64 (DensePropMatrix columns per frame)."""
    nw = ((1 << depth) + 63) // 64
    if out is None:
        out = np.zeros((frames, props, nw), np.uint64)
    ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
    _lib().synth_props(seed, depth, props, frame0, frames, ptr)
    return out
