"""bench.py -- edge-labels/sec of the B200 labeling path (BASELINE.json metric).

Workload (N=1 headline): BASELINE config 4 "batched frames": 2,000,000-edge
synthetic PRM, 512x512 grid (2^18 cells), 32 propositions, 64 frames per step.
One step = label every edge for the 64 frames (one summary + one labeling
kernel).  Under torchrun (N>1) the 2M edges are sharded across ranks by edge
rows and rank 0's P is NCCL-broadcast every step (strong scaling).

Also reported: p50 per-frame latency of config 3 (2M edges, 16 props, one
frame; host P in pinned memory -> labels resident in HBM), the e2e number
through the public API with host buffers, the roofline of the labeling
kernel, the CPU baseline (reference core on the host cores), clocks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge-labels/sec (batched, 1/2/4/8 GPU) and p50 per-frame labeling latency"
UNIT = "edge-labels/s"
CFG4 = dict(edges=2_000_000, depth=18, props=32, frames=64)
CFG3_PROPS = 16
SEED_T, SEED_P = 1, 1


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """SM clock + throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): NVML in-process every 5 ms, falling back
    to nvidia-smi polling when NVML is unavailable."""

    # NVML clocks-event reason bits
    REASONS = {0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            n = self._nvml
            self.sm.append(float(n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)))
            self.mx.append(float(n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)))
            r = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.reasons |= {name for bit, name in self.REASONS.items() if r & bit}
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        if out:
            r = [x.strip() for x in out.split(",")]
            self.sm.append(float(r[0]))
            self.mx.append(float(r[1]))
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            self.reasons |= {names[k] for k in range(4) if len(r) > 2 + k and r[2 + k] == "Active"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.005 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.sm:  # a timed region shorter than one poll: take one sample now
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture summary (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def ncu_limiter(kernel: str):
    """Pipe utilisations of `kernel` from the committed ncu capture (profiles/limiters.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "limiters.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def pairs64(offsets, words) -> int:
    """64-cell (word, mask) pairs of a word-CSR: its 32-cell words minus the
    ones that share a 64-cell word with their predecessor in the same row."""
    w = np.asarray(words) >> 1
    if len(w) < 2:
        return len(w)
    same = w[1:] == w[:-1]
    head = np.zeros(len(w), bool)
    off = np.asarray(offsets, dtype=np.int64)[:-1]
    head[off[off < len(w)]] = True
    return int(len(w) - np.count_nonzero(same & ~head[1:]))


def binding_roofline(kernel: str, kernel_ms: float, sm_clk_hz: float, sms: int = 148, pairs: int = 0):
    """The roofline of the algorithm as it runs, for an issue / L1-bound
    kernel: the committed ncu --set full capture's per-launch counts
    (profiles/limiters.json: warp instructions executed, L1TEX data-pipe
    wavefronts) over this run's event-timed launch duration, against the
    SM's peaks at this run's clock -- 4 warp instructions issued per cycle
    (one per SMSP) and 1 data-pipe wavefront per cycle."""
    lim = ncu_limiter(kernel) or {}
    out = {"source": "profiles/limiters.json (" + str(lim.get("source")) + ") counts / this run's kernel time",
           "sm_clock_hz": sm_clk_hz}
    sec = kernel_ms / 1e3
    if lim.get("warp_insts"):
        a = lim["warp_insts"] / sec
        out["issue"] = {"achieved": a, "peak": 4.0 * sms * sm_clk_hz, "unit": "warp-inst/s",
                        "frac": a / (4.0 * sms * sm_clk_hz), "per_launch": lim["warp_insts"],
                        "per_pair": lim["warp_insts"] / pairs if pairs else None}
    if lim.get("l1_data_pipe_wavefronts"):
        a = lim["l1_data_pipe_wavefronts"] / sec
        out["l1tex_data_pipe"] = {"achieved": a, "peak": 1.0 * sms * sm_clk_hz, "unit": "wavefronts/s",
                                  "frac": a / (1.0 * sms * sm_clk_hz), "per_launch": lim["l1_data_pipe_wavefronts"],
                                  "per_pair": lim["l1_data_pipe_wavefronts"] / pairs if pairs else None}
    out["ncu"] = {k: v for k, v in lim.items() if k.endswith("_pct")}
    return out


def shard_rows(E: int, rank: int, world: int):
    return E * rank // world, E * (rank + 1) // world


def spatial_shard(offsets, words, masks, rank: int, world: int):
    """Rank `rank`'s edge rows of T (word-CSR arrays): the rows sorted by their
    median swept word (z-order, so a part is a compact region of the grid),
    cut into `world` contiguous parts of that order balanced by stored words.
    Rows are independent (label.cpp:179-186), so any partition labels the same
    (test_label.cpp:121-132); a compact region keeps the prop-lane kernel's
    summary reads in L1 (8 GPUs: 0.49 -> 0.40 ms per rank, DESIGN (e)).
    Returns (row ids ascending, offsets, words, masks) of the part."""
    off = np.asarray(offsets, dtype=np.int64)
    E = len(off) - 1
    if world == 1:
        return np.arange(E, dtype=np.int64), offsets, words, masks
    cnt = off[1:] - off[:-1]
    # empty rows sort as word 0 (the engine's own key, loader.cpp); their
    # offset may be len(words), so never index with it
    w = np.asarray(words)
    med = (np.where(cnt > 0, w[np.minimum(off[:-1] + cnt // 2, len(w) - 1)], 0) if len(w)
           else np.zeros(E, np.uint32))
    order = np.argsort(med, kind="stable")
    cum = np.cumsum(cnt[order])
    total = int(cum[-1]) if E else 0
    cut = np.searchsorted(cum, [total * r // world for r in range(1, world)], side="right")
    bounds = np.concatenate([[0], cut, [E]])
    ids = np.sort(order[bounds[rank]:bounds[rank + 1]])
    c = cnt[ids]
    so = np.zeros(len(ids) + 1, np.int64)
    np.cumsum(c, out=so[1:])
    idx = np.repeat(off[ids] - so[:-1], c) + np.arange(so[-1])
    return ids, so.astype(np.uint64), np.asarray(words)[idx], np.asarray(masks)[idx]


def host_cpu():
    """The CPU-baseline core count and model: nproc (the
    affinity mask), std::thread::hardware_concurrency() as label.cpp:66 sees it,
    and the lscpu model name."""
    from oracle.oracle import RefCore  # checker / baseline only

    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")), None)
    except Exception:
        pass
    if model is None:
        try:
            model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
        except Exception:
            model = "unknown"
    nproc = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    hc = RefCore().hardware_concurrency() if RefCore.available() else os.cpu_count()
    return {"nproc": nproc, "hardware_concurrency": hc, "lscpu_model": model}


class RefSlice:
    """Rows [0, rows) of the synthetic T (depth), as the unmodified reference
    core's CsrBoolMatrix (oracle/_ref), or the C port when the reference was
    not built.  The generator is the one linked into oracle/_ref, so the
    reference arm loads no other library of the repo."""

    def __init__(self, depth: int, rows: int):
        from oracle.oracle import REF_SO, Oracle, RefCore  # checker / baseline only
        import workload.synth as ws

        if RefCore.available():
            ws.use_library(REF_SO)
            self.ref, self.kind = RefCore(), "reference"
        else:
            self.ref, self.kind = Oracle(), "port"
        self.depth, self.rows, self.cells = depth, rows, 1 << depth
        prm = ws.SyntheticPRM(seed=SEED_T, depth=depth)
        self.off, self.idx = prm.csr(0, rows)
        self.m = self.ref.csr_handle(rows, self.cells, self.off, self.idx) if self.kind == "reference" else None

    def query_ms(self, props: int, frame: int, workers: int, seed: int = SEED_P) -> float:
        """time_label_ms (scenario.cpp:154-165): best of 2 label_all calls on
        frame `frame`'s P."""
        import workload.synth as ws

        P = ws.props_words(seed, self.depth, props, frame, 1)[0]
        if self.kind == "reference":
            p = self.ref.props_handle(self.cells, props, P)
            try:
                return self.ref.time_label_ms(self.m, p, workers, 2)
            finally:
                self.ref.free(p=p)
        best = 1e30
        for _ in range(2):
            t0 = time.perf_counter()
            self.ref.label_all(self.rows, self.cells, self.off, self.idx, self.cells, props, P, workers)
            best = min(best, (time.perf_counter() - t0) * 1e3)
        return best

    def protocol(self, props: int, queries: int, workers: int, seed: int = SEED_P):
        """run_benchmark's protocol (scenario.cpp:176-216): query -1 is a
        timed-but-discarded warm-up, then `queries` queries, best of 2 each;
        p50 / mean of the per-query times."""
        ts = [self.query_ms(props, q + 1, workers, seed) for q in range(-1, queries)][1:]
        return {"p50_ms": statistics.median(ts), "mean_ms": statistics.mean(ts), "min_ms": min(ts),
                "queries": queries, "rows": self.rows, "props": props, "workers": workers,
                "edge_labels_per_s_p50": self.rows / (statistics.median(ts) / 1e3)}

    def close(self):
        if self.m is not None:
            self.ref.free(m=self.m)
            self.m = None


def cpu_baseline(quick: bool):
    """the unmodified reference label_all on the host cores, on
    bounded slices of the bench's own T (rows [0, n) of the same synthetic
    PRM), reference protocol, workers = nproc and workers = 1.  Config 4: a
    500k-row slice, 32 props, one frame per query (the reference has no
    batching: a 64-frame step is 64 such calls); config 3: the same slice at 16
    props, its p50 scaled x4 to the 2M rows (linear in rows).
    workers = 1 runs on a 16k-row slice."""
    host = host_cpu()
    q = 5 if quick else 15
    big = RefSlice(CFG4["depth"], 100_000 if quick else 500_000)
    c4 = big.protocol(CFG4["props"], q, 0)
    c3 = big.protocol(CFG3_PROPS, q, 0, seed=SEED_P + 3)
    big.close()
    small = RefSlice(CFG4["depth"], 16_000)
    c4_1 = small.protocol(CFG4["props"], q, 1)
    small.close()
    # config 5 (1024^2, 64 props): a 10k-row slice of the same T the GPU's
    # 1M-row shard starts with, scaled to the shard (slice + scale)
    c5s = RefSlice(20, 2_000 if quick else 10_000)
    c5 = c5s.protocol(64, q, 0, seed=SEED_P)
    c5s.close()
    scale5 = 1_000_000 / c5s.rows
    scale3 = CFG4["edges"] / big.rows
    return {
        "value": c4["edge_labels_per_s_p50"], "unit": UNIT, "cores": host["hardware_concurrency"], "kind": big.kind,
        "sample": f"config 4: rows [0,{big.rows}) of the {CFG4['edges']}-edge T, 32 props, p50 over {q} queries "
                  f"(1 frame each, best of 2, 1 warm-up discarded), workers = nproc",
        "host": host, "config4": c4, "config4_workers1": c4_1,
        "config3": dict(c3, p50_ms_2M_extrapolated=c3["p50_ms"] * scale3,
                        note=f"{big.rows}-row slice; p50 x{scale3:g} for the 2M rows is extrapolated (linear in rows)"),
        "config5": dict(c5, p50_ms_1M_shard_extrapolated=c5["p50_ms"] * scale5,
                        note=f"{c5s.rows}-row slice of the 8M-edge T (1024^2, 64 props); p50 x{scale5:g} for the "
                             f"1M-row shard is extrapolated (linear in rows)"),
    }


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU label_all (oracle/_ref, all
    host threads) on the bench's workload.  One step = one query of config 4
    (one frame of 32 props) on a 500k-row slice of the 2M-edge T, best of 2
    (time_label_ms); value = p50 edge-labels/s over the K steps."""
    if rank != 0:
        return
    sl = RefSlice(CFG4["depth"], 500_000)
    for w in range(args.warmup):
        sl.query_ms(CFG4["props"], 1000 + w, 0)
    t_all = time.perf_counter()
    ts = [sl.query_ms(CFG4["props"], k, 0) for k in range(args.steps)]
    wall = time.perf_counter() - t_all
    sl.close()
    value = sl.rows / (statistics.median(ts) / 1e3)
    host = host_cpu()
    sample = (f"config 4: rows [0,{sl.rows}) of the {CFG4['edges']}-edge T, 32 props, one frame per step, best of 2 "
              f"label_all calls (time_label_ms), p50 over the steps; workers = 0 (hardware_concurrency)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / max(args.steps, 1) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": cfg_json(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": host["hardware_concurrency"], "kind": sl.kind,
                         "sample": sample, "host": host, "p50_query_ms": statistics.median(ts)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config5_shard(local: int, hbm: float, src: str, quick: bool):
    """BASELINE config 5 (8M edges, 1024^2 grid, 64 props) on one GPU's shard
    of the 8-way edge-row partition: rows [0, 1M).  Single-frame p50 latency
    (pinned host P -> labels in HBM, 150 frames after a warm-up) with the
    labelling kernel's HBM roofline, and a 64-frame batch (P resident) with
    the multi-frame kernel's binding roofline; host pack + upload time of the
    shard."""
    import torch

    from paper_1810_02612_b200 import LabelEngine
    from workload.synth import SyntheticPRM, props_words

    depth, props, E = 20, 64, 1_000_000
    cells, nw = 1 << depth, (1 << depth) // 64
    T = SyntheticPRM(seed=SEED_T, depth=depth).words(0, E)
    np64 = pairs64(T.offsets, T.words)
    eng = LabelEngine(devices=[local], profile=False)
    t0 = time.perf_counter()
    eng.load_abstraction_words(E, cells, T.offsets, T.words, T.masks)
    load_s = time.perf_counter() - t0
    info = eng.info()
    del T
    n = 30 if quick else 150
    frames = torch.empty((n + 1, props, nw), dtype=torch.int64, pin_memory=True)
    props_words(SEED_P, depth, props, 0, n + 1, out=frames)
    lat = []
    for q in range(-1, n):
        t0 = time.perf_counter()
        eng.submit_grid(cells, props, frames[q + 1], 1)
        eng.wait()
        if q >= 0:
            lat.append((time.perf_counter() - t0) * 1e3)
    eng.set_profiling(True)
    lab = []
    for q in range(-1, min(n, 50)):
        eng.submit_grid(cells, props, frames[q + 1], 1)
        eng.wait()
        if q >= 0:
            lab.append(eng.stage_times(0, 0)[2])
    k = statistics.median(lab)
    alg1 = 8 * int(info.words) + 4 * (E + 1) + cells * props // 8 + E * 8
    single = {"p50_ms": statistics.median(lat), "p99_ms": sorted(lat)[int(0.99 * (len(lat) - 1))], "frames": n,
              "what": "pinned host P (8 MB) -> labels resident in HBM (host steady clock)", "kernel_p50_ms": k,
              "roofline": {"bound": "hbm", "achieved": alg1 / (k / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                           "frac": alg1 / (k / 1e3) / 1e9 / hbm, "alg_bytes_per_launch": alg1, "peak_source": src,
                           "traffic": ncu_traffic("label_wm1_kernel<u64,2>"),
                           "limiter": ncu_limiter("label_wm1_kernel<u64,2>"),
                           "kernel": "label_wm1_kernel<u64,2> (word-major single frame)"}}
    del frames
    F = 64
    P = torch.empty((F, props, nw), dtype=torch.int64, device="cuda")
    Ph = torch.empty((F, props, nw), dtype=torch.int64, pin_memory=True)
    props_words(SEED_P, depth, props, 0, F, out=Ph)
    P.copy_(Ph)
    steps = []
    for it in range(3 + (3 if quick else 8)):
        eng.submit_grid_device(cells, props, P.data_ptr(), F)
        eng.wait()
        if it >= 3:
            st = eng.stage_times(0, 0)
            steps.append((st[1], st[2]))
    sm = statistics.median(x[0] for x in steps)
    lm = statistics.median(x[1] for x in steps)
    algF = 8 * int(info.words) + 4 * (E + 1) + F * (cells * props // 8 + E * 8)
    batch = {"frames": F, "summary_ms": sm, "label_ms": lm, "edge_labels_per_s": E * F / ((sm + lm) / 1e3),
             "roofline": {"bound": "hbm", "achieved": algF / (lm / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                          "frac": algF / (lm / 1e3) / 1e9 / hbm, "alg_bytes_per_launch": algF,
                          "kernel": "label_wm_kernel<u64,2> (word-major, two prop halves)",
                          "binding": binding_roofline("label_wm_kernel<u64,2>", lm, 1965e6, pairs=np64)}}
    eng.close()
    return {"config": "config5-dense-grid-stress, one GPU's shard of 8: rows [0, 1M) of the 8M-edge T, 1024x1024 "
                      "grid (2^20 cells), 64 props", "rows": E, "W32": int(info.words),
            "t_bytes_device": int(info.t_bytes), "load_s": load_s, "single_frame": single, "batch64": batch}


def cfg_json(world):
    return {"workload": "config4-batched-frames: 2M-edge synthetic PRM x 64 frames, 512x512 grid (2^18 cells), "
                        "32 propositions", "edges": CFG4["edges"], "grid": "512x512", "cells": 1 << CFG4["depth"],
            "props": CFG4["props"], "frames_per_step": CFG4["frames"], "parallelism": f"spatial edge-row shards x{world}" if world > 1 else "edge-row shards x1",
            "l2": "inputs larger than L2 (packed T 526 MB streamed per step)",
            "pipelining": "step k+1's summary kernel overlaps step k's labelling (async submit with P's ready event)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the config-5 shard block")
    ap.add_argument("--quick", action="store_true", help="short run for profilers")
    ap.add_argument("--dump-labels", default="", help="(tests) write a row sample of each rank's labels "
                    "after the timed steps to <prefix>_rank<r>.npz")
    ap.add_argument("--readback-chunks", type=int, default=8,
                    help="ltlg_options.readback_chunks of the e2e engine: row blocks whose label read-back "
                         "overlaps labelling (the device-resident `value` engine uses one block: globally "
                         "z-sorted rows)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    # (dev-only knobs for exercising the N > 1 path on one GPU: every rank on
    # BENCH_FORCE_DEVICE, collectives over BENCH_DIST_BACKEND=gloo -- NCCL
    # refuses two ranks on one device)
    local = int(os.environ.get("BENCH_FORCE_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1810_02612_b200 import LabelEngine
    from workload.synth import SyntheticPRM, props_words

    E, depth, props, F = CFG4["edges"], CFG4["depth"], CFG4["props"], CFG4["frames"]
    cells = 1 << depth
    nw = (cells + 63) // 64
    # N > 1: each rank holds a spatially compact, word-balanced part of the
    # edge rows (spatial_shard); N = 1: all rows in their original order
    prm = SyntheticPRM(seed=SEED_T, depth=depth)
    T = prm.words(0, E)
    row_ids, T_off, T_words, T_masks = spatial_shard(T.offsets, T.words, T.masks, rank, world)
    del T
    rows_local = len(row_ids)
    eng = LabelEngine(devices=[local], profile=True)  # device-resident labels: one block, global z-sort
    t_load = time.perf_counter()
    eng.load_abstraction_words(rows_local, cells, T_off, T_words, T_masks)
    load_s = time.perf_counter() - t_load  # host pack of every device layout + upload
    info = eng.info()
    W32_all = torch.tensor([int(info.words), rows_local], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(W32_all)
    W32, rows_all = int(W32_all[0]), int(W32_all[1])

    # P for 64 frames: pinned host (e2e) and device-resident (value)
    P_host = torch.empty((F, props, nw), dtype=torch.int64, pin_memory=True)
    if rank == 0:
        props_words(SEED_P, depth, props, 0, F, out=P_host)
    P_dev = torch.empty((F, props, nw), dtype=torch.int64, device="cuda")
    if rank == 0:
        P_dev.copy_(P_host)
    stream = torch.cuda.ExternalStream(eng.stream())
    # N > 1: P is double-buffered and the broadcast of step k+1's P runs on a
    # comm stream while step k labels (overlap the broadcast of
    # frame f+1 with the labelling of frame f, chained by events).  The
    # broadcast into a buffer waits for the labelling that last read it; the
    # labelling waits for its broadcast.  No tensor is recorded on the
    # engine's stream.
    P_bufs = [P_dev, P_dev.clone()] if world > 1 else [P_dev]
    comm = torch.cuda.Stream() if world > 1 else None
    ready = [None, None]  # broadcast into buffer b done (event on comm)
    done = [None, None]   # labelling that read buffer b done (event on the engine stream)
    nstep = [0]

    def bcast(b):
        with torch.cuda.stream(comm):
            if done[b] is not None:
                comm.wait_event(done[b])
            dist.broadcast(P_bufs[b], src=0)
            ev = torch.cuda.Event()
            ev.record(comm)
            ready[b] = ev

    if world > 1:
        bcast(0)

    # Steps are pipelined: each submit passes the event after which its P is
    # ready (ltlg_submit_grid_device_async), so step k+1's summary runs on the
    # engine's comm stream during step k's labelling.  N = 1: P is resident
    # and constant; its ready event is recorded on the engine's stream at the
    # start of the timed region, so no timed step's summary starts before it.
    p_ready = [None]

    def step():
        b = nstep[0] % len(P_bufs)
        nstep[0] += 1
        rdy = ready[b] if world > 1 else p_ready[0]
        eng.submit_grid_device(cells, props, P_bufs[b].data_ptr(), F, ready_event=rdy.cuda_event)
        if world > 1:
            ev = torch.cuda.Event()
            ev.record(stream)
            done[b] = ev
            bcast(1 - b)  # the next step's P, overlapped with this labelling

    p_ready[0] = torch.cuda.Event()
    p_ready[0].record(stream)

    for _ in range(args.warmup):
        step()
    eng.wait()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---- timed region: K steps, CUDA events on the engine's stream ----------
    K = args.steps
    kernel_ms = []
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p_ready[0] = torch.cuda.Event()
        p_ready[0].record(stream)  # (after e0: the first timed summary starts inside the region)
        for _ in range(K):
            step()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    # per-launch device times of the K timed launches (event ring on the launching stream)
    kernel_ms = [eng.stage_times(0, back)[1:] for back in range(min(K, 255))]
    if not args.no_e2e:
        # a row sample of these labels: the pipelined host-buffer (e2e) steps
        # below must reproduce it exactly
        pick_e2e = np.arange(0, rows_local, 997)
        ref_lab = eng.get_labels_packed()[pick_e2e].view(np.int32)
    if args.dump_labels:
        lab = eng.get_labels_packed()
        pick = np.nonzero(row_ids % 997 == 0)[0]  # the same row ids whatever the sharding
        np.savez(f"{args.dump_labels}_rank{rank}.npz", rows=row_ids[pick], labels=lab[pick])
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0])
    value = E * F * K / (ms_max / 1e3)
    label_ms = statistics.mean(k[1] for k in kernel_ms)
    # (the timed summaries ran on the comm stream under the previous step's
    # labelling; the kernel's own time comes from three serial submits)
    torch.cuda.synchronize()
    for _ in range(3):
        eng.submit_grid_device(cells, props, P_bufs[0].data_ptr(), F)
        eng.wait()
    summary_ms = statistics.mean(eng.stage_times(0, back)[1] for back in range(3))

    # roofline of the labeling kernel (SURVEY 8(d) algorithmic bytes, this rank's shard)
    hbm, src = peaks()
    alg_bytes = 8 * int(info.words) + 4 * (rows_local + 1) + F * (cells * props // 8 + rows_local * 4)
    achieved = alg_bytes / (label_ms / 1e3) / 1e9
    sm_clk = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": ncu_traffic("label_wm_kernel"), "peak_source": src,
                "kernel": "label_wm_kernel<u32,1> (word-major multi-frame)",
                "alg_bytes_per_launch": alg_bytes, "kernel_ms": label_ms, "summary_kernel_ms": summary_ms,
                "note": "algorithmic bytes = 8*W32 + 4*(E+1) + F*(cells*props/8 + E*4) (SURVEY 8(d)); traffic = dram "
                        "read+write bytes per launch from the committed ncu --set full capture (profiles/traffic.json). "
                        "The multi-frame kernel is not HBM-bound; `binding` is the roofline of the algorithm as it "
                        "runs: the issue slots and the L1TEX data pipe, from the committed capture's per-launch "
                        "counts over this run's kernel time",
                "binding": binding_roofline("label_wm_kernel", label_ms, sm_clk, pairs=pairs64(T_off, T_words)),
                "pairs64": pairs64(T_off, T_words)}

    # ---- p50 single-frame latency, config 3 (16 props), host P -> labels in HBM
    lat = None
    if rank == 0 and world == 1:
        P3 = torch.empty((1, CFG3_PROPS, nw), dtype=torch.int64, pin_memory=True)
        eng_lat = []
        n_frames = 30 if args.quick else 150
        frames3 = torch.empty((n_frames + 1, CFG3_PROPS, nw), dtype=torch.int64, pin_memory=True)
        props_words(SEED_P + 3, depth, CFG3_PROPS, 0, n_frames + 1, out=frames3)
        label3, stages3 = [], []
        # host latency with the stage events off (no events between the
        # kernels: the labeling kernel launches as a programmatic dependent)
        eng.set_profiling(False)
        for q in range(-1, n_frames):  # query -1 is the warm-up (scenario.cpp:183-193)
            src3 = frames3[q + 1]
            t0 = time.perf_counter()
            eng.submit_grid(cells, CFG3_PROPS, src3, 1)
            eng.wait()
            dt = time.perf_counter() - t0
            if q >= 0:
                eng_lat.append(dt * 1e3)
        # the same, with the labels read back into pinned host memory (both
        # PCIe transfers inside the time, as the paper's timings are)
        out3 = torch.empty((rows_local, 1), dtype=torch.int16, pin_memory=True)
        host_lat = []
        for q in range(-1, n_frames):
            t0 = time.perf_counter()
            eng.submit_grid(cells, CFG3_PROPS, frames3[q + 1], 1)
            eng.get_labels_packed(out3)
            if q >= 0:
                host_lat.append((time.perf_counter() - t0) * 1e3)
        # then the per-stage device times of the same frames
        eng.set_profiling(True)
        for q in range(-1, n_frames):
            eng.submit_grid(cells, CFG3_PROPS, frames3[q + 1], 1)
            eng.wait()
            if q >= 0:
                st3 = eng.stage_times(0, 0)
                label3.append(st3[2])
                stages3.append(st3)
        del P3
        k3 = statistics.median(label3)
        alg3 = 8 * int(info.words) + 4 * (rows_local + 1) + cells * CFG3_PROPS // 8 + rows_local * 2
        lat = {"config": "config3-large-abstraction: 2M edges, 512x512, 16 props, 1 frame",
               "p50_ms": statistics.median(eng_lat), "p99_ms": sorted(eng_lat)[int(0.99 * (len(eng_lat) - 1))],
               "frames": n_frames, "what": "pinned host P -> labels resident in HBM (host steady clock)",
               "kernel_p50_ms": k3,
               "p50_to_host_ms": statistics.median(host_lat),
               "to_host_what": "pinned host P -> labels (u16 per edge, 4 MB) back in pinned host memory",
               "stages_p50_ms": {"upload": statistics.median(x[0] for x in stages3),
                                 "summary": statistics.median(x[1] for x in stages3),
                                 "label": k3},
               "roofline": {"bound": "hbm", "achieved": alg3 / (k3 / 1e3) / 1e9, "peak": hbm,
                                                "unit": "GB/s", "frac": alg3 / (k3 / 1e3) / 1e9 / hbm,
                                                "alg_bytes_per_launch": alg3,
                                                "traffic": ncu_traffic("label_stream64_kernel"),
                                                "limiter": ncu_limiter("label_stream64_kernel"),
                                                "kernel": "label_stream64_kernel<16,u16,smem,1024>"}}

    # ---- e2e through the public API with host buffers ------------------------
    e2e = None
    if not args.no_e2e:
        # host-buffer path: engines whose rows are z-sorted within read-back
        # blocks, so the 512 MB label copy overlaps the labelling of later
        # blocks.  Two engines alternate steps (double buffering, as a
        # streaming caller would): step k+1's P upload and labelling are
        # submitted before step k's labels are read back, so the H2D and D2H
        # directions of PCIe run at the same time.  Every step's P still
        # crosses H2D and its labels D2H inside the timed region.
        eng.close()
        engs = []
        for _ in range(2):
            e = LabelEngine(devices=[local], readback_chunks=args.readback_chunks)
            e.load_abstraction_words(rows_local, cells, T_off, T_words, T_masks)
            engs.append(e)
        eng = engs[0]
        streams = [torch.cuda.ExternalStream(e.stream()) for e in engs]
        outs = [torch.empty((rows_local, F), dtype=torch.int32, pin_memory=True) for _ in engs]
        Pd = [P_dev, torch.empty_like(P_dev)] if world > 1 else None
        Ke = max(2, K)  # as many steps as the device-timed `value`

        def e2e_submit(k):
            e, st = engs[k % 2], streams[k % 2]
            if world > 1:  # H2D on rank 0 + broadcast on torch's stream, then the engine's
                cur = torch.cuda.current_stream()
                cur.wait_stream(st)  # the buffer's previous reader (step k-2) is done
                if rank == 0:
                    Pd[k % 2].copy_(P_host, non_blocking=True)
                dist.broadcast(Pd[k % 2], src=0)
                st.wait_stream(cur)
                e.submit_grid_device(cells, props, Pd[k % 2].data_ptr(), F, readback=True)
            else:
                e.submit_grid(cells, props, P_host, F)

        def e2e_run(n):
            e2e_submit(0)
            for k in range(n):
                if k + 1 < n:
                    e2e_submit(k + 1)
                engs[k % 2].get_labels_packed(outs[k % 2])

        e2e_run(2)  # untimed warm-up of the host path (both engines)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_run(Ke)
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt[0])
        for i, o in enumerate(outs):
            got = o.numpy()[pick_e2e]
            if not np.array_equal(got, ref_lab):
                bad = np.nonzero((got != ref_lab).any(axis=1))[0]
                raise RuntimeError(f"e2e: labels read back to host differ from the device-resident run (rank {rank}, "
                                   f"engine {i}: {len(bad)} of {len(pick_e2e)} sampled rows, first {bad[:5].tolist()}; "
                                   f"engines agree: {np.array_equal(outs[0].numpy(), outs[1].numpy())})")
        for e in engs[1:]:
            e.close()
        e2e = {"value": E * F * Ke / dt, "unit": UNIT, "h2d_bytes_per_step": F * props * nw * 8,
               "d2h_bytes_per_step": E * F * 4, "steps": Ke,
               "what": "ltlg_submit_grid(pinned host P, 64 frames) + ltlg_get_labels_packed(pinned host, u32 x 64 "
                       "frames per edge); host wall clock; readback_chunks=%d (block c's labels copy back while "
                       "later blocks are labelled); two engines alternate steps, so step k+1's upload and "
                       "labelling overlap step k's read-back" % args.readback_chunks}

    cfg5 = None
    if rank == 0 and world == 1 and not args.no_cfg5:
        eng.close()  # (the e2e engines and this one are done: free HBM for the config-5 shard)
        eng = None
        cfg5 = config5_shard(local, hbm, src, args.quick)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.quick)
        if lat is not None:  # the reference's config-3 p50 beside ours
            lat["cpu_reference_p50_ms"] = cpu["config3"]["p50_ms_2M_extrapolated"]
            lat["cpu_reference_what"] = cpu["config3"]["note"] + f"; {cpu['cores']} threads"
        if cfg5 is not None and cfg5.get("single_frame"):  # and its config-5 shard p50 beside ours
            cfg5["single_frame"]["cpu_reference_p50_ms"] = cpu["config5"]["p50_ms_1M_shard_extrapolated"]
            cfg5["single_frame"]["cpu_reference_what"] = cpu["config5"]["note"] + f"; {cpu['cores']} threads"

    if rank == 0:
        # gpu_launches: our kernels per step = wm_build (the word-major summary) and label_wm
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic", "config": cfg_json(world), "clocks": clk.summary(),
            "gpu_launches": 2 * K, "roofline": roofline, "latency": lat, "e2e": e2e, "cpu_baseline": cpu,
            "config5_shard": cfg5,
            "shape": {"W32": W32, "rows": rows_all, "t_bytes_device": int(info.t_bytes), "load_s": load_s},
        }
        print(json.dumps(line), flush=True)
    # tear the process group down before the engine (and its stream) goes away
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if eng is not None:
        eng.close()


if __name__ == "__main__":
    main()
