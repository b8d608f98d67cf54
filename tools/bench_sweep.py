"""Swept-volume build on the GPU vs the reference CPU.

  python tools/bench_sweep.py [--edges 200000] [--depth 18] [--reps 5]

Trajectories: the reference's own build_abstraction (Rect region, the
AbstractionConfig defaults: 72 m x 72 m, 8-14 m/s, tau_limit 7.2 s) through
oracle/_ref; grid: default_bench_grid (scenario.cpp:20-22, 72 x 72 m x 7.2 s).
GPU: ltlg_swept_volume kernel time (CUDA events, both passes) and end to end
(host trajectories in -> host CSR out).  CPU: the reference
swept_volume_matrix with all host threads.  The two CSRs must be identical.
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FOOTPRINT = (4.6, 2.0, -1.4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=200_000)
    ap.add_argument("--depth", type=int, default=18)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-reps", type=int, default=1)
    a = ap.parse_args()
    from oracle.oracle import RefCore
    from paper_1810_02612_b200 import FootprintSpec, swept_volume

    ref = RefCore()
    t = time.perf_counter()
    off, smp = ref.abstraction(x=(0.0, 72.0), y=(0.0, 72.0), speed=(8.0, 14.0), tau=(0.0, 0.0), tau_limit=7.2,
                               target_edges=a.edges, seed=1)
    gen_s = time.perf_counter() - t
    bounds = ((0.0, 72.0), (0.0, 72.0), (0.0, 7.2))
    lo, hi = [b[0] for b in bounds], [b[1] for b in bounds]
    fp = FootprintSpec(*FOOTPRINT)
    sv = swept_volume((off, smp), fp, bounds, a.depth)  # warm-up
    gpu = sv.to_csr()
    sv.close()
    kern, e2e = [], []
    for _ in range(a.reps):
        t = time.perf_counter()
        sv = swept_volume((off, smp), fp, bounds, a.depth)
        m = sv.to_csr()
        e2e.append(time.perf_counter() - t)
        kern.append(sv.build_ms / 1e3)
        sv.close()
    cpu = []
    for _ in range(a.cpu_reps):
        t = time.perf_counter()
        rows, cols = ref.swept_volume(a.depth, lo, hi, FOOTPRINT, off, smp, workers=0)
        cpu.append(time.perf_counter() - t)
    same = bool(np.array_equal(rows, gpu.row_offsets) and np.array_equal(cols, gpu.col_indices)
                and np.array_equal(m.col_indices, gpu.col_indices))
    E = off.size - 1
    out = {
        "metric": "swept-volume rows/s (swept_volume_matrix)", "edges": int(E), "samples": int(smp.shape[0]),
        "nnz": int(gpu.nnz()), "depth": a.depth, "grid": "72 x 72 m x 7.2 s (default_bench_grid)",
        "gpu_kernel_ms_p50": float(np.median(kern) * 1e3), "gpu_e2e_ms_p50": float(np.median(e2e) * 1e3),
        "gpu_rows_per_s": E / float(np.median(kern)), "gpu_e2e_rows_per_s": E / float(np.median(e2e)),
        "cpu_ms": float(min(cpu) * 1e3), "cpu_rows_per_s": E / min(cpu), "cpu_threads": os.cpu_count(),
        "identical": same, "trajectory_gen_s": gen_s,
    }
    print(json.dumps(out))
    if not same:
        sys.exit(1)


if __name__ == "__main__":
    main()
