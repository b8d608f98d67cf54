"""The paper's own experiment (arXiv 1810.02612, Table "Transition system size
and labeling function construction times") on one B200.

  python tools/paper_table.py [--queries 150] [--cpu-queries 3] [--sizes ...]

Per system size (the paper's five transition counts):
  * the roadmap is the reference benchmark's own (loop_abstraction_config +
    build_abstraction, seed 1, through oracle/_ref) on default_bench_grid at
    depth 21 (2^21 cells, as in the paper);
  * T = swept_volume_matrix built on the GPU (ltlg_swept_volume), loaded into
    the engine (identical to the reference's CSR: checked at the smallest size);
  * per query (one warm-up + --queries), the two propositions of
    generate_scenario (moving_vehicle, not_nominal_lane), each labelled
    separately like the paper: pinned host P -> labels back in pinned host
    memory, so the time includes both PCIe transfers, as the paper's does;
  * the reference CPU label_all on the same T and P (all host threads, best
    of 2 per query, time_label_ms) for --cpu-queries queries.
Prints one JSON line per size and a markdown table.
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PAPER = {154776: (3.67, 2.01), 295700: (6.60, 3.25), 568958: (12.77, 5.95), 836276: (18.46, 8.40),
         1097702: (24.40, 11.02)}  # GTX 1080 ms (moving_vehicle, not_nominal_lane)
DEPTH = 21
BOUNDS = ((0.0, 72.0), (0.0, 72.0), (0.0, 7.2))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--queries", type=int, default=150)
    ap.add_argument("--cpu-queries", type=int, default=3)
    ap.add_argument("--sizes", type=int, nargs="*", default=sorted(PAPER))
    a = ap.parse_args()
    import torch

    from oracle.oracle import RefCore
    from paper_1810_02612_b200 import FootprintSpec, LabelEngine, ScenarioConfig, generate_scenario, swept_volume

    ref = RefCore()
    cells = 1 << DEPTH
    nw = cells // 64
    cfg = ScenarioConfig()
    # P of every query (GPU generate_scenario, bit-exact with the reference's)
    nq = a.queries + 1
    P = torch.empty((nq, 2, nw), dtype=torch.int64, pin_memory=True)
    for q in range(nq):
        mv, nn = generate_scenario(cfg, BOUNDS, DEPTH, q)
        P[q, 0] = torch.from_numpy(mv.words.view(np.int64))
        P[q, 1] = torch.from_numpy(nn.words.view(np.int64))
    occ = [float(np.unpackbits(P[:, j].numpy().view(np.uint8)).mean()) for j in range(2)]
    rows_out = []
    for target in a.sizes:
        t0 = time.perf_counter()
        off, smp = ref.loop_abstraction(DEPTH, target, 1)
        gen_s = time.perf_counter() - t0
        E = off.size - 1
        sv = swept_volume((off, smp), FootprintSpec(), BOUNDS, DEPTH)
        sweep_ms = sv.build_ms
        csr = sv.to_csr()
        if target == min(a.sizes):  # the GPU T is the reference's T
            rr, rc = ref.swept_volume(DEPTH, [b[0] for b in BOUNDS], [b[1] for b in BOUNDS],
                                      (4.6, 2.0, -1.4), off, smp)
            assert np.array_equal(rr, csr.row_offsets) and np.array_equal(rc, csr.col_indices)
        eng = LabelEngine(devices=[0])
        eng.load_swept_volume(sv)
        sv.close()
        out = torch.empty((E, 1), dtype=torch.uint8, pin_memory=True)
        res = {}
        for j, name in enumerate(("moving_vehicle", "not_nominal_lane")):
            ts = []
            for q in range(nq):  # query 0 is the warm-up (scenario.cpp:183-193)
                src = P[q, j]
                t = time.perf_counter()
                eng.submit_grid(cells, 1, src, 1)
                eng.get_labels_packed(out)
                dt = (time.perf_counter() - t) * 1e3
                if q:
                    ts.append(dt)
            res[name] = {"mean_ms": statistics.mean(ts), "p50_ms": statistics.median(ts),
                         "var_ms": statistics.pvariance(ts)}
        eng.close()
        cpu = {}
        if a.cpu_queries:
            m = ref.csr_handle(E, cells, csr.row_offsets, csr.col_indices)
            for j, name in enumerate(("moving_vehicle", "not_nominal_lane")):
                ts = []
                for q in range(1, a.cpu_queries + 1):
                    p = ref.props_handle(cells, 1, P[q, j].numpy().view(np.uint64))
                    ts.append(ref.time_label_ms(m, p, 0, 2))
                    ref.free(p=p)
                cpu[name] = statistics.mean(ts)
            ref.free(m=m)
        paper = PAPER.get(target)
        line = {"transitions": E, "cells": cells, "row_occupancy_pct": 100.0 * csr.nnz() / E / cells,
                "moving_vehicle_occupancy_pct": 100 * occ[0], "not_nominal_lane_occupancy_pct": 100 * occ[1],
                "gpu_ms": res, "cpu_reference_ms": cpu, "cpu_threads": os.cpu_count(),
                "paper_gtx1080_ms": {"moving_vehicle": paper[0], "not_nominal_lane": paper[1]} if paper else None,
                "swept_volume_gpu_ms": sweep_ms, "roadmap_build_s": gen_s, "queries": a.queries}
        print(json.dumps(line), flush=True)
        rows_out.append(line)
    print("\n| transitions | B200 moving_vehicle (ms) | B200 not_nominal_lane (ms) | GTX 1080 (paper) mv / nnl | "
          "reference CPU mv / nnl (ms) |")
    print("|---|---|---|---|---|")
    for r in rows_out:
        g = r["gpu_ms"]
        p = r["paper_gtx1080_ms"]
        c = r["cpu_reference_ms"]
        print(f"| {r['transitions']:,} | {g['moving_vehicle']['mean_ms']:.3f} | {g['not_nominal_lane']['mean_ms']:.3f} | "
              f"{p['moving_vehicle'] if p else '-'} / {p['not_nominal_lane'] if p else '-'} | "
              f"{c.get('moving_vehicle', float('nan')):.1f} / {c.get('not_nominal_lane', float('nan')):.1f} |")


if __name__ == "__main__":
    main()
