#!/usr/bin/env python
"""Time the self-term kernel alone (bie_apply_parts(SELF): pack + VSHT + scale +
inverse, rows a2 + a4-a6) per kernel variant (bie_set_self_kernel: 0 batched
DMMA, 1 batched DFMA, 2 round-1 per-sphere) on BASELINE configs; L2 flushed
(256 MB write) before every timed call, CUDA events on the launching stream.
Reports ms and achieved HBM GB/s at the algorithmic 168 B/node (f, q in: 48;
u: 24 and packed records: 96 out) against MEASURED_PEAKS.json's hbm_gbs.
Usage: python tools/self_bench.py [cfg ...] [--variants 0,1,2] [--p P --ns NS]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="*", type=int, default=[3, 4, 5])
    ap.add_argument("--variants", default="0,1,2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--p", type=int, action="append", default=[], help="extra synthetic order")
    ap.add_argument("--ns", type=int, default=4096)
    args = ap.parse_args()
    import torch
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    cases = []
    for cfg in args.cfgs:
        d = make_config(cfg, with_targets=False)
        cases.append((f"cfg{cfg}", d["centres"], d["radii"], d["p"], d["mu"]))
    for p in args.p:  # lattice of unit spheres, spacing 3
        k = int(round(args.ns ** (1 / 3))) + 1
        c = np.array([[3.0 * i, 3.0 * j, 3.0 * l] for i in range(k) for j in range(k) for l in range(k)])[: args.ns]
        cases.append((f"lattice{len(c)}_p{p}", c, np.ones(len(c)), p, 1.0))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for name, cen, rad, p, mu in cases:
        ctx = bie.bie_create(cen, rad, p, mu)
        N = bie.bie_num_nodes(ctx)
        g = np.random.default_rng(0)
        F = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        U = torch.empty_like(F)
        ref = None
        for v in [int(x) for x in args.variants.split(",")]:
            bie.bie_set_self_kernel(ctx, v)
            for _ in range(3):
                bie.bie_apply_parts(ctx, F, Q, U, bie.BIE_PART_SELF)
            torch.cuda.synchronize()
            out = U.clone()
            if ref is None:
                ref = out
            diff = float((out - ref).norm() / ref.norm())
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                bie.bie_apply_parts(ctx, F, Q, U, bie.BIE_PART_SELF)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            print(json.dumps({"case": name, "p": p, "n_spheres": len(rad), "n_nodes": N, "variant": v,
                              "self_ms_median": round(ms, 5), "self_ms_min": round(min(ts), 5),
                              "GBps": round(168.0 * N / (ms / 1e3) / 1e9, 1),
                              "hbm_frac_of_measured": round(168.0 * N / (ms / 1e3) / 1e9 / hbm, 4),
                              "rel_diff_vs_first_variant": diff}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
