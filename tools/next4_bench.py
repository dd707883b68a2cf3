#!/usr/bin/env python
"""NEXT-4 crossover study (PAPER §4.2, Fig 3's experiment on B200): time and
node accuracy of the rotated, pole-aligned near evaluation (bie_set_near_mode
1) against the direct evaluation (mode 0, NEXT-1) for p in {8, 12, 16, 24, 32}.

Workload: an 8x8x8 lattice of unit spheres at spacing 2.6 (gap 0.6), eta = 0.5,
so each sphere's 6 face neighbours are near (eq 4.5) and nothing else; f, q
iid N(0,1).  Per p it reports, from the library's own CUDA events
(bie_get_profile) over `reps` applies:
  exact_direct_ms   exterior field evaluated at the target nodes (mode 2, k_near
                    exterior part only)
  exact_next4_ms    rotate -> pole-aligned discs -> re-expand -> rotate back
                    (mode 3, k_n4)
  near_direct_ms    the whole direct correction (mode 0: k_near_coef + k_near)
  near_next4_ms     the whole NEXT-4 correction (mode 1: k_near_coef + k_n4 +
                    smooth-only k_near + the extra self-term pass)
  err_rel_u         max |u_mode1 - u_mode0| / max |u_mode0| at the nodes (and _smooth)
  acc_vs_direct     max |u_mode1 - u_mode0| / max |u_mode0 - u_eta0| at the nodes:
                    NEXT-4's truncation relative to the size of the near correction,
                    for white-noise densities (BASELINE's inputs) and, as
                    acc_vs_direct_smooth, for smooth (degree <= 2) densities
Usage: python tools/next4_bench.py [--p 8 12 ...] [--reps 5]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, nargs="*", default=[8, 12, 16, 24, 32])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--spacing", type=float, default=2.6)
    ap.add_argument("--eta", type=float, default=0.5)
    args = ap.parse_args()
    import torch
    import paper_1707_06551_b200 as bie
    g = np.arange(args.k) * args.spacing
    c = np.array([[x, y, z] for x in g for y in g for z in g])
    a = np.ones(len(c))
    for p in args.p:
        nsn = (p + 1) * (2 * p + 2)
        N = len(c) * nsn
        rng = np.random.default_rng(p)
        F = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        ctx = bie.bie_create(c, a, p, 1.0)
        # smooth densities (degree <= 2 polynomials of the position on each sphere),
        # the paper's setting (decaying spectra), for the accuracy column
        xg = torch.empty((N, 3), dtype=torch.float64, device="cuda")
        bie.bie_get_nodes(ctx, xg)
        xs = xg.cpu().numpy() - np.repeat(c, nsn, 0)
        Fs = torch.from_numpy(np.stack([xs[:, 1] * xs[:, 2], xs[:, 0] ** 2 - 0.3, xs[:, 1]], 1)).cuda()
        Qs = torch.from_numpy(np.stack([xs[:, 2], xs[:, 0] * xs[:, 1], 1.0 - xs[:, 2] ** 2], 1)).cuda()
        us = {}
        u = {}
        times = {}
        for mode in (None, 0, 2, 1, 3):
            bie.bie_set_near(ctx, 0.0 if mode is None else args.eta)
            if mode is not None:
                bie.bie_set_near_mode(ctx, mode)
            out = torch.empty((N, 3), dtype=torch.float64, device="cuda")
            bie.bie_apply_SLDL(ctx, F, Q, out)  # warm-up
            torch.cuda.synchronize()
            bie.bie_reset_profile(ctx)
            bie.bie_set_profiling(ctx, True)
            for _ in range(args.reps):
                bie.bie_apply_SLDL(ctx, F, Q, out)
            prof = bie.bie_get_profile(ctx)
            bie.bie_set_profiling(ctx, False)
            times[mode] = {k: v[0] / args.reps for k, v in prof.items() if v[1]}
            u[mode] = out.cpu().numpy()
            if mode in (None, 0, 1):
                bie.bie_apply_SLDL(ctx, Fs, Qs, out)
                torch.cuda.synchronize()
                us[mode] = out.cpu().numpy()
        npairs = bie.bie_near_pairs(ctx)
        ctx.close()
        dn = np.abs(u[0] - u[None]).max()
        rec = {"p": p, "n_spheres": len(c), "near_pairs": int(npairs), "n_nodes": N,
               "exact_direct_ms": times[2].get("near", 0.0),
               "exact_next4_ms": times[3].get("near4", 0.0) + times[3].get("near", 0.0),
               "near_direct_ms": times[0].get("near", 0.0),
               "near_next4_ms": times[1].get("near", 0.0) + times[1].get("near4", 0.0)
                                + times[1].get("self", 0.0) - times[0].get("self", 0.0),
               "k_n4_ms": times[1].get("near4", 0.0),
               "acc_vs_direct": float(np.abs(u[1] - u[0]).max() / dn),
               "near_correction_rel": float(dn / np.abs(u[0]).max()),
               "acc_vs_direct_smooth": float(np.abs(us[1] - us[0]).max() / np.abs(us[0] - us[None]).max()),
               "err_rel_u": float(np.abs(u[1] - u[0]).max() / np.abs(u[0]).max()),
               "err_rel_u_smooth": float(np.abs(us[1] - us[0]).max() / np.abs(us[0]).max()),
               "near_correction_rel_smooth": float(np.abs(us[0] - us[None]).max() / np.abs(us[0]).max()),
               "ms_by_kind": {str(k): v for k, v in times.items()}}
        rec["speedup_exact"] = rec["exact_direct_ms"] / max(rec["exact_next4_ms"], 1e-9)
        rec["speedup_total"] = rec["near_direct_ms"] / max(rec["near_next4_ms"], 1e-9)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
