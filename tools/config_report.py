#!/usr/bin/env python
"""Per-configuration report for BASELINE.md §4: for each BASELINE.json config,
GPU apply time (median/min of --reps after a warm-up, CUDA events), pairs/s,
FP64-pipe fraction, self-term HBM GB/s, parity vs the CPU oracle on the seeded
subset (rel-L2, max-norm), and the oracle's own pair rate on the host cores.
Run on the GPU box:  python tools/config_report.py --configs 1 2 3 4 5
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OPS = 30
OPS_OFF = 32
LANES = 148 * 64 * 1.965e9


def err(got, ref):
    return (float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
            float(np.abs(got - ref).max() / np.abs(ref).max()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import oracle
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config, rigid_field

    for cfg in args.configs:
        d = make_config(cfg)
        p, mu = d["p"], d["mu"]
        nsn = (p + 1) * (2 * p + 2)
        N = d["n_nodes"]
        f, q = d["f"], d["q"]
        if d["rigid"] is not None:
            x, _, _ = oracle.nodes(d["centres"], d["radii"], p)
            q = rigid_field(*d["rigid"], x, d["centres"], nsn)
        if d["same_fq"]:
            f = q
        ctx = bie.bie_create(d["centres"], d["radii"], p, mu)
        F = torch.from_numpy(np.ascontiguousarray(f)).cuda()
        Q = torch.from_numpy(np.ascontiguousarray(q)).cuda()
        U = torch.empty_like(F)
        bie.bie_apply_SLDL(ctx, F, Q, U)
        torch.cuda.synchronize()
        bie.bie_reset_profile(ctx)
        bie.bie_set_profiling(ctx, True)
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bie.bie_apply_SLDL(ctx, F, Q, U)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        prof = bie.bie_get_profile(ctx)
        bie.bie_set_profiling(ctx, False)
        pairs = N * (N - nsn)
        med = float(np.median(ts))
        nb_ms = prof["nbody"][0] / args.reps if prof["nbody"][1] else float("nan")
        self_ms = prof["self"][0] / args.reps
        u = U.cpu().numpy()
        sub = d["subset"] if d["subset"] is not None else np.arange(N)
        t0 = time.perf_counter()
        far = oracle.far(d["centres"], d["radii"], p, mu, f, q, sub)
        t_far = time.perf_counter() - t0
        t0 = time.perf_counter()
        slf = oracle.self_term(d["centres"], d["radii"], p, mu, f, q, sub)
        t_self = time.perf_counter() - t0
        rel, mx = err(u[sub], far + slf)
        rec = {"config": cfg, "n_spheres": int(len(d["radii"])), "p": p, "n_nodes": int(N),
               "pairs": int(pairs), "apply_ms_median": med, "apply_ms_min": float(min(ts)),
               "pairs_per_s": pairs / (med / 1e3), "nbody_ms": nb_ms,
               "nbody_fp64_pipe_frac": pairs * OPS / (nb_ms / 1e3) / LANES if nb_ms == nb_ms else None,
               "self_ms": self_ms, "self_hbm_GBps": 168.0 * N / (self_ms / 1e3) / 1e9,
               "self_hbm_frac_of_6451": 168.0 * N / (self_ms / 1e3) / 6451.5e9,
               "parity_targets": int(len(sub)), "rel_l2": rel, "max_norm": mx,
               "oracle_far_pairs_per_s": len(sub) * (N - nsn) / t_far, "oracle_self_s": t_self,
               "oracle_cores": oracle.num_threads(), "kernels": prof}
        if d["targets"] is not None:
            tg = torch.from_numpy(d["targets"]).cuda()
            M = tg.shape[0]
            UO = torch.empty((M, 3), dtype=torch.float64, device="cuda")
            PO = torch.empty(M, dtype=torch.float64, device="cuda")
            bie.bie_eval_offsurface(ctx, F, Q, tg, UO, PO)
            torch.cuda.synchronize()
            to = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                bie.bie_eval_offsurface(ctx, F, Q, tg, UO, PO)
                e1.record()
                e1.synchronize()
                to.append(e0.elapsed_time(e1))
            ts_ = d["target_subset"]
            t0 = time.perf_counter()
            uref, pref = oracle.offsurface(d["centres"], d["radii"], p, mu, f, q, d["targets"][ts_])
            t_off = time.perf_counter() - t0
            ru, mu_ = err(UO.cpu().numpy()[ts_], uref)
            rp, mp = err(PO.cpu().numpy()[ts_], pref)
            om = float(np.median(to))
            rec["offsurface"] = {"targets": int(M), "pairs": int(M * N), "ms_median": om,
                                 "pairs_per_s": M * N / (om / 1e3),
                                 "fp64_pipe_frac_upper": M * N * OPS_OFF / (om / 1e3) / LANES,
                                 "parity_targets": int(len(ts_)), "u_rel_l2": ru, "u_max_norm": mu_,
                                 "p_rel_l2": rp, "p_max_norm": mp,
                                 "oracle_pairs_per_s": len(ts_) * N / t_off}
        ctx.close()
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
