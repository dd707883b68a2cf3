#!/usr/bin/env python
"""Cost of the off-surface near correction on cfg 5 (1e6 targets, eta = 0.5, 1)
per schedule (bie_set_near_off_schedule: 0 grouped by sphere, 1 per target).
Usage: python tools/near_off_bench.py [--scheds 0,1] [--etas 0,0.5,1]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scheds", default="0,1")
    ap.add_argument("--etas", default="0,0.5,1")
    args = ap.parse_args()
    import torch
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config
    d = make_config(5)
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    N = d["n_nodes"]
    g = np.random.default_rng(0)
    F = torch.from_numpy(g.standard_normal((N, 3))).cuda()
    Q = torch.from_numpy(g.standard_normal((N, 3))).cuda()
    tg = torch.from_numpy(d["targets"]).cuda()
    M = tg.shape[0]
    u = torch.empty((M, 3), dtype=torch.float64, device="cuda")
    pr = torch.empty(M, dtype=torch.float64, device="cuda")
    for eta in [float(x) for x in args.etas.split(",")]:
        bie.bie_set_near(ctx, eta)
        for sched in [int(x) for x in args.scheds.split(",")]:
            if eta == 0.0 and sched:
                continue
            bie.bie_set_near_off_schedule(ctx, sched)
            bie.bie_eval_offsurface(ctx, F, Q, tg, u, pr)
            torch.cuda.synchronize()
            bie.bie_reset_profile(ctx)
            bie.bie_set_profiling(ctx, True)
            bie.bie_eval_offsurface(ctx, F, Q, tg, u, pr)
            prof = bie.bie_get_profile(ctx)
            bie.bie_set_profiling(ctx, False)
            print(json.dumps({"config": 5, "eta": eta, "schedule": sched, "near_ms": prof["near"][0],
                              "near_launches": prof["near"][1], "n_near_pairs_spheres": bie.bie_near_pairs(ctx),
                              "offsurface_ms": prof["offsurface"][0],
                              "total_ms": sum(v[0] for v in prof.values())}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
