#!/usr/bin/env python
"""GMRES solve of BIE 5.4 (bie_solve_porous) on BASELINE geometries in a
uniform imposed flow, with the near correction (eta = 1): iterations, true
residual, wall time, and the share of the Krylov vector kernels."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config
    for cfg in [int(a) for a in sys.argv[1:]] or [2, 3]:
        d = make_config(cfg, with_targets=False)
        ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
        bie.bie_set_near(ctx, 1.0)
        N = d["n_nodes"]
        uinf = torch.zeros((N, 3), dtype=torch.float64, device="cuda")
        uinf[:, 2] = 1.0
        mu = torch.empty_like(uinf)
        bie.bie_reset_profile(ctx)
        bie.bie_set_profiling(ctx, True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pc = os.environ.get("PRECOND", "1") == "1"
        restart = int(os.environ.get("RESTART", "50"))
        max_iter = int(os.environ.get("MAX_ITER", "200"))
        it, res = bie.bie_solve_porous(ctx, uinf, mu, tol=1e-10, max_iter=max_iter, restart=restart,
                                       precond=pc)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        prof = bie.bie_get_profile(ctx)
        dev_ms = sum(v[0] for v in prof.values())
        print(json.dumps({"config": cfg, "precond": pc, "restart": restart, "max_iter": max_iter,
                          "n_nodes": N, "iterations": it, "rel_resid": res,
                          "wall_s": wall, "device_ms": dev_ms,
                          "krylov_ms": prof["krylov"][0], "nbody_ms": prof["nbody"][0],
                          "near_ms": prof["near"][0], "self_ms": prof["self"][0],
                          "ms_per_iteration": 1e3 * wall / max(it, 1)}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
