#!/usr/bin/env python
"""Cost of the near-singular correction (bie_set_near) on BASELINE configs:
k_near device time per apply, number of near (target, source) sphere pairs,
and the apply time with and without the correction."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config
    eta = float(os.environ.get("ETA", "1.0"))
    for cfg in [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]:
        d = make_config(cfg, with_targets=False)
        p = d["p"]
        nsn = (p + 1) * (2 * p + 2)
        nlm = (p + 1) * (p + 2) // 2
        ctx = bie.bie_create(d["centres"], d["radii"], p, d["mu"])
        bie.bie_set_near(ctx, eta)
        npairs = bie.bie_near_pairs(ctx)
        N = d["n_nodes"]
        g = np.random.default_rng(0)
        F = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        U = torch.empty_like(F)
        reps = 3 if cfg in (4, 5) else 10
        bie.bie_apply_SLDL(ctx, F, Q, U)
        torch.cuda.synchronize()
        bie.bie_reset_profile(ctx)
        bie.bie_set_profiling(ctx, True)
        for _ in range(reps):
            bie.bie_apply_SLDL(ctx, F, Q, U)
        prof = bie.bie_get_profile(ctx)
        near_ms = prof["near"][0] / reps
        # FP64 work per (target node, near source sphere): exterior expansion
        # ~ 40 flops per (n, m) (round 2: the smooth rule of near pairs is
        # excluded inside the far-field kernel, nothing is subtracted)
        flops = npairs * nsn * (40.0 * nlm)
        print(json.dumps({"config": cfg, "eta": eta, "p": p, "near_pairs": npairs,
                          "near_ms": near_ms, "apply_ms": sum(v[0] for v in prof.values()) / reps,
                          "nbody_ms": prof["nbody"][0] / reps,
                          "near_share": near_ms / (sum(v[0] for v in prof.values()) / reps),
                          "near_tflops_est": flops / (near_ms / 1e3) / 1e12 if near_ms else None}),
              flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
