#!/usr/bin/env python
"""Throughput of the traction operator apply (bie_apply_K) on BASELINE configs."""
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
    for cfg in [int(a) for a in sys.argv[1:]] or [3, 4, 5]:
        d = make_config(cfg, with_targets=False)
        p = d["p"]
        nsn = (p + 1) * (2 * p + 2)
        N = d["n_nodes"]
        ctx = bie.bie_create(d["centres"], d["radii"], p, d["mu"])
        S = torch.from_numpy(np.random.default_rng(0).standard_normal((N, 3))).cuda()
        U = torch.empty_like(S)
        bie.bie_apply_K(ctx, S, U)
        torch.cuda.synchronize()
        reps = 3 if cfg in (4, 5) else 5
        bie.bie_reset_profile(ctx)
        bie.bie_set_profiling(ctx, True)
        for _ in range(reps):
            bie.bie_apply_K(ctx, S, U)
        prof = bie.bie_get_profile(ctx)
        ms = prof["kfar"][0] / reps
        pairs = N * (N - nsn)
        rec = {"config": cfg, "pairs": pairs, "kfar_ms": ms, "pairs_per_s": pairs / (ms / 1e3),
               "fp64_pipe_frac": pairs / (ms / 1e3) * 25 / (148 * 64 * 1.965e9),
               "apply_K_ms": sum(v[0] for v in prof.values()) / reps}
        # near-singular correction (eta = 1) and the completion operator L (eq 5.8)
        bie.bie_set_near(ctx, 1.0)
        bie.bie_apply_K(ctx, S, U, 7)
        torch.cuda.synchronize()
        bie.bie_reset_profile(ctx)
        for _ in range(reps):
            bie.bie_apply_K(ctx, S, U, 7)
        prof = bie.bie_get_profile(ctx)
        rec.update({"near_pairs_eta1": bie.bie_near_pairs(ctx), "near_K_ms": prof["near"][0] / reps,
                    "completion_ms": prof["complete"][0] / reps,
                    "apply_K_near_L_ms": sum(v[0] for v in prof.values()) / reps})
        print(json.dumps(rec), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
