#!/usr/bin/env python
"""Time the self-term kernel alone (bie_apply_parts(SELF): pack + VSHT + scale +
inverse) for BASELINE configs; report ms and achieved HBM GB/s at the
algorithmic 168 B/node (f, q in; u, packed records out)."""
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
    cfgs = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]
    for cfg in cfgs:
        d = make_config(cfg, with_targets=False)
        ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
        N = d["n_nodes"]
        g = np.random.default_rng(0)
        F = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        U = torch.empty_like(F)
        for _ in range(3):
            bie.bie_apply_parts(ctx, F, Q, U, bie.BIE_PART_SELF)
        torch.cuda.synchronize()
        bie.bie_reset_profile(ctx)
        bie.bie_set_profiling(ctx, True)
        reps = 20
        for _ in range(reps):
            bie.bie_apply_parts(ctx, F, Q, U, bie.BIE_PART_SELF)
        prof = bie.bie_get_profile(ctx)
        ms = prof["self"][0] / reps
        print(json.dumps({"config": cfg, "p": d["p"], "n_nodes": N, "self_ms": ms,
                          "GBps": 168.0 * N / (ms / 1e3) / 1e9,
                          "frac_of_6451": 168.0 * N / (ms / 1e3) / 6451.5e9}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
