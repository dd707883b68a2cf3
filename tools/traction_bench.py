#!/usr/bin/env python
"""Off-surface traction evaluator (bie_eval_traction, NEXT-3) on the BASELINE
configs' off-surface targets (or 1e6 random ones) with random unit normals:
far-field pairs/s and the near-correction cost at eta = 1."""
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
    for cfg in [int(a) for a in sys.argv[1:]] or [3, 5]:
        d = make_config(cfg, with_targets=True)
        N = d["n_nodes"]
        g = np.random.default_rng(0)
        if d.get("targets") is not None:
            tg = np.ascontiguousarray(d["targets"][:1000000])
        else:  # uniform in the suspension's bounding box (throughput only)
            lo, hi = d["centres"].min(0) - 2.0, d["centres"].max(0) + 2.0
            tg = lo + (hi - lo) * g.uniform(size=(1000000, 3))
        M = len(tg)
        nv = g.standard_normal((M, 3))
        nv /= np.linalg.norm(nv, axis=1)[:, None]
        ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
        S = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        T = torch.from_numpy(tg).cuda()
        NV = torch.from_numpy(nv).cuda()
        out = torch.empty_like(T)
        rec = {"config": cfg, "targets": M, "pairs": M * N}
        for eta in (0.0, 1.0):
            if eta > 0:
                bie.bie_set_near(ctx, eta)
            bie.bie_eval_traction(ctx, S, T, NV, out)
            torch.cuda.synchronize()
            reps = 3
            bie.bie_reset_profile(ctx)
            bie.bie_set_profiling(ctx, True)
            for _ in range(reps):
                bie.bie_eval_traction(ctx, S, T, NV, out)
            prof = bie.bie_get_profile(ctx)
            far = (prof["kfar"][0] + prof["reduce"][0]) / reps
            tot = sum(v[0] for v in prof.values()) / reps
            if eta == 0:
                rec.update({"far_ms": far, "pairs_per_s": M * N / (far / 1e3),
                            "fp64_pipe_frac": M * N / (far / 1e3) * 25 / (148 * 64 * 1.965e9),
                            "total_ms": tot})
            else:
                rec.update({"near_ms_eta1": prof["near"][0] / reps, "total_ms_eta1": tot})
        print(json.dumps(rec), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
