#!/usr/bin/env python
"""Far-field schedules (bie_set_far_reduction): 0 stream-K persistent CTAs,
1 source chunks + HBM partials + k_reduce (round 1), 2/3/4 on-chip
thread-block-cluster reductions through distributed shared memory (clusters
of 8/4/16), 5 source chunks summed inside the kernel (chained, ticket order),
7 constant-bank source batches over two streams (k_nbody_c.cuh).
FR_MODES=1,5 selects the schedules.  Times bie_apply_SLDL's far
field (kind nbody + reduce) and the off-surface evaluator on BASELINE configs,
L2 flushed before every timed call.  Usage: python tools/far_reduction_bench.py [cfg ...]"""
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
    cfgs = [int(x) for x in sys.argv[1:]] or [5, 4]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for cfg in cfgs:
        d = make_config(cfg, with_targets=(cfg == 5))
        ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
        N = d["n_nodes"]
        rng = np.random.default_rng(1)
        F = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        U = torch.empty_like(F)
        tg = torch.from_numpy(d["targets"]).cuda() if d["targets"] is not None else None
        for mode in [int(x) for x in os.environ.get("FR_MODES", "0,1,2,3,4,5").split(",")]:
            bie.bie_set_far_reduction(ctx, mode)
            bie.bie_apply_SLDL(ctx, F, Q, U)
            torch.cuda.synchronize()
            bie.bie_reset_profile(ctx)
            bie.bie_set_profiling(ctx, True)
            reps = 2
            for _ in range(reps):
                flush.zero_()
                bie.bie_apply_SLDL(ctx, F, Q, U)
                if tg is not None:
                    uo = torch.empty_like(tg)
                    po = torch.empty(tg.shape[0], dtype=torch.float64, device="cuda")
                    flush.zero_()
                    bie.bie_eval_offsurface(ctx, F, Q, tg, uo, po)
            prof = bie.bie_get_profile(ctx)
            bie.bie_set_profiling(ctx, False)
            nsn = (d["p"] + 1) * (2 * d["p"] + 2)
            far_ms = (prof["nbody"][0] + prof["reduce"][0] * (0.5 if tg is not None else 1.0)) / reps
            rec = {"cfg": cfg, "far_reduction": mode, "nbody_ms": prof["nbody"][0] / reps,
                   "reduce_ms": prof["reduce"][0] / reps, "apply_far_ms": far_ms,
                   "apply_pairs_per_s": N * (N - nsn) / (prof["nbody"][0] / reps / 1e3)}
            if tg is not None:
                rec["offsurface_ms"] = prof["offsurface"][0] / reps
                rec["offsurface_pairs_per_s"] = tg.shape[0] * N / (prof["offsurface"][0] / reps / 1e3)
            print(json.dumps(rec), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
