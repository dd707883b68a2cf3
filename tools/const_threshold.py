#!/usr/bin/env python
"""Where does the constant-bank far field (bie_set_far_reduction 7, k_nbody_c)
overtake the shared-memory kernel (schedule 5: chunks, chained)?  Unit spheres
on a cubic lattice of spacing 3, p = 6 (98 nodes per sphere), white-noise
densities; L2 flushed before every timed apply; far-field time from the
library's own events.  BIE_CONST_SUB is read by bie_create (0 = one target
range).  Usage: python tools/const_threshold.py [n_spheres ...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1707_06551_b200 as bie
    sizes = [int(x) for x in sys.argv[1:]] or [1000, 2000, 3000, 4000, 5000, 6200, 8000]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    p = 6
    for ns in sizes:
        m = int(np.ceil(ns ** (1 / 3)))
        g = np.stack(np.meshgrid(*[np.arange(m)] * 3, indexing="ij"), -1).reshape(-1, 3)[:ns] * 3.0
        ctx = bie.bie_create(g, np.ones(ns), p, 1.0)
        N = bie.bie_num_nodes(ctx)
        rng = np.random.default_rng(ns)
        F = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        U = torch.empty_like(F)
        rec = {"n_spheres": ns, "n_nodes": N, "const_sub": os.environ.get("BIE_CONST_SUB", "default")}
        for mode in (5, 7):
            bie.bie_set_far_reduction(ctx, mode)
            bie.bie_apply_SLDL(ctx, F, Q, U)
            torch.cuda.synchronize()
            bie.bie_reset_profile(ctx)
            bie.bie_set_profiling(ctx, True)
            reps = 3
            for _ in range(reps):
                flush.zero_()
                bie.bie_apply_SLDL(ctx, F, Q, U)
            prof = bie.bie_get_profile(ctx)
            bie.bie_set_profiling(ctx, False)
            ms = (prof["nbody"][0] + prof["reduce"][0]) / reps
            rec[f"ms_mode{mode}"] = round(ms, 3)
            rec[f"pairs_per_s_mode{mode}"] = N * (N - 98) / (ms / 1e3)
        rec["ratio_5_over_7"] = round(rec["ms_mode5"] / rec["ms_mode7"], 4)
        print(json.dumps(rec), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
