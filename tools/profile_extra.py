#!/usr/bin/env python
"""Driver for ncu captures of the round-1 extension kernels:
  --what K      : bie_apply_K on cfg 3           (k_nbody MODE=1)
  --what near   : apply with eta = 1 on cfg 4    (k_near, k_near_coef)
  --what nearoff: off-surface with eta = 1, cfg 5, 200k targets (k_near_off)
  --what self   : self term only, cfg 5          (k_self_t)
  --what nearK  : K apply with eta = 1 on cfg 4   (k_near<STAGE, K = true>, k_near_coef_K)"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", required=True)
    a = ap.parse_args()
    import torch
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config
    cfg = {"K": 3, "near": 4, "nearoff": 5, "self": 5, "nearK": 4}[a.what]
    d = make_config(cfg, with_targets=(a.what == "nearoff"))
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    N = d["n_nodes"]
    g = np.random.default_rng(0)
    F = torch.from_numpy(g.standard_normal((N, 3))).cuda()
    Q = torch.from_numpy(g.standard_normal((N, 3))).cuda()
    U = torch.empty_like(F)
    if a.what == "K":
        bie.bie_apply_K(ctx, F, U)
    elif a.what == "nearK":
        bie.bie_set_near(ctx, 1.0)
        bie.bie_apply_K(ctx, F, U)
    elif a.what == "near":
        bie.bie_set_near(ctx, 1.0)
        bie.bie_apply_SLDL(ctx, F, Q, U)
    elif a.what == "nearoff":
        bie.bie_set_near(ctx, 1.0)
        tg = torch.from_numpy(np.ascontiguousarray(d["targets"][:200000])).cuda()
        uo = torch.empty_like(tg)
        po = torch.empty(tg.shape[0], dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, F, Q, tg, uo, po)
    else:
        for _ in range(3):
            bie.bie_apply_parts(ctx, F, Q, U, bie.BIE_PART_SELF)
    torch.cuda.synchronize()
    ctx.close()
    print("ok")


if __name__ == "__main__":
    main()
