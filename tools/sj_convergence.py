#!/usr/bin/env python
"""Two fixed equal spheres in a uniform flow along their line of centres
(Problem 1, BIE 5.4) solved on the GPU with the near-singular correction:
relative error of the drag against the Stimson-Jeffery series vs p and gap."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1707_06551_b200 as bie
    from tests.test_oracle_porous import stimson_jeffery
    for gap in (2.0, 1.0, 0.5, 0.25, 0.1):
        c = 1.0 + gap / 2
        lam = stimson_jeffery(c)
        for p in (6, 8, 12, 16, 20, 24, 30):
            cen = np.array([[0.0, 0.0, -c], [0.0, 0.0, c]])
            ctx = bie.bie_create(cen, np.ones(2), p, 1.0)
            bie.bie_set_near(ctx, 10.0)
            N = bie.bie_num_nodes(ctx)
            uinf = torch.zeros((N, 3), dtype=torch.float64, device="cuda")
            uinf[:, 2] = 1.0
            mu = torch.empty_like(uinf)
            it, res = bie.bie_solve_porous(ctx, uinf, mu, tol=1e-14, max_iter=400, restart=200)
            w = torch.empty(N, dtype=torch.float64, device="cuda")
            bie.bie_get_nodes(ctx, None, None, w)
            torch.cuda.synchronize()
            nsn = N // 2
            F = -(w[:nsn, None] * mu[:nsn]).sum(0).cpu().numpy()
            ctx.close()
            print(json.dumps({"gap": gap, "p": p, "iterations": it, "rel_resid": res,
                              "lambda_SJ": lam, "lambda_gpu": F[2] / (6 * np.pi),
                              "rel_err": abs(F[2] / (6 * np.pi) - lam) / lam}), flush=True)


if __name__ == "__main__":
    main()
