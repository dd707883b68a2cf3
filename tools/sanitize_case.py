#!/usr/bin/env python
"""Small end-to-end exercise of every kernel (apply with near correction,
chunked and unchunked far field, off-surface with pressure) for
compute-sanitizer runs: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config
    d = make_config(2, with_targets=False)
    for chunks in (0, 1, 3):
        ctx = bie.bie_create(d["centres"][:12], d["radii"][:12], 5, 1.3)
        bie.bie_set_source_chunks(ctx, chunks)
        bie.bie_set_near(ctx, 2.0)
        N = bie.bie_num_nodes(ctx)
        g = np.random.default_rng(chunks)
        F = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(g.standard_normal((N, 3))).cuda()
        U = torch.empty_like(F)
        bie.bie_apply_SLDL(ctx, F, Q, U)
        bie.bie_apply_parts(ctx, F, None, U, bie.BIE_PART_FAR)
        tg = torch.from_numpy(g.uniform(-5, 25, (777, 3))).cuda()
        uo = torch.empty_like(tg)
        po = torch.empty(777, dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, F, Q, tg, uo, po)
        torch.cuda.synchronize()
        assert torch.isfinite(U).all()
        ctx.close()
    print("ok")


if __name__ == "__main__":
    main()
