#!/usr/bin/env python
"""B200 analogue of the paper's scaling experiment (E6, PAPER §6 P:604-618,
Fig 9 -- whose data is missing from the extracted text): apply time of the
double layer D and of the traction operator K versus the number of spheres
n_b, on cubic lattices of unit spheres (spacing 3, i.e. the "q = 1" loose
lattice reading r_v = 1 - 2^-1 of the unit cell half-width), p in {4, 8}.
The paper's far field is an FMM (slopes -> 1); here it is the direct O(N^2)
sum, so the expected slope is 2 once the GPU is full.  Near correction off
(the paper's near scheme is NEXT-1 here; its cost is reported separately)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lattice(k, spacing=3.0):
    g = np.arange(k) * spacing
    return np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)


def main():
    import torch
    import paper_1707_06551_b200 as bie
    for p in (4, 8):
        for k in (2, 3, 5, 9, 17, 25):
            c = lattice(k)
            a = np.ones(len(c))
            ctx = bie.bie_create(c, a, p, 1.0)
            N = bie.bie_num_nodes(ctx)
            x = torch.randn(N, 3, dtype=torch.float64, device="cuda")
            u = torch.empty_like(x)
            res = {}
            for op in ("D", "K"):
                call = (lambda: bie.bie_apply_DL(ctx, x, u)) if op == "D" else (lambda: bie.bie_apply_K(ctx, x, u))
                call()
                torch.cuda.synchronize()
                reps = 3 if N > 300000 else 10
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    call()
                e1.record()
                e1.synchronize()
                res[op] = e0.elapsed_time(e1) / reps
            print(json.dumps({"p": p, "lattice": f"{k}^3", "n_b": len(c), "N": N,
                              "D_ms": res["D"], "K_ms": res["K"]}), flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
