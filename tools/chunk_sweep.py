#!/usr/bin/env python
"""Far-field time of one config vs the number of source chunks (the
library's planner = 0), CUDA events, median of many reps."""
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
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    chunks = [int(a) for a in sys.argv[2:]] or [0, 9, 14, 20, 27, 40, 54, 81]
    d = make_config(cfg, with_targets=False)
    N = d["n_nodes"]
    nsn = (d["p"] + 1) * (2 * d["p"] + 2)
    g = np.random.default_rng(0)
    F = torch.from_numpy(g.standard_normal((N, 3))).cuda()
    Q = torch.from_numpy(g.standard_normal((N, 3))).cuda()
    U = torch.empty_like(F)
    for ch in chunks:
        ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
        if ch:
            bie.bie_set_source_chunks(ctx, ch)
        for _ in range(5):
            bie.bie_apply_parts(ctx, F, Q, U, bie.BIE_PART_FAR)
        torch.cuda.synchronize()
        ts = []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bie.bie_apply_parts(ctx, F, Q, U, bie.BIE_PART_FAR)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        pairs = N * (N - nsn)
        print(json.dumps({"config": cfg, "chunks": ch, "far_ms": ms, "pairs_per_s": pairs / ms * 1e3,
                          "fp64_pipe_frac": pairs / ms * 1e3 * 30 / (148 * 64 * 1.965e9)}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
