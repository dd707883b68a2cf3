#!/usr/bin/env python
"""How much of the self-term kernel's time is the record packing alone: time
the self-term launch of bie_apply_parts with SELF (pack + transforms) and with
FAR only (the same kernel writes the records and zeros, no transforms), per
config, L2 flushed before every call.  Usage: python tools/self_split_probe.py [cfg ...]"""
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
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for cfg in [int(x) for x in sys.argv[1:]] or [3, 5]:
        d = make_config(cfg, with_targets=False)
        ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
        N = bie.bie_num_nodes(ctx)
        rng = np.random.default_rng(5)
        F = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        Q = torch.from_numpy(rng.standard_normal((N, 3))).cuda()
        U = torch.empty_like(F)
        out = {"cfg": cfg, "p": d["p"], "n_nodes": N}
        for name, parts in (("self_and_pack", bie.BIE_PART_SELF), ("pack_only", bie.BIE_PART_FAR)):
            bie.bie_apply_parts(ctx, F, Q, U, parts)
            torch.cuda.synchronize()
            bie.bie_reset_profile(ctx)
            bie.bie_set_profiling(ctx, True)
            reps = 10
            for _ in range(reps):
                flush.zero_()
                bie.bie_apply_parts(ctx, F, Q, U, parts)
            prof = bie.bie_get_profile(ctx)
            bie.bie_set_profiling(ctx, False)
            out[name + "_ms"] = prof["self"][0] / reps
        print(json.dumps(out), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
