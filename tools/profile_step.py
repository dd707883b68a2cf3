#!/usr/bin/env python
"""Minimal driver for ncu / compute-sanitizer: build config `--config` and run
`--reps` apply steps (plus off-surface for cfg 5 unless --no-off).  Exits 0 on
success.  Example (on the GPU box):
  ncu --set full -k regex:k_nbody -c 1 -o gpurun_out/prof python tools/profile_step.py --config 3
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--no-off", action="store_true")
    ap.add_argument("--targets", type=int, default=0, help="limit off-surface targets (0 = all)")
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--far-reduction", type=int, default=1, help="bie_set_far_reduction mode (1 = library default)")
    ap.add_argument("--self-kernel", type=int, default=-1, help="bie_set_self_kernel variant (-1 = auto)")
    ap.add_argument("--eta", type=float, default=0.0, help="bie_set_near (0 = off)")
    ap.add_argument("--near-mode", type=int, default=0, help="bie_set_near_mode")
    args = ap.parse_args()
    import torch
    import paper_1707_06551_b200 as bie
    from bie_inputs import make_config, rigid_field
    d = make_config(args.config, with_targets=(args.config == 5 and not args.no_off))
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    if args.chunks:
        bie.bie_set_source_chunks(ctx, args.chunks)
    bie.bie_set_far_reduction(ctx, args.far_reduction)
    bie.bie_set_self_kernel(ctx, args.self_kernel)
    if args.eta > 0:
        bie.bie_set_near(ctx, args.eta)
        bie.bie_set_near_mode(ctx, args.near_mode)
    N = bie.bie_num_nodes(ctx)
    f_np, q_np = d["f"], d["q"]
    if d["rigid"] is not None:
        x = torch.empty((N, 3), dtype=torch.float64, device="cuda")
        bie.bie_get_nodes(ctx, x)
        q_np = rigid_field(*d["rigid"], x.cpu().numpy(), d["centres"], (d["p"] + 1) * (2 * d["p"] + 2))
    if d["same_fq"]:
        f_np = q_np
    f = torch.from_numpy(np.ascontiguousarray(f_np)).cuda()
    q = torch.from_numpy(np.ascontiguousarray(q_np)).cuda()
    u = torch.empty_like(f)
    tg = None
    if d["targets"] is not None:
        t = d["targets"] if args.targets == 0 else d["targets"][: args.targets]
        tg = torch.from_numpy(np.ascontiguousarray(t)).cuda()
        uo = torch.empty_like(tg)
        po = torch.empty(tg.shape[0], dtype=torch.float64, device="cuda")
    for _ in range(args.reps):
        bie.bie_apply_SLDL(ctx, f, q, u)
        if tg is not None:
            bie.bie_eval_offsurface(ctx, f, q, tg, uo, po)
    torch.cuda.synchronize()
    assert torch.isfinite(u).all()
    ctx.close()
    print("ok", N)


if __name__ == "__main__":
    main()
