import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1707_06551_b200 as bie
from bie_inputs import make_config
for cfg in (2, 4, 5):
    d = make_config(cfg, with_targets=False)
    p = d["p"]; nsn = (p+1)*(2*p+2); ns = len(d["radii"])
    ctx = bie.bie_create(d["centres"], d["radii"], p, 1.0)
    N = bie.bie_num_nodes(ctx)
    x = torch.empty((N, 3), dtype=torch.float64, device="cuda"); bie.bie_get_nodes(ctx, x)
    xc = x.cpu().numpy()
    g = np.random.default_rng(cfg)
    U = g.standard_normal((ns, 3)); Om = g.standard_normal((ns, 3))
    s = np.arange(N) // nsn
    q = U[s] + np.cross(Om[s], xc - d["centres"][s])
    Q = torch.from_numpy(q).cuda(); u = torch.empty_like(Q)
    for eta in (0.0, 1.0, 2.0, 3.0):
        bie.bie_set_near(ctx, eta)
        bie.bie_apply_DL(ctx, Q, u); torch.cuda.synchronize()
        err = np.abs(u.cpu().numpy() + 0.5*q).max() / np.abs(q).max()
        print(cfg, p, eta, bie.bie_near_pairs(ctx), f"{err:.3e}", flush=True)
    ctx.close()
