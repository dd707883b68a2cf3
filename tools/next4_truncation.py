#!/usr/bin/env python
"""Why NEXT-4 (FFT-accelerated near evaluation with rotations, PAPER §4.2,
Fig 2) is not built: its stage 3 re-expands the neighbour's
exterior field on the TARGET sphere in VSH of degree <= p (forward transform
on the target grid, rotate, inverse transform).  At the Nystrom nodes that is
a projection P_p of a field that is not band-limited, so NEXT-4's near
contribution differs from the exact one (what k_near evaluates) by the
degree > p tail.  This script measures that tail with the oracle:
    err_trunc  = |P_p[u_ext] - u_ext| / |u_ext|   at the target nodes
    err_smooth = |u_smooth - u_ext| / |u_ext|      (no near correction at all)
for two unit spheres at gap g, a random band-limited density on the source.
CPU only (oracle + numpy least squares on the target grid)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def vsh_basis(p, pts, c, a):
    from tests import _harmonics as H
    cols = []
    th, ph = H.angles((pts - c) / a)
    for n in range(0, p + 1):
        for m in range(-n, n + 1):
            V, W, X = H.vsh(n, m, th, ph)
            for ch, Z in enumerate((V, W, X)):
                if n == 0 and ch:
                    continue
                cols.append(Z.reshape(-1))
    return np.stack(cols, 1)


def main():
    import oracle
    from tests.test_oracle_near_K import _bandlimited
    for p in (4, 6, 8, 12):
        for g in (0.1, 0.2, 0.5, 1.0):
            c = np.array([[0.0, 0.0, 0.0], [0.3, -0.4, 0.0]])
            c[1] *= (2.0 + g) / np.linalg.norm(c[1])
            a = np.ones(2)
            x, _, w = oracle.nodes(c, a, p)
            nsn = (p + 1) * (2 * p + 2)
            sig = np.zeros_like(x)
            sig[nsn:] = _bandlimited(5, p, x[nsn:], c[1], a[1])
            tgt = x[:nsn]
            u_ext = oracle.exterior_eval(p, c[1], 1.0, 1.0, sig[nsn:], None, tgt)
            u_smooth = oracle.far(c, a, p, 1.0, sig, None, np.arange(nsn))
            B = vsh_basis(p, tgt, c[0], 1.0)
            coef, *_ = np.linalg.lstsq(B, u_ext.reshape(-1).astype(complex), rcond=None)
            u_proj = np.real(B @ coef).reshape(-1, 3)
            sc = np.abs(u_ext).max()
            print(json.dumps({"p": p, "gap": g,
                              "err_trunc": float(np.abs(u_proj - u_ext).max() / sc),
                              "err_smooth": float(np.abs(u_smooth - u_ext).max() / sc)}), flush=True)


if __name__ == "__main__":
    main()
