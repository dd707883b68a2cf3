"""Seeded generators for the BASELINE.json configurations.

No method arithmetic lives here: only placement of sphere centres by random
sequential addition (RSA), iid normal densities, rigid-body fields
U + Omega x (x - c) evaluated at caller-supplied node positions, and
off-surface target draws.  Every random number comes from
numpy.random.Generator(PCG64(seed)); batched draws consume the stream in
exactly the order of one-at-a-time draws (checked in tests/test_inputs.py),
so the batching below is an implementation detail, not part of the recipe.
"""
from __future__ import annotations

import numpy as np

try:  # scipy's k-d tree is only an accelerator for the RSA distance test
    from scipy.spatial import cKDTree as _KDTree
except Exception:  # pragma: no cover - scipy is in the image
    _KDTree = None

#: name -> short description; the numbers follow BASELINE.json "configs"
CONFIGS = {
    1: "2 unit spheres at (0,0,0),(3,0,0), p=4, mu=1, f,q ~ N(0,1) seed 0",
    2: "64 unit spheres, RSA in [0,20]^3 gap>=0.5, p=8, f,q ~ N(0,1)",
    3: "1000 spheres a~U[0.5,1.5], RSA at volume fraction 0.10, gap>=0.2*min(a), p=8, "
       "f ~ N(0,1), q = U + Omega x (x-c)",
    4: "4096 unit spheres, jittered cubic lattice spacing 3 (+-0.25), p=12, D[q]+S[q] with f:=q",
    5: "10000 unit spheres, RSA in [0,60]^3 gap>=0.5, p=6, f,q ~ N(0,1); "
       "1e6 off-surface targets >=0.25 from every surface",
}


def node_count(n_spheres: int, p: int) -> int:
    """N = n_spheres * (p+1) * (2p+2) (eq 4.2 grid)."""
    return int(n_spheres) * (p + 1) * (2 * p + 2)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def rsa_uniform(g: np.random.Generator, n: int, side: float, dmin: float) -> np.ndarray:
    """Random sequential addition of n centres in [0, side]^3.

    Candidate j is g.uniform(0, side, 3); it is accepted iff its distance to
    every previously accepted centre is >= dmin.  Identical to the plain
    one-candidate-at-a-time loop: candidates are drawn in batches (same
    stream), screened against the centres accepted before the batch with a
    k-d tree, then resolved in draw order against the centres accepted
    inside the batch.
    """
    acc = np.empty((n, 3))
    cnt = 0
    batch = 1024
    drawn = 0
    while cnt < n:
        cand = g.uniform(0.0, side, (batch, 3))
        drawn += batch
        if cnt and _KDTree is not None:
            d, _ = _KDTree(acc[:cnt]).query(cand, k=1, distance_upper_bound=dmin * 1.001)
            ok = d >= dmin
        elif cnt:
            d = np.sqrt(((cand[:, None, :] - acc[None, :cnt, :]) ** 2).sum(-1)).min(1)
            ok = d >= dmin
        else:
            ok = np.ones(batch, dtype=bool)
        start = cnt
        for j in np.nonzero(ok)[0]:
            c = cand[j]
            if cnt > start:
                dd = np.sqrt(((acc[start:cnt] - c) ** 2).sum(1))
                if np.any(dd < dmin):
                    continue
            acc[cnt] = c
            cnt += 1
            if cnt == n:
                break
        rate = max((cnt - start) / batch, 1e-5)
        batch = int(min(1 << 18, max(1024, 1.5 * (n - cnt) / rate)))
    return acc


def rsa_polydisperse(g: np.random.Generator, radii: np.ndarray, side: float,
                     gap_frac: float) -> np.ndarray:
    """RSA in index order: sphere i draws g.uniform(0, side, 3) until
    |c_i - c_j| >= a_i + a_j + gap_frac*min(a_i, a_j) for all j < i."""
    n = len(radii)
    acc = np.empty((n, 3))
    for i in range(n):
        while True:
            c = g.uniform(0.0, side, 3)
            if i == 0:
                break
            d = np.sqrt(((acc[:i] - c) ** 2).sum(1))
            lim = radii[:i] + radii[i] + gap_frac * np.minimum(radii[:i], radii[i])
            if np.all(d >= lim):
                break
        acc[i] = c
    return acc


def offsurface_targets(g: np.random.Generator, centres: np.ndarray, radius: float,
                       side: float, clearance: float, m: int) -> np.ndarray:
    """Draw candidates U[0,side]^3 (3 draws each, in order) and keep those with
    min_i(|x - c_i| - radius) >= clearance, until m are kept."""
    out = np.empty((m, 3))
    cnt = 0
    tree = _KDTree(centres) if _KDTree is not None else None
    while cnt < m:
        batch = int(min(1 << 20, max(4096, 1.7 * (m - cnt))))
        cand = g.uniform(0.0, side, (batch, 3))
        if tree is not None:
            d, _ = tree.query(cand, k=1)
        else:
            d = np.sqrt(((cand[:, None, :] - centres[None]) ** 2).sum(-1)).min(1)
        keep = cand[(d - radius) >= clearance]
        take = min(len(keep), m - cnt)
        out[cnt:cnt + take] = keep[:take]
        cnt += take
    return out


def rigid_field(U: np.ndarray, Omega: np.ndarray, x: np.ndarray, centres: np.ndarray,
                nodes_per_sphere: int) -> np.ndarray:
    """q_i = U_s + Omega_s x (x_i - c_s) for node i of sphere s (cfg 3)."""
    s = np.arange(x.shape[0]) // nodes_per_sphere
    return U[s] + np.cross(Omega[s], x - centres[s])


def make_config(cfg: int, *, with_targets: bool = True) -> dict:
    """Build config `cfg` (1..5) of BASELINE.json.

    Returns a dict with keys: cfg, p, mu, centres [Ns,3], radii [Ns], n_nodes,
    f [N,3] or None, q [N,3] or None, rigid (U, Omega) or None (cfg 3: q is
    rigid_field(U, Omega, x, ...) at the nodes), same_fq (cfg 4: f := q),
    subset (sorted node indices for the oracle, None = all), targets [M,3] or
    None, target_subset (sorted indices into targets) or None, seeds.
    """
    out = dict(cfg=cfg, mu=1.0, rigid=None, same_fq=False, subset=None,
               targets=None, target_subset=None, f=None, q=None)
    if cfg == 1:
        p = 4
        centres = np.array([[0.0, 0.0, 0.0], [3.0, 0.0, 0.0]])
        radii = np.ones(2)
        N = node_count(2, p)
        g = _rng(0)
        out["f"] = g.standard_normal((N, 3))
        out["q"] = g.standard_normal((N, 3))
        out["seeds"] = {"densities": 0}
    elif cfg == 2:
        p = 8
        centres = rsa_uniform(_rng(2001), 64, 20.0, 2.5)
        radii = np.ones(64)
        N = node_count(64, p)
        g = _rng(2002)
        out["f"] = g.standard_normal((N, 3))
        out["q"] = g.standard_normal((N, 3))
        out["seeds"] = {"geometry": 2001, "densities": 2002}
    elif cfg == 3:
        p = 8
        g = _rng(3001)
        radii = g.uniform(0.5, 1.5, 1000)
        L = (np.sum(4.0 / 3.0 * np.pi * radii ** 3) / 0.10) ** (1.0 / 3.0)
        centres = rsa_polydisperse(g, radii, L, 0.2)
        N = node_count(1000, p)
        g = _rng(3002)
        out["f"] = g.standard_normal((N, 3))
        U = g.standard_normal((1000, 3))
        Om = g.standard_normal((1000, 3))
        out["rigid"] = (U, Om)
        out["box_side"] = L
        out["subset"] = np.sort(_rng(3003).choice(N, 4096, replace=False))
        out["seeds"] = {"geometry": 3001, "densities": 3002, "subset": 3003}
    elif cfg == 4:
        p = 12
        ijk = np.array([(i, j, k) for i in range(16) for j in range(16) for k in range(16)],
                       dtype=np.float64)
        jit = _rng(4001).uniform(-0.25, 0.25, (4096, 3))
        centres = 3.0 * ijk + jit
        radii = np.ones(4096)
        N = node_count(4096, p)
        out["q"] = _rng(4002).standard_normal((N, 3))
        out["same_fq"] = True
        out["subset"] = np.sort(_rng(4003).choice(N, 4096, replace=False))
        out["seeds"] = {"geometry": 4001, "densities": 4002, "subset": 4003}
    elif cfg == 5:
        p = 6
        centres = rsa_uniform(_rng(5001), 10000, 60.0, 2.5)
        radii = np.ones(10000)
        N = node_count(10000, p)
        g = _rng(5002)
        out["f"] = g.standard_normal((N, 3))
        out["q"] = g.standard_normal((N, 3))
        gs = _rng(5003)
        out["subset"] = np.sort(gs.choice(N, 4096, replace=False))
        M = 1_000_000
        if with_targets:
            out["targets"] = offsurface_targets(_rng(5004), centres, 1.0, 60.0, 0.25, M)
        out["target_subset"] = np.sort(gs.choice(M, 4096, replace=False))
        out["seeds"] = {"geometry": 5001, "densities": 5002, "subset": 5003, "targets": 5004}
    else:
        raise ValueError(f"unknown config {cfg}")
    out.update(p=p, centres=np.ascontiguousarray(centres), radii=np.ascontiguousarray(radii),
               n_nodes=node_count(len(radii), p))
    return out
