"""Seeded input generators (bie_inputs): recipes of SURVEY.md §8(d)."""
import numpy as np
import pytest

from bie_inputs import gen


def test_batched_draws_equal_sequential_draws():
    g1 = np.random.default_rng(123)
    a = g1.uniform(0.0, 60.0, (50, 3))
    g2 = np.random.default_rng(123)
    b = np.array([g2.uniform(0.0, 60.0, 3) for _ in range(50)])
    assert np.array_equal(a, b)


def _rsa_plain(seed, n, side, dmin):
    g = np.random.default_rng(seed)
    acc = []
    while len(acc) < n:
        c = g.uniform(0.0, side, 3)
        if all(np.linalg.norm(c - x) >= dmin for x in acc):
            acc.append(c)
    return np.array(acc)


def test_rsa_uniform_equals_plain_loop():
    ref = _rsa_plain(77, 60, 15.0, 2.5)
    got = gen.rsa_uniform(np.random.default_rng(77), 60, 15.0, 2.5)
    assert np.array_equal(ref, got)


def test_config1_matches_baseline_recipe():
    d = gen.make_config(1)
    assert d["p"] == 4 and d["n_nodes"] == 100
    assert np.allclose(d["f"][0], [0.125730221093393, -0.132104863291302, 0.640422650443282], atol=1e-15)
    assert np.allclose(d["q"][0], [1.203258954116498, 0.637073235626183, 0.558339961695143], atol=1e-15)


def test_config2_geometry():
    d = gen.make_config(2)
    c = d["centres"]
    dist = np.linalg.norm(c[:, None] - c[None], axis=-1) + np.eye(64) * 1e9
    assert dist.min() >= 2.5 and d["n_nodes"] == 10368
    assert c.min() >= 0 and c.max() <= 20


def test_config3_geometry():
    d = gen.make_config(3)
    c, a = d["centres"], d["radii"]
    assert abs(d["box_side"] - 36.870) < 5e-4       # SURVEY §8(d) [scratch] L = 36.870
    dist = np.linalg.norm(c[:, None] - c[None], axis=-1)
    lim = a[:, None] + a[None] + 0.2 * np.minimum(a[:, None], a[None])
    np.fill_diagonal(dist, 1e9)
    assert np.all(dist >= lim)
    assert d["subset"].shape == (4096,) and np.all(np.diff(d["subset"]) > 0)


def test_config4_geometry():
    d = gen.make_config(4)
    c = d["centres"]
    assert c.shape == (4096, 3) and d["same_fq"] and d["n_nodes"] == 1384448
    from scipy.spatial import cKDTree
    dd, _ = cKDTree(c).query(c, k=2)
    assert dd[:, 1].min() >= 2.5


@pytest.mark.slow
def test_config5_geometry_and_targets():
    d = gen.make_config(5)
    from scipy.spatial import cKDTree
    t = cKDTree(d["centres"])
    dd, _ = t.query(d["centres"], k=2)
    assert dd[:, 1].min() >= 2.5
    dt, _ = t.query(d["targets"], k=1)
    assert d["targets"].shape == (1_000_000, 3) and (dt - 1.0).min() >= 0.25
