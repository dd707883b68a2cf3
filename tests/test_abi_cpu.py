"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/bie.h declares, and create-time validation returns the documented
status codes before any CUDA work (a valid create on a GPU-less host reports
BIE_ERR_CUDA instead of crashing)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def abi():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1707_06551_b200 import _abi
    return _abi


def test_header_symbols_exported(abi):
    hdr = open(os.path.join(ROOT, "include", "bie.h")).read()
    declared = set(re.findall(r"\b(bie_[a-zA-Z_]+)\s*\(", hdr))
    assert declared == set(abi.SYMBOLS), declared ^ set(abi.SYMBOLS)
    lib = ctypes.CDLL(abi.LIB_PATH)
    for s in declared:
        assert hasattr(lib, s), s


def test_status_strings(abi):
    for st in range(6):
        assert abi._lib.bie_status_string(st)
    assert abi._lib.bie_last_error(None) == b"NULL context"


def _mk(c, a, ns, p, mu, abi):
    c = np.ascontiguousarray(c, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    return abi.raw_create(c.ctypes.data, a.ctypes.data, ns, p, mu)


def test_create_validation(abi):
    c = np.array([[0.0, 0, 0], [3.0, 0, 0]])
    a = np.ones(2)
    assert abi.raw_create(None, a.ctypes.data, 2, 4, 1.0)[0] == abi.BIE_ERR_ARG
    assert _mk(c, a, 0, 4, 1.0, abi)[0] == abi.BIE_ERR_ARG
    assert _mk(c, a, 2, 0, 1.0, abi)[0] == abi.BIE_ERR_UNSUPPORTED
    assert _mk(c, a, 2, abi.BIE_P_MAX + 1, 1.0, abi)[0] == abi.BIE_ERR_UNSUPPORTED
    assert _mk(c, a, 2, 4, 0.0, abi)[0] == abi.BIE_ERR_ARG
    assert _mk(c, a, 2, 4, float("nan"), abi)[0] == abi.BIE_ERR_ARG
    assert _mk(c, [1.0, -1.0], 2, 4, 1.0, abi)[0] == abi.BIE_ERR_ARG
    assert _mk([[0, 0, np.inf], [3, 0, 0]], a, 2, 4, 1.0, abi)[0] == abi.BIE_ERR_ARG
    assert _mk([[0, 0, 0], [1.9, 0, 0]], a, 2, 4, 1.0, abi)[0] == abi.BIE_ERR_GEOMETRY
    # touching is rejected too (SPEC: centre distance > sum of radii): at even p
    # both spheres would carry a node at the contact point
    assert _mk([[0, 0, 0], [2.0, 0, 0]], a, 2, 4, 1.0, abi)[0] == abi.BIE_ERR_GEOMETRY
    rc, h = _mk([[0, 0, 0], [2.0 + 1e-9, 0, 0]], a, 2, 4, 1.0, abi)
    assert rc != abi.BIE_ERR_GEOMETRY


def test_overlap_check_scales_with_cell_list(abi):
    # 20^3 lattice of unit spheres, one pair pushed into overlap at the far corner
    g = np.arange(20) * 2.5
    c = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    c[-1] = c[-2] + np.array([0.0, 0.0, 1.5])
    a = np.ones(len(c))
    assert _mk(c, a, len(c), 4, 1.0, abi)[0] == abi.BIE_ERR_GEOMETRY


def test_no_device_reports_cuda_error(abi):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc, h = _mk([[0, 0, 0], [3.0, 0, 0]], np.ones(2), 2, 4, 1.0, abi)
    assert rc == abi.BIE_ERR_CUDA and h is None


def test_null_context_calls(abi):
    L = abi._lib
    assert L.bie_num_nodes(None) == -1
    assert L.bie_apply_SLDL(None, None, None, None, None) == abi.BIE_ERR_ARG
    assert L.bie_eval_offsurface(None, None, None, None, 0, None, None, None) == abi.BIE_ERR_ARG
    assert L.bie_set_profiling(None, 1) == abi.BIE_ERR_ARG
    L.bie_destroy(None)


def test_package_has_no_cpu_fallback():
    """The product package must not import the oracle or fall back to CPU math."""
    pkg = os.path.join(ROOT, "paper_1707_06551_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn


@pytest.mark.parametrize("seed,ns,eta,poly", [(1, 60, 1.0, True), (2, 120, 0.5, False), (3, 40, 3.0, True),
                                              (4, 1, 1.0, False), (5, 120, 0.0, True)])
def test_near_lists_match_bruteforce_eq45(abi, oracle_mod, seed, ns, eta, poly):
    """The host cell-list neighbour builder (bie_near_lists; what bie_set_near
    uploads) equals the brute-force eq 4.5 test of the oracle (oracle.is_near)
    over all ordered pairs, ascending per target; eta = 0 gives no pairs."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.5, 1.5, ns) if poly else np.ones(ns)
    c = []
    while len(c) < ns:
        x = rng.uniform(0, 3.2 * ns ** (1 / 3) + 2, 3)
        if all(np.linalg.norm(x - y) > a[len(c)] + a[j] + 0.05 for j, y in enumerate(c)):
            c.append(x)
    c = np.array(c)
    off, idx = abi.bie_near_lists(c, a, eta)
    for t in range(ns):
        ref = [s for s in range(ns) if s != t and oracle_mod.is_near(c[s], a[s], c[t], a[t], eta)]
        assert list(idx[off[t]:off[t + 1]]) == ref, t
