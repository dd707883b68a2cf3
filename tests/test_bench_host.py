"""Host-side logic of bench.py's multi-GPU (replicas-only) path, exercised with
torch.distributed over gloo at world_size 2 on CPU."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r "took" 100 + 50 r ms for 2 steps of 1e9 pairs each
    m = bench.max_over_ranks(100.0 + 50.0 * rank, world)
    v = bench.replica_value(10 ** 9, 2, world, m)
    out[rank] = (m, v)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    mp = torch.multiprocessing.get_context("spawn")
    with mp.Manager() as man:
        out = man.dict()
        port = _free_port()
        ps = [mp.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(120)
            assert p.exitcode == 0
        res = dict(out)
    assert res[0] == res[1]
    m, v = res[0]
    assert m == 150.0                         # max over ranks
    assert abs(v - 2 * 2e9 / 0.15) < 1e-3     # all ranks' pairs / max time


def test_single_rank_is_identity():
    import bench
    assert bench.max_over_ranks(12.5, 1) == 12.5
    assert bench.replica_value(10, 3, 1, 1000.0) == 30.0


def test_dist_env_defaults(monkeypatch):
    import bench
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE"):
        monkeypatch.delenv(k, raising=False)
    assert bench.dist_env() == (0, 0, 1)


def test_reference_arm_json_line():
    """bench.py --impl reference (the CPU oracle arm) prints one JSON line with
    the contract's keys; runs on CPU only."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--config", "2", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "pair-interactions/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
