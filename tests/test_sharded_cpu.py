"""CPU tests of the node-sharded solve's host logic: the
deterministic load-balancing plan and the torch.distributed host transport the
C++ loop calls back into, over a world-size-2 gloo group."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def run_ranks(nproc, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
           str(_free_port()), os.path.join(ROOT, "tests", "_sharded_worker.py"), *map(str, args)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{\"rank\"")]
    assert len(lines) == nproc, out.stdout
    return sorted(lines, key=lambda d: d["rank"])


def test_balance_plan_cases(bnb):
    assert bnb.balance_plan([5, 5]) is None            # balanced
    assert bnb.balance_plan([1, 0]) is None            # nothing to give
    assert bnb.balance_plan([0]) is None               # single rank
    mv = bnb.balance_plan([7, 0])                      # idle rank starves
    assert mv.tolist() == [[0, 3], [0, 0]]
    mv = bnb.balance_plan([40, 2, 3, 1])               # skewed: donors give surplus over target
    assert mv.sum(axis=1)[0] == 40 - 12 and (mv[1:] == 0).all()
    assert mv.sum(axis=0).tolist() == [0, 10, 8, 10]
    rng = np.random.default_rng(0)
    for _ in range(200):                               # conservation, no self moves
        w = int(rng.integers(2, 9))
        c = rng.integers(0, 50, size=w)
        mv = bnb.balance_plan(c)
        if mv is None:
            continue
        assert (np.diag(mv) == 0).all() and (mv >= 0).all()
        after = c - mv.sum(axis=1) + mv.sum(axis=0)
        assert after.sum() == c.sum() and (after >= 0).all()
        assert after.max() - after.min() <= max(c.max() - c.min(), 1)


def test_host_transport_gloo_world2():
    res = run_ranks(2, "host-ops")
    for d in res:
        assert d["rc"] == [0, 0]
        assert d["allgather"] == [0.0, 10.0, 0.0, 1.0, 11.0, -1.0]
        assert d["alltoallv_ok"]
