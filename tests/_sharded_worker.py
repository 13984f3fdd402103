"""Worker for the multi-process sharded-solve tests (run under torch.distributed.run).

python tests/_sharded_worker.py transport|host-ops n p k rho loss seed [batch]
Prints one JSON line per rank.
"""
import json
import os
import sys


def emit(obj):
    """One result line per rank in a single write(2): the ranks share the
    launcher's stdout pipe, and writes below PIPE_BUF do not interleave."""
    sys.stdout.flush()
    os.write(1, (json.dumps(obj) + "\n").encode())


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def host_ops_check():
    """The host transport's callbacks, driven exactly as the C++ loop drives them."""
    import ctypes as C
    import torch.distributed as dist
    from paper_2605_22188_b200 import sharded
    dist.init_process_group("gloo")
    tr = sharded.HostTransport()
    r, w = tr.rank, tr.world
    send = (C.c_double * 3)(r, 10.0 + r, -r)
    recv = (C.c_double * (3 * w))()
    rc1 = tr.ops.allgather(None, C.cast(send, C.c_void_p), 24, C.cast(recv, C.c_void_p))
    # rank r sends (q + 1) * (r + 1) bytes to peer q, filled with 16 r + q
    sb = [(q + 1) * (r + 1) for q in range(w)]
    rb = [(r + 1) * (q + 1) for q in range(w)]
    payload = bytes(b for q in range(w) for b in [16 * r + q] * sb[q])
    sbuf = C.create_string_buffer(payload, len(payload))
    rbuf = C.create_string_buffer(sum(rb))
    rc2 = tr.ops.alltoallv(None, C.cast(sbuf, C.c_void_p), (C.c_int64 * w)(*sb),
                           C.cast(rbuf, C.c_void_p), (C.c_int64 * w)(*rb))
    got = list(rbuf.raw)
    exp = [16 * q + r for q in range(w) for _ in range(rb[q])]
    emit({"rank": r, "rc": [rc1, rc2], "allgather": list(recv), "alltoallv_ok": got == exp})
    dist.destroy_process_group()


def solve(transport, n, p, k, rho, loss, seed, batch, time_limit=float("inf")):
    import torch
    import torch.distributed as dist
    import paper_2605_22188_b200 as P
    local = int(os.environ.get("LOCAL_RANK", 0))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if transport == "nccl" else "gloo")
    inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss,
                                                   seed=seed))
    cfg = P.SolverConfig(batch_size=batch, time_limit=time_limit)
    with P.Engine(inst, device=dev) as eng:
        try:
            cert = eng.solve_sharded(cfg, transport=transport)
        except Exception as e:  # noqa: BLE001 -- reported, every rank must get here
            emit({"rank": dist.get_rank(), "error": f"{type(e).__name__}: {e}"})
            return
        stats = eng.shard_stats()
    emit({"rank": dist.get_rank(), "support": cert.support, "value": cert.optimal_value,
          "nodes": cert.nodes_processed, "status": cert.status, "lb_batches": cert.lb_batches,
          "sent": stats["sent"], "received": stats["received"],
          "batch_per_pass": stats["batch_per_pass"]})
    dist.destroy_process_group()


if __name__ == "__main__":
    if sys.argv[1] == "host-ops":
        host_ops_check()
    else:
        a = sys.argv[2:]
        solve(sys.argv[1], int(a[0]), int(a[1]), int(a[2]), float(a[3]), int(a[4]), int(a[5]),
              int(a[6]) if len(a) > 6 else 0, float(a[7]) if len(a) > 7 else float("inf"))
