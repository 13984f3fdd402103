"""Node-sharded certified solve over torch.distributed ranks.

The C++ host loop (bnbg_solve_sharded) drives the exchange; this module only
binds a transport:

* ``nccl``: rank 0 draws an NCCL unique id, the group broadcasts it, every
  rank binds its handle (bnbg_nccl_init); incumbent records and node records
  then move device-to-device over NVLink inside the engine.
* ``host``: the engine calls back into ``torch.distributed`` (gloo) with host
  buffers -- all_gather for the per-pass records, all_to_all_single for node
  records.  This is what the multi-process CPU tests and several ranks sharing
  one GPU use.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional


from . import _lib as _L


def _torch_dist():
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("solve_sharded needs an initialised torch.distributed process group")
    return torch, dist


class HostTransport:
    """bnbg_comm_ops over a torch.distributed group with CPU tensors."""

    def __init__(self, group=None):
        torch, dist = _torch_dist()
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._ag = _L.ALLGATHER_FN(self._allgather)
        self._a2a = _L.ALLTOALLV_FN(self._alltoallv)
        self.ops = _L.CommOpsC(None, self.rank, self.world, self._ag, self._a2a)
        self.error = None

    def _allgather(self, _ctx, send, nbytes, recv):
        try:
            t = self.torch
            src = t.frombuffer(C.string_at(send, nbytes), dtype=t.uint8) if nbytes else \
                t.empty(0, dtype=t.uint8)
            outs = [t.empty(nbytes, dtype=t.uint8) for _ in range(self.world)]
            self.dist.all_gather(outs, src.clone(), group=self.group)
            buf = b"".join(o.numpy().tobytes() for o in outs)
            C.memmove(recv, buf, len(buf))
            return 0
        except Exception as e:  # surfaced by solve_sharded
            self.error = e
            return 1

    def _alltoallv(self, _ctx, send, send_bytes, recv, recv_bytes):
        try:
            t = self.torch
            ss = [int(send_bytes[q]) for q in range(self.world)]
            rs = [int(recv_bytes[q]) for q in range(self.world)]
            src = t.frombuffer(bytearray(C.string_at(send, sum(ss))), dtype=t.uint8) \
                if sum(ss) else t.empty(0, dtype=t.uint8)
            out = t.empty(sum(rs), dtype=t.uint8)
            self.dist.all_to_all_single(out, src, rs, ss, group=self.group)
            if sum(rs):
                C.memmove(recv, out.numpy().tobytes(), sum(rs))
            return 0
        except Exception as e:
            self.error = e
            return 1


_UIDS = {}  # (group, world) -> NCCL unique id shared by every engine of this process


def nccl_bind(engine, group=None):
    """Bind the engine to an NCCL communicator over the group's ranks.  The
    unique id is drawn and broadcast once per group; later engines of the
    process reuse the library's cached communicator (no re-initialisation)."""
    torch, dist = _torch_dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    key = (id(group), world)
    if key not in _UIDS:
        uid = C.create_string_buffer(128)
        if rank == 0:
            if _L.lib().bnbg_nccl_unique_id(uid) != 0:
                raise RuntimeError("bnbg_nccl_unique_id failed")
        obj = [bytes(uid.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        _UIDS[key] = obj[0]
    from . import _check
    _check(_L.lib().bnbg_nccl_init(engine.handle, _UIDS[key], rank, world), engine.handle)


def solve_sharded(engine, config=None, group=None, transport: Optional[str] = None):
    from . import SolverConfig, _cert_from_c, _check
    torch, dist = _torch_dist()
    if transport is None:
        transport = "nccl" if dist.get_backend(group) == "nccl" else "host"
    cfg = (config or SolverConfig()).to_c()
    k = engine.inst.k
    sup = (C.c_int32 * (k + 1))()
    coef = (C.c_double * (k + 1))()
    cc = _L.CertC()
    cc.support = C.cast(sup, C.POINTER(C.c_int32))
    cc.coefficients = C.cast(coef, C.POINTER(C.c_double))
    if transport == "nccl":
        if not getattr(engine, "_nccl_bound", False):
            nccl_bind(engine, group)
            engine._nccl_bound = True
        rc = _L.lib().bnbg_solve_sharded(engine.handle, C.byref(cfg), None, C.byref(cc))
        _check(rc, engine.handle)
    elif transport == "host":
        tr = HostTransport(group)
        rc = _L.lib().bnbg_solve_sharded(engine.handle, C.byref(cfg), C.byref(tr.ops), C.byref(cc))
        if tr.error is not None:
            raise tr.error
        _check(rc, engine.handle)
    else:
        raise ValueError(f"unknown transport {transport!r}")
    return _cert_from_c(cc, sup, coef)
