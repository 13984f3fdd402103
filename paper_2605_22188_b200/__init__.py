"""B200-native batched branch-and-bound for cardinality-constrained GLMs.

Python mirror of the reference bnbglm API (``/root/reference/proj/include/bnbglm``)
for the node-processing path, over the C-ABI of ``libbnbg.so`` (include/bnbg.h).
Names, fields, defaults and error behaviour follow the reference:

=======================  ==========================================================
this module              reference
=======================  ==========================================================
``ProblemInstance``      problem.hpp:24-34
``validate``             problem.hpp:36-51
``generate_synthetic``   problem.hpp:53-132 (GeneratorSpec + generator)
``smoothness_constant``  losses.hpp:86-112 (power iteration on the device)
``RelaxConfig``          relaxation.hpp:26-33
``SolverConfig``         bnb_engine.hpp:28-36
``Certificate``          bnb_engine.hpp:40-60
``DebugHooks``           bnb_engine.hpp:63-66
``auto_batch_size``      bnb_engine.hpp:75-88
``Engine.solve_batch_relaxation``  relaxation.hpp:163-255
``Engine.round_support`` primal_heuristics.hpp:134-146
``Engine.select_branch_variable``  primal_heuristics.hpp:148-163
``Engine.reoptimize_supports``     primal_heuristics.hpp:174-227
``solve``                bnb_engine.hpp:299-309
``collect_rashomon``     rashomon.hpp:149-218
``prox_step``            prox_kernel.hpp:284-301
``batched_conjugate_prox``         prox_kernel.hpp:214-229
``g_value`` / ``g_conjugate_value``  prox_kernel.hpp:374-387
``Engine.pool_root`` / ``pool_relax`` / ``pool_branch``  the device-resident per-pass
                         seam (bnb_engine.hpp:140, :188-206, :243-255)
``solve_sharded``        node-parallel solving over GPUs (new)
``io.load_csv`` / ``io.save_csv``  problem.hpp:208-288
``io.certificate_to_json``         serialize.hpp:40-64
``io.file_fingerprint``            serialize.hpp:149-161
=======================  ==========================================================

Errors: ``InputError`` (input_error), ``NumericError`` (numeric_error),
``LogicError`` (std::logic_error), ``io.ParseError`` (parse_error), ``CudaError``
(new; no CPU fallback exists).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as _L

__all__ = [
    "LossKind", "CoordState", "NodeStatus", "ProblemInstance", "GeneratorSpec", "NodeState",
    "RelaxConfig", "SolverConfig", "Certificate", "ComponentProfile", "DebugHooks",
    "RashomonConfig", "RashomonResult", "RelaxationResult", "ReoptResult", "Engine",
    "InputError", "NumericError", "LogicError", "CudaError", "validate", "generate_synthetic",
    "smoothness_constant", "auto_batch_size", "solve", "collect_rashomon", "prox_step",
    "batched_conjugate_prox", "g_value", "g_conjugate_value", "root_node", "lib_path",
    "balance_plan", "solve_sharded",
]


class InputError(ValueError):
    """bnbglm::input_error (errors.hpp:9-12)."""


class NumericError(ArithmeticError):
    """bnbglm::numeric_error (errors.hpp:21-24)."""


class LogicError(RuntimeError):
    """std::logic_error (node_model.hpp:81-82, primal_heuristics.hpp:161)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside libbnbg.so."""


_ERRS = {1: InputError, 2: NumericError, 3: LogicError, 4: CudaError}


def _check(rc: int, handle=None):
    if rc == 0:
        return
    msg = _L.lib().bnbg_last_error(handle)
    raise _ERRS.get(rc, RuntimeError)(msg.decode() if msg else f"bnbg error {rc}")


def lib_path() -> str:
    return _L.LIB_PATH


class LossKind:
    SQUARED = 0
    LOGISTIC = 1


class CoordState:
    FREE = 0
    FIXED_ONE = 1
    FIXED_ZERO = 2


class NodeStatus:
    PRUNABLE = 0
    CONVERGED = 1
    ITERATION_CAPPED = 2


@dataclass
class ProblemInstance:
    """problem.hpp:24-34.  X is n x p (stored column-major, float64)."""
    X: np.ndarray
    y: np.ndarray
    loss: int = LossKind.SQUARED
    k: int = 1
    M: float = 1.0
    lambda2: float = 1.0

    def __post_init__(self):
        self.X = np.asfortranarray(self.X, dtype=np.float64)
        self.y = np.ascontiguousarray(self.y, dtype=np.float64)

    def n(self) -> int:
        return int(self.X.shape[0])

    def p(self) -> int:
        return int(self.X.shape[1])

    def xflat(self) -> np.ndarray:
        return self.X.ravel(order="F")


@dataclass
class GeneratorSpec:
    """problem.hpp:53-63."""
    n: int = 0
    p: int = 0
    k: int = 1
    correlation: float = 0.0
    loss: int = LossKind.SQUARED
    snr: float = 5.0
    seed: int = 0
    M: float = 2.0
    lambda2: float = 1.0


@dataclass
class NodeState:
    """node_model.hpp:22-37."""
    fixed_zero: List[int] = field(default_factory=list)
    fixed_one: List[int] = field(default_factory=list)
    warm_start: Optional[np.ndarray] = None
    lower_bound: float = -math.inf
    depth: int = 0

    def p(self) -> int:
        return len(self.warm_start)

    def reduced_budget(self, k: int) -> int:
        return k - len(self.fixed_one)

    def is_leaf(self, k: int) -> bool:
        return self.reduced_budget(k) <= 0 or len(self.fixed_zero) + len(self.fixed_one) >= self.p()

    def states(self) -> np.ndarray:
        st = np.zeros(self.p(), dtype=np.uint8)
        st[list(self.fixed_zero)] = CoordState.FIXED_ZERO
        st[list(self.fixed_one)] = CoordState.FIXED_ONE
        return st


def root_node(p: int, k: int) -> NodeState:
    """node_model.hpp:47-52."""
    if p < 1 or k < 1 or k > p:
        raise InputError("root_node: need 1 <= k <= p")
    return NodeState(warm_start=np.zeros(p))


@dataclass
class RelaxConfig:
    """relaxation.hpp:26-33."""
    max_iterations: int = 2000
    gap_tolerance: float = 1e-6
    check_interval: int = 10
    acceleration: bool = True
    smoothness: float = 0.0
    workers: int = 1

    def to_c(self) -> _L.RelaxCfgC:
        return _L.RelaxCfgC(self.max_iterations, self.gap_tolerance, self.check_interval,
                            int(self.acceleration), self.smoothness, self.workers)


@dataclass
class SolverConfig:
    """bnb_engine.hpp:28-36."""
    batch_size: int = 0
    memory_budget: int = 1 << 30
    time_limit: float = math.inf
    prune_slack: float = 1e-6
    relax: RelaxConfig = field(default_factory=RelaxConfig)
    profile: bool = False
    workers: int = 1

    def to_c(self) -> _L.SolverCfgC:
        return _L.SolverCfgC(self.batch_size, self.memory_budget, self.time_limit,
                             self.prune_slack, self.relax.to_c(), int(self.profile), self.workers)


@dataclass
class ComponentProfile:
    """bnb_engine.hpp:40-46."""
    lower_bound_seconds: float = 0.0
    reoptimization_seconds: float = 0.0
    transfer_seconds: float = 0.0
    branch_generate_seconds: float = 0.0
    total_seconds: float = 0.0


@dataclass
class Certificate:
    """bnb_engine.hpp:48-60 (+ device counters)."""
    optimal_value: float
    support: List[int]
    coefficients: np.ndarray
    gap_percent: float
    lower_bound: float
    nodes_processed: int
    lb_batches: int
    reopt_batches: int
    batch_size_used: int
    profile: ComponentProfile
    status: str
    relax_iterations: int = 0
    node_iterations: int = 0
    reopt_supports: int = 0


@dataclass
class DebugHooks:
    """bnb_engine.hpp:63-66.  on_dual_bound(node, psi) gets a NodeState with
    fixed_zero / fixed_one only (no warm start)."""
    on_dual_bound: Optional[Callable[[NodeState, float], None]] = None
    on_batch_boundary: Optional[Callable[[float, float], None]] = None


@dataclass
class RashomonConfig:
    """rashomon.hpp:26-29."""
    epsilon: float = 0.0
    cap: int = -1


@dataclass
class RashomonResult:
    certificate: Certificate
    pool: List[Tuple[List[int], np.ndarray, float]]  # (sequence, coefficients, objective)


@dataclass
class RelaxationResult:
    """relaxation.hpp:149-154."""
    beta: np.ndarray  # p x m
    bounds: np.ndarray
    status: np.ndarray
    iterations: np.ndarray


@dataclass
class ReoptResult:
    """primal_heuristics.hpp:165-168."""
    coefficients: List[np.ndarray]
    objectives: List[float]


def validate(inst: ProblemInstance) -> None:
    _check(_L.lib().bnbg_validate(inst.xflat(), inst.y, inst.n(), inst.p(), inst.loss, inst.k,
                                  inst.M, inst.lambda2))


def generate_synthetic(spec: GeneratorSpec) -> Tuple[ProblemInstance, List[int]]:
    """problem.hpp:70-132; returns (instance, true_support)."""
    n, p = spec.n, spec.p
    X = np.zeros(max(n * p, 1), dtype=np.float64)
    y = np.zeros(max(n, 1), dtype=np.float64)
    sup = np.zeros(max(spec.k, 1), dtype=np.int32)
    _check(_L.lib().bnbg_generate_synthetic(n, p, spec.k, spec.correlation, spec.loss, spec.snr,
                                            spec.seed, X, y, sup))
    inst = ProblemInstance(X[: n * p].reshape(p, n).T, y[:n], spec.loss, spec.k, spec.M,
                           spec.lambda2)
    validate(inst)
    return inst, sup.tolist()


def auto_batch_size(memory_budget: int, n: int, p: int, k: int, kind: int) -> int:
    r = _L.lib().bnbg_auto_batch_size(memory_budget, n, p, k, kind)
    if r < 0:
        raise InputError("auto_batch_size: budget must be positive")
    return r


def _cert_from_c(cc: _L.CertC, sup, coef) -> Certificate:
    L = cc.support_len
    return Certificate(
        optimal_value=cc.optimal_value, support=[int(sup[t]) for t in range(L)],
        coefficients=np.array([coef[t] for t in range(L)]), gap_percent=cc.gap_percent,
        lower_bound=cc.lower_bound, nodes_processed=cc.nodes_processed,
        lb_batches=cc.lb_batches, reopt_batches=cc.reopt_batches,
        batch_size_used=cc.batch_size_used,
        profile=ComponentProfile(cc.lower_bound_seconds, cc.reoptimization_seconds,
                                 cc.transfer_seconds, cc.branch_generate_seconds,
                                 cc.total_seconds),
        status="optimal" if cc.status == 0 else "time_limit",
        relax_iterations=cc.relax_iterations, node_iterations=cc.node_iterations,
        reopt_supports=cc.reopt_supports)


def _col_arrays(states: np.ndarray, kbar: Sequence[int]):
    st = np.ascontiguousarray(np.asarray(states, dtype=np.uint8).T)  # m x p, row = column
    kb = np.ascontiguousarray(np.asarray(kbar, dtype=np.int32))
    return st, kb


class Engine:
    """One GPU's copy of an instance (the C-ABI handle, include/bnbg.h).

    X and y are uploaded once; every method below runs on the device.
    """

    def __init__(self, inst: ProblemInstance, device: int = 0, smoothness: float = 0.0):
        self.inst = inst
        h = C.c_void_p()
        _check(_L.lib().bnbg_create(inst.xflat(), inst.y, inst.n(), inst.p(), inst.loss, inst.k,
                                    inst.M, inst.lambda2, smoothness, device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _L.lib().bnbg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def smoothness(self) -> float:
        return _L.lib().bnbg_smoothness(self._h)

    def kernel_launches(self) -> int:
        return _L.lib().bnbg_kernel_launches(self._h)

    def set_timing(self, on: bool):
        _L.lib().bnbg_set_timing(self._h, int(on))

    KERNEL_CLASSES = ("gemm_xv", "gemm_xtr", "prox_fista", "eval", "reopt", "pass")

    def kernel_stats(self):
        """{class: (ms, flops, launches)} -- ms only while timing is enabled."""
        out = {}
        for kc, name in enumerate(self.KERNEL_CLASSES):
            ms, fl, ln = C.c_double(), C.c_double(), C.c_longlong()
            _L.lib().bnbg_kernel_stats(self._h, kc, C.byref(ms), C.byref(fl), C.byref(ln))
            out[name] = (ms.value, fl.value, ln.value)
        return out

    PASS_PHASES = ("xv", "xtr", "prox", "eval_xb", "eval_xtz", "eval_cols", "compact")

    def pass_profile(self):
        """{phase: ms} of the persistent pass kernel (needs BNBG_PASS_PROF=1 at create)."""
        buf = np.zeros(16)
        c = _L.lib().bnbg_pass_profile(self._h, buf, len(buf))
        out = {nm: buf[i] / 1e6 for i, nm in enumerate(self.PASS_PHASES) if i < c}
        out.update({nm + "_work": buf[8 + i] / 1e6 for i, nm in enumerate(self.PASS_PHASES)
                    if 8 + i < c})
        return out

    def pass_profile_raw(self):
        """The raw 32-slot profile buffer in ns (see bnbg_pass_profile)."""
        buf = np.zeros(32)
        _L.lib().bnbg_pass_profile(self._h, buf, len(buf))
        return buf

    def shard_stats(self):
        """Last sharded solve on this engine: {"sent", "received", "batch_per_pass"}."""
        cap = 1 << 16
        buf = (C.c_longlong * cap)()
        cnt = _L.lib().bnbg_shard_stats(self._h, buf, cap)
        vals = list(buf[:min(cnt, cap)])
        return {"sent": vals[0], "received": vals[1], "batch_per_pass": vals[3:]}

    def transfer_bytes(self):
        a, b = C.c_longlong(), C.c_longlong()
        _L.lib().bnbg_transfer_bytes(self._h, C.byref(a), C.byref(b))
        return a.value, b.value

    def gemm_stats(self):
        ms, fl, ln = C.c_double(), C.c_double(), C.c_longlong()
        _L.lib().bnbg_gemm_stats(self._h, C.byref(ms), C.byref(fl), C.byref(ln))
        return ms.value, fl.value, ln.value

    # -- relaxation.hpp:163-255 ------------------------------------------
    def solve_batch_relaxation(self, batch, config: Optional[RelaxConfig] = None,
                               prune_threshold: float = math.inf,
                               dual_trace: Optional[Callable[[int, float], None]] = None
                               ) -> RelaxationResult:
        """``batch`` is a list of NodeState, or a tuple (states p x m, kbar, warm p x m)."""
        if isinstance(batch, tuple):
            states, kbar, warm = batch
        else:
            if len(batch) == 0:
                raise InputError("solve_batch_relaxation: empty batch")
            k = self.inst.k
            states = np.stack([nd.states() for nd in batch], axis=1)
            kbar = [max(0, nd.reduced_budget(k)) for nd in batch]
            warm = np.stack([np.asarray(nd.warm_start, dtype=np.float64) for nd in batch], axis=1)
        p = self.inst.p()
        warm = np.asarray(warm, dtype=np.float64)
        m = warm.shape[1] if warm.ndim == 2 else 0
        if m == 0:
            raise InputError("solve_batch_relaxation: empty batch")
        st, kb = _col_arrays(states, kbar)
        wm = np.ascontiguousarray(warm.T)
        beta = np.zeros((m, p))
        bounds = np.zeros(m)
        status = np.zeros(m, dtype=np.int32)
        iters = np.zeros(m, dtype=np.int32)
        cfg = (config or RelaxConfig()).to_c()
        cb = _L.TRACE_FN(lambda _u, b, psi: dual_trace(b, psi)) if dual_trace else _L.TRACE_FN()
        _check(_L.lib().bnbg_relax_batch(self._h, C.byref(cfg), m, st.ravel(), kb, wm.ravel(),
                                         prune_threshold, beta.ravel(), bounds, status, iters, cb,
                                         None), self._h)
        return RelaxationResult(beta.T.copy(), bounds, status, iters)

    # -- primal_heuristics.hpp:134-163 ----------------------------------------
    # -- prox_kernel.hpp:52-90 BatchMeta::from_nodes (the device packer) -------
    def pack_batch(self, nodes: Sequence[NodeState]):
        """Returns (state p x m uint8 CoordState, reduced_budget[m], free_count[m])
        as built on the device by the packer (VK1)."""
        m, p = len(nodes), self.inst.p()
        if m == 0:
            raise InputError("batch meta: empty batch")

        def csr(lists):
            off = np.zeros(m + 1, dtype=np.int32)
            for b, lst in enumerate(lists):
                off[b + 1] = off[b] + len(lst)
            idx = np.ascontiguousarray([j for lst in lists for j in lst] or [0], dtype=np.int32)
            return off, idx

        z_off, z_idx = csr([nd.fixed_zero for nd in nodes])
        o_off, o_idx = csr([nd.fixed_one for nd in nodes])
        state = np.zeros(p * m, dtype=np.uint8)
        kbar = np.zeros(m, dtype=np.int32)
        free = np.zeros(m, dtype=np.int32)
        _check(_L.lib().bnbg_pack_batch(self._h, m, z_off, z_idx, o_off, o_idx, state, kbar, free),
               self._h)
        return state.reshape(m, p).T.copy(), kbar.tolist(), free.tolist()

    def round_support_batch(self, beta: np.ndarray, nodes: Sequence[NodeState]) -> List[List[int]]:
        p, m = beta.shape
        k = self.inst.k
        states = np.stack([nd.states() for nd in nodes], axis=1)
        kb = [max(0, nd.reduced_budget(k)) for nd in nodes]
        off = np.zeros(m + 1, dtype=np.int32)
        for b, nd in enumerate(nodes):
            off[b + 1] = off[b] + len(nd.fixed_one)
        idx = np.ascontiguousarray([j for nd in nodes for j in nd.fixed_one] or [0], dtype=np.int32)
        st, kbc = _col_arrays(states, kb)
        sup = np.zeros(m * max(k, 1), dtype=np.int32)
        ln = np.zeros(m, dtype=np.int32)
        _check(_L.lib().bnbg_round_support(self._h, m, np.ascontiguousarray(beta.T).ravel(),
                                           st.ravel(), kbc, off, idx, sup, ln), self._h)
        return [sup[b * k: b * k + ln[b]].tolist() for b in range(m)]

    def round_support(self, beta: np.ndarray, node: NodeState, k: Optional[int] = None):
        return self.round_support_batch(np.asarray(beta, dtype=np.float64)[:, None], [node])[0]

    def select_branch_variable_batch(self, beta: np.ndarray, nodes: Sequence[NodeState]):
        p, m = beta.shape
        states = np.stack([nd.states() for nd in nodes], axis=1)
        st, _ = _col_arrays(states, [0] * m)
        j = np.zeros(m, dtype=np.int32)
        _check(_L.lib().bnbg_select_branch(self._h, m, np.ascontiguousarray(beta.T).ravel(),
                                           st.ravel(), j), self._h)
        if (j < 0).any():
            raise LogicError("select_branch_variable: no free coordinate")
        return j.tolist()

    def select_branch_variable(self, beta: np.ndarray, node: NodeState) -> int:
        return self.select_branch_variable_batch(np.asarray(beta, dtype=np.float64)[:, None],
                                                 [node])[0]

    # -- primal_heuristics.hpp:174-227 ------------------------------------------
    def reoptimize_supports(self, supports: Sequence[Sequence[int]]) -> ReoptResult:
        ns = len(supports)
        if ns == 0:
            return ReoptResult([], [])
        off = np.zeros(ns + 1, dtype=np.int32)
        for t, s in enumerate(supports):
            off[t + 1] = off[t] + len(s)
        idx = np.ascontiguousarray([j for s in supports for j in s] or [0], dtype=np.int32)
        coef = np.zeros(max(1, int(off[-1])))
        obj = np.zeros(ns)
        _check(_L.lib().bnbg_reoptimize(self._h, ns, off, idx, coef, obj), self._h)
        return ReoptResult([coef[off[t]:off[t + 1]].copy() for t in range(ns)], obj.tolist())

    def gemm(self, B: np.ndarray, trans: bool) -> np.ndarray:
        """Probe of the DMMA contraction: X @ B (trans False) or X.T @ B."""
        K, m = B.shape
        out_rows = self.inst.p() if trans else self.inst.n()
        Cm = np.zeros((m, out_rows))
        _check(_L.lib().bnbg_gemm(self._h, int(trans), m, np.ascontiguousarray(B.T).ravel(),
                                  Cm.ravel()), self._h)
        return Cm.T.copy()

    # -- bnb_engine.hpp:299-309 -------------------------------------------------
    def solve(self, config: Optional[SolverConfig] = None,
              hooks: Optional[DebugHooks] = None) -> Certificate:
        cfg = (config or SolverConfig()).to_c()
        k = self.inst.k
        sup = (C.c_int32 * (k + 1))()
        coef = (C.c_double * (k + 1))()
        cc = _L.CertC()
        cc.support = C.cast(sup, C.POINTER(C.c_int32))
        cc.coefficients = C.cast(coef, C.POINTER(C.c_double))
        dh = _L.DUAL_HOOK()
        bh = _L.BOUNDARY_HOOK()
        if hooks and hooks.on_dual_bound:
            def _dh(_u, n0, j0, n1, j1, psi):
                hooks.on_dual_bound(NodeState([j0[t] for t in range(n0)],
                                              [j1[t] for t in range(n1)]), psi)
            dh = _L.DUAL_HOOK(_dh)
        if hooks and hooks.on_batch_boundary:
            bh = _L.BOUNDARY_HOOK(lambda _u, lb, ub: hooks.on_batch_boundary(lb, ub))
        _check(_L.lib().bnbg_solve(self._h, C.byref(cfg), C.byref(cc), dh, bh, None), self._h)
        return _cert_from_c(cc, sup, coef)

    # -- device-resident node pool, per pass (include/bnbg.h bnbg_pool_*) -------
    def pool_root(self, slot: int = 0):
        """root_node (node_model.hpp:47-52) into pool `slot`."""
        _check(_L.lib().bnbg_pool_root(self._h, slot), self._h)

    def pool_relax(self, slots, prune_threshold: float = math.inf,
                   config: Optional[RelaxConfig] = None):
        """Lower bounds + rounding + branch variable of the nodes in `slots`
        (relaxation.hpp:163-255).  Returns (bounds, status, iterations,
        supports) with supports in construction order (J1 ++ top-kbar free)."""
        sl = np.ascontiguousarray(np.asarray(slots, dtype=np.int32))
        m, k = len(sl), max(self.inst.k, 1)
        cfg = (config or RelaxConfig()).to_c()
        bd, st, it = np.zeros(m), np.zeros(m, np.int32), np.zeros(m, np.int32)
        sup, ln = np.zeros(m * k, np.int32), np.zeros(m, np.int32)
        _check(_L.lib().bnbg_pool_relax(self._h, C.byref(cfg), m, sl, prune_threshold, bd, st, it,
                                        sup, ln), self._h)
        rows = [sup[b * k: b * k + ln[b]].tolist() for b in range(m)]
        return bd, st, it, rows

    def pool_branch(self, lb, post_threshold: float, free_slots):
        """Prune test + branch of the last pool_relax batch (bnb_engine.hpp:242-256).
        Returns one (slot, is_leaf, fixed_one, depth, lower_bound) per child."""
        lb = np.ascontiguousarray(np.asarray(lb, dtype=np.float64))
        fs = np.ascontiguousarray(np.asarray(free_slots, dtype=np.int32))
        m, k = len(lb), max(self.inst.k, 1)
        rec = np.zeros(2 * m * (4 + k), np.int32)
        clb = np.zeros(2 * m)
        surv = C.c_int32()
        _check(_L.lib().bnbg_pool_branch(self._h, m, lb, post_threshold, fs, C.byref(surv), rec,
                                         clb), self._h)
        out = []
        for c in range(2 * surv.value):
            r = rec[c * (4 + k):(c + 1) * (4 + k)]
            out.append((int(r[0]), bool(r[1]), r[4:4 + r[2]].tolist(), int(r[3]), float(clb[c])))
        return out

    # -- node-sharded solve over ranks (include/bnbg.h) ------------
    def solve_sharded(self, config: Optional[SolverConfig] = None, group=None,
                      transport: Optional[str] = None) -> Certificate:
        """Certified solve with the open nodes sharded over the ranks of a
        torch.distributed group (one process and one Engine per GPU, X and y
        replicated).  transport "nccl": the engine's own NCCL communicator
        (device-to-device node exchange; the default when the group's backend
        is NCCL); "host": node records staged through host memory over the
        group (gloo) -- for CPU-driven tests and several ranks on one GPU."""
        from . import sharded
        return sharded.solve_sharded(self, config, group, transport)

    # -- rashomon.hpp:149-218 ---------------------------------------------------
    def collect_rashomon(self, config: Optional[SolverConfig] = None,
                         rconfig: Optional[RashomonConfig] = None) -> RashomonResult:
        cfg = (config or SolverConfig()).to_c()
        rc = rconfig or RashomonConfig()
        k = self.inst.k
        sup = (C.c_int32 * (k + 1))()
        coef = (C.c_double * (k + 1))()
        cc = _L.CertC()
        cc.support = C.cast(sup, C.POINTER(C.c_int32))
        cc.coefficients = C.cast(coef, C.POINTER(C.c_double))
        pool = C.c_void_p()
        _check(_L.lib().bnbg_collect_rashomon(self._h, C.byref(cfg), rc.epsilon, rc.cap,
                                              C.byref(cc), C.byref(pool)), self._h)
        recs = []
        try:
            seq = np.zeros(k + 1, dtype=np.int32)
            cf = np.zeros(k + 1)
            ob = C.c_double()
            for t in range(_L.lib().bnbg_pool_size(pool)):
                ln = _L.lib().bnbg_pool_record(pool, t, seq, cf, C.byref(ob))
                recs.append((seq[:ln].tolist(), cf[:ln].copy(), ob.value))
        finally:
            _L.lib().bnbg_pool_free(pool)
        return RashomonResult(_cert_from_c(cc, sup, coef), recs)


def balance_plan(counts) -> Optional[np.ndarray]:
    """The sharded solve's deterministic load-balancing plan: queue sizes per
    rank -> moves[donor, receiver], or None when nothing moves."""
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
    w = len(c)
    mv = np.zeros(w * w, dtype=np.int64)
    moved = _L.lib().bnbg_balance_plan(w, c, mv)
    return mv.reshape(w, w) if moved else None


def smoothness_constant(kind: int, X: np.ndarray, device: int = 0) -> float:
    """losses.hpp:86-112 (power iteration on the device)."""
    X = np.asfortranarray(X, dtype=np.float64)
    if X.size == 0:
        raise InputError("smoothness_constant: empty matrix")
    n, p = X.shape
    y = np.ones(n) if kind == LossKind.LOGISTIC else np.zeros(n)
    with Engine(ProblemInstance(X, y, kind, 1, 1.0, 1.0), device) as eng:
        return eng.smoothness()


def solve(inst: ProblemInstance, config: Optional[SolverConfig] = None,
          hooks: Optional[DebugHooks] = None, device: int = 0) -> Certificate:
    """bnb_engine.hpp:299-309: certified solve; uploads the instance, runs the
    BnB loop with device node processing, returns the certificate."""
    cfg = config or SolverConfig()
    with Engine(inst, device, cfg.relax.smoothness) as eng:
        return eng.solve(cfg, hooks)


def solve_sharded(inst: ProblemInstance, config: Optional[SolverConfig] = None, group=None,
                  transport: Optional[str] = None, device: Optional[int] = None) -> Certificate:
    """Node-sharded certified solve: one process per GPU in a torch.distributed
    group, X and y replicated, open nodes dealt over the ranks (include/bnbg.h
    bnbg_solve_sharded).  device defaults to the current CUDA device."""
    cfg = config or SolverConfig()
    if device is None:
        import torch
        device = torch.cuda.current_device()
    with Engine(inst, device, cfg.relax.smoothness) as eng:
        return eng.solve_sharded(cfg, group, transport)


def collect_rashomon(inst: ProblemInstance, config: Optional[SolverConfig] = None,
                     rconfig: Optional[RashomonConfig] = None, device: int = 0) -> RashomonResult:
    cfg = config or SolverConfig()
    with Engine(inst, device, cfg.relax.smoothness) as eng:
        return eng.collect_rashomon(cfg, rconfig)


def prox_step(U: np.ndarray, eta: float, lambda2: float, states: np.ndarray, kbar, M: float,
              device: int = 0) -> np.ndarray:
    """prox_kernel.hpp:284-301 (U, states: p x m)."""
    U = np.asarray(U, dtype=np.float64)
    p, m = U.shape
    st, kb = _col_arrays(states, kbar)
    out = np.zeros((m, p))
    _check(_L.lib().bnbg_prox_step(device, p, m, np.ascontiguousarray(U.T).ravel(), eta, lambda2,
                                   st.ravel(), kb, M, out.ravel()))
    return out.T.copy()


def batched_conjugate_prox(U_scaled: np.ndarray, states: np.ndarray, kbar, weight: float,
                           M: float, device: int = 0) -> np.ndarray:
    """prox_kernel.hpp:214-229."""
    U = np.asarray(U_scaled, dtype=np.float64)
    p, m = U.shape
    st, kb = _col_arrays(states, kbar)
    out = np.zeros((m, p))
    _check(_L.lib().bnbg_conjugate_prox(device, p, m, np.ascontiguousarray(U.T).ravel(), weight,
                                        st.ravel(), kb, M, out.ravel()))
    return out.T.copy()


def g_value(beta: np.ndarray, states: np.ndarray, kbar, M: float, device: int = 0) -> np.ndarray:
    """prox_kernel.hpp:310-347 per column (beta p x m)."""
    B = np.asarray(beta, dtype=np.float64)
    if B.ndim == 1:
        B = B[:, None]
        states = np.asarray(states).reshape(-1, 1)
        kbar = [kbar] if np.isscalar(kbar) else kbar
    p, m = B.shape
    st, kb = _col_arrays(states, kbar)
    out = np.zeros(m)
    _check(_L.lib().bnbg_g_value(device, p, m, np.ascontiguousarray(B.T).ravel(), st.ravel(), kb,
                                 M, out))
    return out


def g_conjugate_value(q: np.ndarray, states: np.ndarray, kbar, M: float,
                      device: int = 0) -> np.ndarray:
    """prox_kernel.hpp:351-370 per column (q p x m)."""
    Q = np.asarray(q, dtype=np.float64)
    if Q.ndim == 1:
        Q = Q[:, None]
        states = np.asarray(states).reshape(-1, 1)
        kbar = [kbar] if np.isscalar(kbar) else kbar
    p, m = Q.shape
    st, kb = _col_arrays(states, kbar)
    out = np.zeros(m)
    _check(_L.lib().bnbg_g_conjugate(device, p, m, np.ascontiguousarray(Q.T).ravel(), st.ravel(),
                                     kb, M, out))
    return out
