"""The exported per-pass pool API (include/bnbg.h bnbg_pool_*): run_bnb's
node-processing body (bnb_engine.hpp:151-265) written by a caller over
(bound, sequence, slot) reproduces bnbg_solve exactly."""
import heapq
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def caller_loop(eng, inst, batch_size, slack=1e-6):
    def thr(ub):
        return math.inf if not math.isfinite(ub) else ub - slack * max(1.0, abs(ub))

    free, nxt = [], [0]

    def take():
        if free:
            return free.pop()
        nxt[0] += 1
        return nxt[0] - 1

    heap, seq = [], 0
    root = take()
    eng.pool_root(root)
    heapq.heappush(heap, (-math.inf, seq, root))
    seq += 1
    pending, inc, inc_sup, nodes, passes = [], math.inf, [], 0, 0
    while heap or pending:
        t = thr(inc)
        batch, lbs, popped, disc = [], [], 0, 0
        while heap and popped < batch_size:          # assemble_batch (node_model.hpp:158-172)
            lb, _, s = heapq.heappop(heap)
            if lb >= t:
                disc += 1
                free.append(s)
                continue
            batch.append(s)
            lbs.append(lb)
            popped += 1
        nodes += popped + disc + len(pending)
        leaves = [(lb, j1) for lb, j1 in pending if lb < t]
        pending = []
        if not batch and not leaves:
            continue
        supports, status = [j1 for _, j1 in leaves], None
        if batch:
            passes += 1
            bd, status, _, rows = eng.pool_relax(batch, t)
            supports += [rows[b] for b in range(len(batch)) if status[b] != 0]
        if supports:
            r = eng.reoptimize_supports(supports)
            for sq, cf, ob in zip(supports, r.coefficients, r.objectives):
                if ob < inc:
                    inc, inc_sup = ob, sorted(sq)
        post = thr(inc)
        if batch:
            fs = [take() for _ in range(2 * len(batch))]
            kids = eng.pool_branch(lbs, post, fs)
            for s in reversed(fs[2 * (len(kids) // 2):]):
                free.append(s)
            for slot, leaf, j1, _, lb in kids:
                if leaf:
                    pending.append((lb, j1))
                    free.append(slot)
                else:
                    heapq.heappush(heap, (lb, seq, slot))
                    seq += 1
            free.extend(batch)
    return inc, inc_sup, nodes, passes


@pytest.mark.parametrize("loss,n,p,k,rho,seed,batch", [(0, 300, 60, 5, 0.8, 2, 4),
                                                       (1, 400, 80, 6, 0.7, 1, 8),
                                                       (1, 200, 40, 4, 0.8, 7, 16)])
def test_caller_loop_over_pool_api_equals_solve(bnb, loss, n, p, k, rho, seed, batch):
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss,
                                                       seed=seed))
    with bnb.Engine(inst) as eng:
        ref = eng.solve(bnb.SolverConfig(batch_size=batch))
        inc, sup, nodes, passes = caller_loop(eng, inst, batch)
    assert sup == ref.support
    assert inc == ref.optimal_value
    assert nodes == ref.nodes_processed and passes == ref.lb_batches


def test_pool_api_errors(bnb):
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=50, p=10, k=3, seed=0))
    with bnb.Engine(inst) as eng:
        eng.pool_root(0)
        with pytest.raises(bnb.InputError):
            eng.pool_relax([], math.inf)
        with pytest.raises(bnb.InputError):
            eng.pool_relax([10 ** 6], math.inf)
        eng.pool_relax([0], math.inf)
        with pytest.raises(bnb.InputError):
            eng.pool_branch([0.0, 0.0], math.inf, [1, 2, 3, 4])  # batch size mismatch
