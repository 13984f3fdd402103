import sys, math
sys.path.insert(0, '.')
import numpy as np
import paper_2605_22188_b200 as bnb
from oracle import oracle as orc
from tests.test_gpu_kernels import _engine, rnd_batch
orc.build()
for p in (4000, 8200):
    for loss in (0,):
        inst, eng = _engine(bnb, orc, 60, p, 2, 0.5, loss, seed=4)
        st = np.zeros((p, 1), dtype=np.uint8); kb = [2]; warm = np.zeros((p, 1))
        L = orc.smoothness(loss, inst.X)
        for its in (40, 100, 200, 400, 1000):
            tr_d, tr_o = [], []
            res = eng.solve_batch_relaxation((st, kb, warm), bnb.RelaxConfig(smoothness=L, max_iterations=its), math.inf,
                                             dual_trace=lambda b, v: tr_d.append(v))
            ob, obnd, ost, oit = orc.relax_batch(inst, st, kb, warm, math.inf, orc.relax_cfg(smoothness=L, max_iterations=its),
                                                 trace=lambda b, v: tr_o.append(v))
            d = np.abs(np.array(tr_d[:len(tr_o)]) - np.array(tr_o[:len(tr_d)]))
            first = int(np.argmax(d > 1e-6)) if (d > 1e-6).any() else -1
            print(p, loss, its, 'bounds', res.bounds[0], obnd[0], 'iters', res.iterations[0], oit[0], 'beta diff', np.abs(res.beta - ob).max(), 'first trace diff at eval', first, 'of', len(tr_o), flush=True)
