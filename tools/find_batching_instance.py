import sys, time
sys.path.insert(0, '.')
import paper_2605_22188_b200 as P
for (n, p, k, rho) in [(100, 60, 5, 0.9), (150, 80, 6, 0.9), (200, 100, 6, 0.9), (120, 100, 6, 0.8), (300, 300, 8, 0.9)]:
    inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=0, seed=0))
    with P.Engine(inst) as eng:
        eng.solve(P.SolverConfig(batch_size=256, time_limit=1.0))
        t = time.time(); c = eng.solve(P.SolverConfig(batch_size=256, time_limit=20)); t256 = time.time() - t
        t = time.time(); c1 = eng.solve(P.SolverConfig(batch_size=1, time_limit=20)); t1 = time.time() - t
    print(n, p, k, rho, "b256", c.status, c.nodes_processed, round(t256, 3), "b1", c1.status, c1.nodes_processed, round(t1, 3), flush=True)
