"""The node-sharded solve on the device: several ranks certify
the same support and objective as the single-GPU solve.  The box has one GPU,
so the multi-rank runs share it over the host transport (gloo); the NCCL
transport runs at world size 1 (the same code path, trivial exchange)."""
import pytest

from tests.test_sharded_cpu import run_ranks

pytestmark = pytest.mark.gpu

REL = 1e-6


@pytest.mark.parametrize("loss,n,p,k,rho,seed,batch", [(0, 300, 60, 5, 0.8, 2, 4),
                                                       (1, 400, 80, 6, 0.7, 1, 8)])
def test_sharded_host_transport_matches_single(bnb, loss, n, p, k, rho, seed, batch):
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss,
                                                       seed=seed))
    ref = bnb.solve(inst, bnb.SolverConfig(batch_size=batch))
    for nproc in (2, 3):
        res = run_ranks(nproc, "host", n, p, k, rho, loss, seed, batch)
        for d in res:
            assert d["status"] == "optimal"
            assert d["support"] == ref.support
            assert abs(d["value"] - ref.optimal_value) <= REL * abs(ref.optimal_value)
        assert len({d["nodes"] for d in res}) == 1  # every rank reports the global count


def test_sharded_nccl_world1(bnb):
    n, p, k, rho, loss, seed = 300, 60, 5, 0.8, 1, 4
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss,
                                                       seed=seed))
    ref = bnb.solve(inst)
    (d,) = run_ranks(1, "nccl", n, p, k, rho, loss, seed)
    assert d["support"] == ref.support and d["status"] == "optimal"
    assert abs(d["value"] - ref.optimal_value) <= REL * abs(ref.optimal_value)
    assert d["nodes"] == ref.nodes_processed  # one rank: the same search
