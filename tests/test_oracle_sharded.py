"""The patch-sharded oracle (oracle/sharded.py, used for the full-size C5 dump) computes the same
numbers as oracle/ieti.py: bitwise with the same primal-basis route, and the PCG basis route
(SURVEY O8 A-route) equals the KKT-LU basis of Eq. (6) to 1e-11."""
import numpy as np
import pytest

from oracle.ieti import IetiOracle
from oracle.sharded import ShardedIetiOracle
from workloads import make_workload


@pytest.mark.parametrize("name,kw", [("C5", dict(m=4, grid=(3, 2, 2))), ("C4", dict(m=4, grid=(2, 2, 3))),
                                     ("C3", dict(m=8, grid=(3, 2)))])
def test_sharded_equals_single_process(name, kw):
    wl = make_workload(name, **kw)
    ref = IetiOracle(wl)
    a = ref.solve(tol=1e-8)
    sh = ShardedIetiOracle(wl, workers=3, basis="kkt", topo=ref.topo)
    try:
        b = sh.solve(tol=1e-8)
        assert a.iters == b.iters
        assert all(np.array_equal(x, y) for x, y in zip(a.u, b.u))
        assert np.array_equal(a.lam, b.lam) and a.history == b.history
    finally:
        sh.close()


@pytest.mark.parametrize("name,kw", [("C5", dict(m=4, grid=(3, 2, 2))), ("C4", dict(m=4, grid=(2, 2, 3)))])
def test_pcg_primal_basis_route_equals_kkt(name, kw):
    wl = make_workload(name, **kw)
    kkt = IetiOracle(wl)
    pcg = IetiOracle(wl, basis="pcg", topo=kkt.topo)
    T = kkt.topo
    for k in range(T.n_patches):
        P1, P2 = kkt.Phi[k], pcg.Phi[k]
        assert np.abs(P1 - P2).max() <= 1e-11 * np.abs(P1).max(), k
        # Eq. (6) directly: C Phibar = I; Phibar^T K v = 0 for v in ker C
        C = T.C[k].toarray()
        assert np.allclose(C @ P2, np.eye(C.shape[0]), atol=1e-12)
        v = np.random.default_rng(k).standard_normal(P2.shape[0])
        v -= C.T @ np.linalg.solve(C @ C.T, C @ v)
        assert abs(P2.T @ (kkt.K[k] @ v)).max() <= 1e-10 * np.abs(kkt.K[k] @ v).max()
    assert np.abs(kkt.S_PiPi - pcg.S_PiPi).max() <= 1e-11 * np.abs(kkt.S_PiPi).max()
