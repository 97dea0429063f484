"""GPU brick-wall layers (paper_2301_12814_b200.mps: Θ + SVD per gate through the C ABI) against the
pinned layer oracle (oracle/layer.py, itself pinned to dense state-vector evolution): bond charges
exact, Schmidt values λ ≤ 1e-10 relative after every layer (unique despite the per-bond phase gauge),
and the phase-free dense state for small M."""
import numpy as np
import pytest

import oracle.layer as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


@pytest.mark.parametrize("M,N,d,chi,chi_max,seed", [(5, 3, 4, 10, 10 ** 6, 0), (6, 3, 4, 12, 8, 1),
                                                    (6, 4, 3, 16, 12, 2)])
def test_layers_match_oracle(tn, M, N, d, chi, chi_max, seed):
    from paper_2301_12814_b200.mps import MPS
    st = L.random_mps(M, N, d, chi, seed)
    ref = L.copy_state(st)
    mps = MPS.from_state(st)
    rng = np.random.default_rng(seed + 100)
    for parity in (0, 1, 0, 1):
        gates = list(range(parity, M - 1, 2))
        th, ph = rng.uniform(0, np.pi / 2, len(gates)), rng.uniform(0, 2 * np.pi, len(gates))
        d_ref = L.apply_layer(ref, parity, th, ph, chi_max)
        d_gpu = mps.apply_layer(parity, th, ph, chi_max)
        got = mps.to_state()
        for b in range(M + 1):
            assert np.array_equal(got["q"][b], ref["q"][b]), (parity, b)
            assert np.max(np.abs(got["lam"][b] - ref["lam"][b]), initial=0.0) <= 1e-10 * ref["lam"][b].max(), (parity, b)
        for x, y in zip(d_gpu, d_ref):
            assert abs(x - y) <= 1e-10 * max(y, 1e-30) + 1e-28
    psi_ref, psi = L.dense_state(ref), L.dense_state(got)
    assert np.linalg.norm(psi - psi_ref) <= 1e-10 * np.linalg.norm(psi_ref)
