"""GPU brick-wall layers (paper_2301_12814_b200.mps: Θ + SVD per gate through the C ABI, right-canonical update)
against the pinned layer oracle (oracle/layer.py in form "b", itself pinned to dense state-vector evolution):
bond charges exact, Schmidt values λ ≤ 1e-10 relative after every layer (unique despite the per-bond phase gauge),
and the phase-free dense state for small M — at SPEC.md's cutoff 1e-14 for MPS and MPO layers alike."""
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
    ref = L.to_bform(st)
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


# ------------------------------------------------------------------ MPO (vectorized density matrix) layers
# every SVD algorithm: the no-truncation case produces small rank-deficient sectors on which cuSOLVER's
# polar-decomposition SVD reports h_err_sigma up to 5e-8 — both Xgesvdp uses fall back to Jacobi there
@pytest.mark.parametrize("algo", ["gram", "gesvdp", "gesvdj"])
@pytest.mark.parametrize("M,N,d,chi,chi_max,seed", [(4, 2, 3, 6, 10 ** 6, 0), (5, 2, 3, 8, 10, 1), (4, 3, 3, 9, 14, 2)])
def test_mpo_layers_match_oracle(tn, M, N, d, chi, chi_max, seed, algo, monkeypatch):
    monkeypatch.setenv("TN_SVD_ALGO", algo)
    from paper_2301_12814_b200.mps import MPO
    st = L.random_mpo(M, N, d, chi, seed)
    # unit-norm state, so the rounding noise of rank-deficient sectors (~ε‖Θ‖) sits far below SPEC.md's absolute
    # 1e-14 cutoff on both sides; the right-canonical update divides by no small λ, so no amplification either
    nrm = np.linalg.norm(L.dense_state2(st)) ** (1.0 / M)
    st["gam"] = [g / nrm for g in st["gam"]]
    ref = L.to_bform(st)
    mpo = MPO.from_state(st)
    rng = np.random.default_rng(seed + 200)
    # SPEC.md's 1e-14 for the default Gram/Ritz path and one-sided Jacobi; cuSOLVER's polar-decomposition SVD
    # (TN_SVD_ALGO=gesvdp, selectable) returns the exact zeros of rank-deficient sectors only to ~1e-13 absolute,
    # so at 1e-14 its noise values would be kept where the oracle's are not
    cut = 1e-12 if algo == "gesvdp" else 1e-14
    for parity in (0, 1, 0, 1):
        gates = list(range(parity, M - 1, 2))
        th, ph = rng.uniform(0, np.pi / 2, len(gates)), rng.uniform(0, 2 * np.pi, len(gates))
        d_ref = L.apply_layer2(ref, parity, th, ph, chi_max, cut)
        d_gpu = mpo.apply_layer(parity, th, ph, chi_max, cut)
        got = mpo.to_state()
        for b in range(M + 1):
            assert np.array_equal(got["q1"][b], ref["q1"][b]) and np.array_equal(got["q2"][b], ref["q2"][b]), (parity, b)
            assert np.max(np.abs(got["lam"][b] - ref["lam"][b]), initial=0.0) <= 1e-10 * ref["lam"][b].max(), (parity, b)
        for x, y in zip(d_gpu, d_ref):
            assert abs(x - y) <= 1e-10 * max(y, 1e-30) + 1e-16
    rho_ref, rho = L.dense_state2(ref), L.dense_state2(got)
    assert np.linalg.norm(rho - rho_ref) <= 1e-10 * np.linalg.norm(rho_ref)
