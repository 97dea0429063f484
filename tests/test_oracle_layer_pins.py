"""Pins of the brick-wall layer oracle (oracle/layer.py): without truncation, a layer of TEBD updates
(Θ of Eq. S5 + SVD + Vidal-form update) must reproduce the DENSE evolution of the state vector under the
same beam splitters, built independently from scipy expm of the two-mode generator (`-m "not gpu"`)."""
import itertools

import numpy as np
import pytest
import scipy.linalg

import oracle.layer as L


def _u4(theta, phi, d, N):
    D = N + 1
    a = np.diag(np.sqrt(np.arange(1, D)), 1)
    A, B = np.kron(a, np.eye(D)), np.kron(np.eye(D), a)
    G = theta * (np.exp(1j * phi) * A.conj().T @ B - np.exp(-1j * phi) * A @ B.conj().T)
    Uf = scipy.linalg.expm(G).reshape(D, D, D, D)
    U4 = np.zeros((d, d, d, d), dtype=np.complex128)
    m = min(d, D)
    for i, ip, j, jp in itertools.product(range(m), repeat=4):
        if i + ip == j + jp:
            U4[i, ip, j, jp] = Uf[i, ip, j, jp]
    return U4


@pytest.mark.parametrize("form", ["vidal", "b"])
@pytest.mark.parametrize("M,N,d,chi,seed", [(4, 2, 3, 4, 0), (5, 3, 3, 5, 1), (4, 3, 4, 6, 2), (5, 2, 2, 4, 3)])
def test_layer_without_truncation_is_dense_evolution(M, N, d, chi, seed, form):
    # both update forms of oracle/svd.py (Vidal; right-canonical B, Hastings) evolve the state exactly
    st = L.random_mps(M, N, d, chi, seed)
    if form == "b":
        st = L.to_bform(st)
    psi = L.dense_state(st)
    rng = np.random.default_rng(seed + 10)
    for parity in (0, 1, 0):
        gates = list(range(parity, M - 1, 2))
        th = rng.uniform(0, np.pi / 2, len(gates))
        ph = rng.uniform(0, 2 * np.pi, len(gates))
        disc = L.apply_layer(st, parity, th, ph, chi_max=10 ** 6)
        assert max(disc, default=0.0) < 1e-20
        for g, k in enumerate(gates):
            psi = L.dense_gate(psi, k, _u4(th[g], ph[g], d, N))
        got = L.dense_state(st)
        assert np.linalg.norm(got - psi) <= 1e-11 * np.linalg.norm(psi)


def test_truncation_reports_discarded_weight():
    st = L.random_mps(5, 3, 3, 6, 7)
    disc = L.apply_layer(st, 0, [0.6, 1.1], [0.3, 2.0], chi_max=3)
    assert sum(disc) > 0 and min(disc) >= 0
    assert all(len(st["lam"][k]) <= 3 for k in (1, 3))


# ------------------------------------------------------------------ MPO (vectorized density matrix) layers
def test_vectorized_pure_mpo_is_outer_product():
    st = L.random_mps(4, 2, 3, 4, 5)
    psi = L.dense_state(st)
    rho = L.dense_state2(L.vectorize_mps(st))
    assert np.allclose(rho, np.multiply.outer(psi, psi.conj()), rtol=0, atol=1e-13 * np.abs(psi).max() ** 2)


@pytest.mark.parametrize("form", ["vidal", "b"])
@pytest.mark.parametrize("M,N,d,chi,seed", [(4, 2, 3, 5, 0), (4, 3, 3, 6, 1), (3, 2, 3, 6, 2)])
def test_mpo_layer_without_truncation_is_dense_evolution(M, N, d, chi, seed, form):
    # ρ → (U⊗U*) ρ on the ket pair (i_k, i_{k+1}) and the bra pair (i'_k, i'_{k+1}) (U → U⊗U*),
    # the dense side built from scipy expm like the single-charge pin above
    st = L.random_mpo(M, N, d, chi, seed)
    if form == "b":
        st = L.to_bform(st)
    rho = L.dense_state2(st)
    rng = np.random.default_rng(seed + 20)
    for parity in (0, 1, 0):
        gates = list(range(parity, M - 1, 2))
        th = rng.uniform(0, np.pi / 2, len(gates))
        ph = rng.uniform(0, 2 * np.pi, len(gates))
        disc = L.apply_layer2(st, parity, th, ph, chi_max=10 ** 6)
        assert max(disc, default=0.0) < 1e-20
        for g, k in enumerate(gates):
            U4 = _u4(th[g], ph[g], d, N)
            rho = L.dense_gate(rho, k, U4)
            rho = L.dense_gate(rho, M + k, U4.conj())
        got = L.dense_state2(st)
        assert np.linalg.norm(got - rho) <= 1e-12 * np.linalg.norm(rho), parity


def test_mpo_layer_on_vectorized_pure_state_matches_mps_layer():
    st = L.random_mps(5, 3, 3, 5, 7)
    mpo = L.vectorize_mps(st)
    rng = np.random.default_rng(70)
    for parity in (0, 1):
        n = len(range(parity, 4, 2))
        th, ph = rng.uniform(0, np.pi / 2, n), rng.uniform(0, 2 * np.pi, n)
        L.apply_layer(st, parity, th, ph, chi_max=10 ** 6)
        L.apply_layer2(mpo, parity, th, ph, chi_max=10 ** 6)
    psi = L.dense_state(st)
    rho = L.dense_state2(mpo)
    assert np.linalg.norm(rho - np.multiply.outer(psi, psi.conj())) <= 1e-11 * np.linalg.norm(rho)


@pytest.mark.parametrize("chi_max", [4, 10 ** 6])
def test_bform_and_vidal_updates_agree(chi_max):
    # with well-conditioned λ (≥ 0.2) the right-canonical and the Vidal update are the same TEBD step: identical
    # charges and λ's, the same (truncated) dense state, and B^{[k]} = Γ^{[k]}λ^{[k+1]} after every layer
    st = L.random_mps(6, 3, 3, 6, 11)
    sb = L.to_bform(st)
    rng = np.random.default_rng(12)
    for parity in (0, 1, 0, 1):
        n = len(range(parity, 5, 2))
        th, ph = rng.uniform(0, np.pi / 2, n), rng.uniform(0, 2 * np.pi, n)
        dv = L.apply_layer(st, parity, th, ph, chi_max)
        db = L.apply_layer(sb, parity, th, ph, chi_max)
        assert np.allclose(dv, db, rtol=1e-10, atol=1e-14)
        for k in range(7):
            assert np.array_equal(st["q"][k], sb["q"][k]) and np.allclose(st["lam"][k], sb["lam"][k], rtol=1e-12)
    psi_v, psi_b = L.dense_state(st), L.dense_state(sb)
    assert np.linalg.norm(psi_v - psi_b) <= 1e-11 * np.linalg.norm(psi_v)
    for k in range(6):
        assert np.allclose(sb["gam"][k], st["gam"][k] * st["lam"][k + 1][None, :], rtol=1e-9, atol=1e-12)


def test_bform_update_needs_no_small_lambda_division():
    # λ spanning 14 decades: Vidal Γ's pick up ~ε/λ_min of rounding, the B form keeps every factor's error at
    # rounding level — its dense state after a truncating layer equals the Vidal one computed in exact-λ
    # conditions only where both are accurate, so check B-form against dense evolution directly (no truncation)
    st = L.random_mps(5, 3, 3, 6, 13)
    for k in range(1, 5):
        n = len(st["lam"][k])
        st["lam"][k] = np.logspace(0, -14, n)
    sb = L.to_bform(st)
    psi = L.dense_state(sb)
    rng = np.random.default_rng(14)
    for parity in (0, 1):
        gates = list(range(parity, 4, 2))
        th, ph = rng.uniform(0, np.pi / 2, len(gates)), rng.uniform(0, 2 * np.pi, len(gates))
        L.apply_layer(sb, parity, th, ph, chi_max=10 ** 6, cutoff=0.0)
        for g, k in enumerate(gates):
            psi = L.dense_gate(psi, k, _u4(th[g], ph[g], 3, 3))
    assert np.linalg.norm(L.dense_state(sb) - psi) <= 1e-12 * np.linalg.norm(psi)
