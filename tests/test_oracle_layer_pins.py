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


@pytest.mark.parametrize("M,N,d,chi,seed", [(4, 2, 3, 4, 0), (5, 3, 3, 5, 1), (4, 3, 4, 6, 2), (5, 2, 2, 4, 3)])
def test_layer_without_truncation_is_dense_evolution(M, N, d, chi, seed):
    st = L.random_mps(M, N, d, chi, seed)
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
