"""Pins of the SVD/truncation oracle (oracle/svd.py) against the mathematics (`-m "not gpu"`):
SPEC.md:76 worked example, known spectra (random unitaries × diag(s)), Eckart–Young on the block-diagonal
Θ, exact reconstruction when χ ≥ rank, orthonormality of the new
canonical factors, and the deterministic tie-break."""
import numpy as np
import pytest

import oracle
import oracle.svd as osvd
import synth


def test_spec_worked_example():
    kept, disc = osvd.global_top_chi([np.array([0.9, 0.1]), np.array([0.5])], 2)
    assert kept == [1, 1] and abs(disc - 0.01) < 1e-15


def test_tie_break_value_then_charge_then_index():
    kept, _ = osvd.global_top_chi([np.array([0.5, 0.2]), np.array([0.5, 0.5])], 2)
    assert kept == [1, 1]                 # the tie at 0.5: charge 0 first, then charge 1 index 0
    kept, _ = osvd.global_top_chi([np.array([0.3]), np.array([0.5, 0.5])], 2)
    assert kept == [0, 2]
    kept, disc = osvd.global_top_chi([np.array([1e-15, 0.0])], 5)   # ≤ cutoff never kept
    assert kept == [0] and disc == 1e-30


def test_known_spectrum():
    rng = np.random.default_rng(3)
    def unitary(n):
        q, r = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        return q * (np.diag(r) / abs(np.diag(r)))
    s = np.sort(rng.random(6))[::-1]
    th = unitary(9)[:, :6] @ np.diag(s) @ unitary(6).conj().T
    (_, got, _), = osvd.sector_svds([th])
    assert np.max(abs(got - s)) < 1e-13


def _reconstruct(case, res, c):
    """λl Γk_new λ_new Γk1_new λr over the new bonds of charge c, on Θ(c)'s rows/cols (sorted order)."""
    perm_l, off_l = oracle.sort_bonds(case.q_l, case.N)
    perm_r, off_r = oracle.sort_bonds(case.q_r, case.N)
    (r0, r1), (k0, k1) = oracle.sector_ranges(off_l, off_r, case.N, case.d, c)
    rows, cols = perm_l[r0:r1], perm_r[k0:k1]
    a = res["q_new"] == c
    A = case.lam_l[rows][:, None] * res["gamma_k_new"][np.ix_(rows, np.nonzero(a)[0])]
    B = res["gamma_k1_new"][np.ix_(np.nonzero(a)[0], cols)] * case.lam_r[cols][None, :]
    return (A * res["lam_new"][a][None, :]) @ B, A


@pytest.mark.parametrize("cfg,chi", [(0, 6), (1, 60), (1, 400)])
def test_eckart_young_and_update(cfg, chi):
    case = synth.make_config(cfg)
    secs, *_ = oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                    case.gamma_k1, case.lam_l, case.lam_r, case.theta, case.phi)
    res = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, secs, case.lam_l, case.lam_r, chi)
    tot = sum(np.linalg.norm(x) ** 2 for x in secs)
    err = 0.0
    for c in range(case.N + 1):
        if secs[c].size == 0:
            continue
        rec, A = _reconstruct(case, res, c)
        err += np.linalg.norm(secs[c] - rec) ** 2
        if A.shape[1]:                                   # U columns orthonormal: λl Γk_new = U_c[:, :k]
            assert np.allclose(A.conj().T @ A, np.eye(A.shape[1]), atol=1e-12)
    assert abs(err - res["discarded"]) <= 1e-12 * tot
    assert res["chi"] == min(chi, sum(len(s) for s in res["svals"]))
    if res["chi"] == sum(len(s) for s in res["svals"]):  # no truncation → exact
        assert res["discarded"] < 1e-20 * tot
    assert np.all(np.diff(res["q_new"]) >= 0)           # new bond sorted by charge


def test_no_truncation_is_exact():
    case = synth.make_config(0)
    secs, *_ = oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                    case.gamma_k1, case.lam_l, case.lam_r, case.theta, case.phi)
    res = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, secs, case.lam_l, case.lam_r, 10 ** 6)
    for c in range(case.N + 1):
        if secs[c].size:
            rec, _ = _reconstruct(case, res, c)
            assert np.linalg.norm(secs[c] - rec) <= 1e-12 * np.linalg.norm(secs[c])
