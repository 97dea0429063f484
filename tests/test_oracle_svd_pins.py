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


# ------------------------------------------------------------------ MPO (pair-charge) truncation
def _theta2(c):
    return oracle.theta2_sectors(c.N, c.d, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, c.gamma_k, c.lam_k,
                                 c.gamma_k1, c.lam_l, c.lam_r, c.theta, c.phi)[0]


@pytest.mark.parametrize("chi", [7, 40, 10 ** 6])
def test_pair_truncation_kronecker_closed_form(chi):
    # vectorized pure state: Θ2(c1,c2) = Θ(c1) ⊗ conj(Θ(c2)) up to row/column order, so its singular values
    # are exactly the products s_i(c1)·s_j(c2) (SVD of a Kronecker product); the kept λ are the top-χ
    # products, and the kept count of every unordered pair {c1, c2} is fixed by them (the ordered split of
    # an exact tie between (c1,c2) and (c2,c1) is decided by rounding, so only the sum is compared)
    base = synth.make_case(3, 4, 9, 8, 10, seed=12, charges="uniform", lam="random")
    vec = synth.vectorize_pure(base)
    single = oracle.theta_sectors(base.N, base.d, base.q_l, base.q_c, base.q_r, base.gamma_k, base.lam_k,
                                  base.gamma_k1, base.lam_l, base.lam_r, base.theta, base.phi)[0]
    sv = [np.linalg.svd(t, compute_uv=False) if t.size else np.zeros(0) for t in single]
    prods = sorted(((a * b, c1, c2) for c1 in range(base.N + 1) for c2 in range(base.N + 1)
                    for a in sv[c1] for b in sv[c2] if a * b > 1e-14), key=lambda x: -x[0])
    top = prods[:chi]
    res = osvd.truncate_update2(vec.N, vec.d, vec.q1_l, vec.q2_l, vec.q1_r, vec.q2_r, _theta2(vec), vec.lam_l,
                                vec.lam_r, chi)
    assert res["chi"] == len(top)
    smax = top[0][0]
    assert np.max(np.abs(np.sort(res["lam_new"])[::-1] - np.array([t[0] for t in top]))) <= 1e-13 * smax
    want, got = {}, {}
    for _, c1, c2 in top:
        want[frozenset((c1, c2))] = want.get(frozenset((c1, c2)), 0) + 1
    for c1, c2 in zip(res["q1_new"], res["q2_new"]):
        got[frozenset((int(c1), int(c2)))] = got.get(frozenset((int(c1), int(c2))), 0) + 1
    assert got == want


def test_pair_truncation_reduces_to_single_charge():
    # a second species that is identically zero: Θ2(c1, 0) = Θ(c1) (U_0 = 1), every other sector empty,
    # so the pair step must return the pinned single-charge step exactly (sector index c1·(N+1) = charge c1)
    base = synth.make_config(1)
    z = lambda q: np.zeros_like(q)
    secs = _theta2(synth.PairCase("q2=0", base.N, base.d, base.q_l, z(base.q_l), base.q_c, z(base.q_c), base.q_r,
                                  z(base.q_r), base.gamma_k, base.gamma_k1, base.lam_l, base.lam_k, base.lam_r,
                                  base.theta, base.phi))
    single = oracle.theta_sectors(base.N, base.d, base.q_l, base.q_c, base.q_r, base.gamma_k, base.lam_k,
                                  base.gamma_k1, base.lam_l, base.lam_r, base.theta, base.phi)[0]
    for c1 in range(base.N + 1):
        assert np.allclose(secs[(c1, 0)], single[c1], rtol=0, atol=1e-13 * max(1.0, np.abs(single[c1]).max(initial=0)))
    for chi in (30, 10 ** 6):
        r2 = osvd.truncate_update2(base.N, base.d, base.q_l, z(base.q_l), base.q_r, z(base.q_r), secs, base.lam_l,
                                   base.lam_r, chi)
        r1 = osvd.truncate_update(base.N, base.d, base.q_l, base.q_r, single, base.lam_l, base.lam_r, chi)
        assert r2["chi"] == r1["chi"]
        assert np.array_equal(r2["q1_new"], r1["q_new"]) and not r2["q2_new"].any()
        assert np.allclose(r2["lam_new"], r1["lam_new"], rtol=1e-12, atol=0)
        # the factors agree up to one phase per kept vector: compare the phase-free products
        P2 = r2["gamma_k_new"] * r2["lam_new"][None, :] @ r2["gamma_k1_new"]
        P1 = r1["gamma_k_new"] * r1["lam_new"][None, :] @ r1["gamma_k1_new"]
        assert np.linalg.norm(P2 - P1) <= 1e-12 * np.linalg.norm(P1)


def test_pair_no_truncation_reconstructs_theta2():
    c = synth.make_pair_config(0)
    secs = _theta2(c)
    res = osvd.truncate_update2(c.N, c.d, c.q1_l, c.q2_l, c.q1_r, c.q2_r, secs, c.lam_l, c.lam_r, 10 ** 6)
    pl, pr = oracle.sort_pair_bonds(c.q1_l, c.q2_l), oracle.sort_pair_bonds(c.q1_r, c.q2_r)
    key = res["q1_new"] * (c.N + 1) + res["q2_new"]
    for c1 in range(c.N + 1):
        for c2 in range(c.N + 1):
            th = secs[(c1, c2)]
            if th.size == 0:
                continue
            rows = pl[oracle.pair_sector_rows(c.q1_l[pl], c.q2_l[pl], c.d, c1, c2)]
            cols = pr[oracle.pair_sector_cols(c.q1_r[pr], c.q2_r[pr], c.d, c1, c2)]
            a = np.nonzero(key == c1 * (c.N + 1) + c2)[0]
            A = c.lam_l[rows][:, None] * res["gamma_k_new"][np.ix_(rows, a)]
            B = res["gamma_k1_new"][np.ix_(a, cols)] * c.lam_r[cols][None, :]
            rec = (A * res["lam_new"][a][None, :]) @ B
            assert np.linalg.norm(rec - th) <= 1e-12 * max(np.linalg.norm(th), 1e-300), (c1, c2)
    assert res["discarded"] <= 1e-24


@pytest.mark.parametrize("chi", [40, 10 ** 6])
def test_bform_update_reconstructs_like_vidal(chi):
    # the right-canonical update (R22) is the same truncation as the Vidal one: identical ranking and
    # λ, λl·B^{[k]}·B^{[k+1]} = λl·Γ^{[k]}·diag(λ)·Γ^{[k+1]}·λr on every sector, B^{[k+1]} rows orthonormal per charge
    import synth
    case = synth.make_config(1)
    secs, *_ = oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                    case.gamma_k1, case.lam_l, case.lam_r, case.theta, case.phi)
    v = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, secs, case.lam_l, case.lam_r, chi)
    b = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, secs, case.lam_l, case.lam_r, chi, form="b")
    assert v["chi"] == b["chi"] and np.array_equal(v["q_new"], b["q_new"])
    assert np.array_equal(v["lam_new"], b["lam_new"]) and v["discarded"] == b["discarded"]
    ll, lr = case.lam_l, case.lam_r
    for c in range(case.N + 1):
        a = np.nonzero(b["q_new"] == c)[0]
        if a.size == 0:
            continue
        rv = (ll[:, None] * v["gamma_k_new"][:, a] * v["lam_new"][a][None, :]) @ (v["gamma_k1_new"][a] * lr[None, :])
        rb = (ll[:, None] * b["gamma_k_new"][:, a]) @ b["gamma_k1_new"][a]
        assert np.linalg.norm(rb - rv) <= 1e-12 * np.linalg.norm(rv)
        B1 = b["gamma_k1_new"][a]
        assert np.abs(B1 @ B1.conj().T - np.eye(a.size)).max() <= 1e-12
