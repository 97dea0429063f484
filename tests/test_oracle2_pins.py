"""Pins of the MPO (doubled-charge) oracle oracle.theta2_sectors against things other than itself
(`-m "not gpu"`):

  * vectorized pure state: for Γ2 = Γ ⊗ conj(Γ), λ2 = λ ⊗ λ and charge pairs (q[α], q[α']), Eq. S5 with
    U → U⊗U* factorises per species, so Θ2(c1,c2)[(α,α'),(β,β')] = Θ(c1)[α,β]·conj(Θ(c2)[α',β']) with Θ
    the (separately pinned) single-charge oracle — SPEC.md:355 "pure-state consistency";
  * dense brute force: Eq. S5 for the vectorized site written out with the doubled gate
    (U⊗U*)[(a,b),(c,e)] = U[a,c]·conj(U[b,e]), U from scipy expm of the two-mode generator,
    and explicit δ tensors for both charge species;
  * θ = 0: Θ2 = λlΓkλkΓk1λr with the centre pair equal to (c1, c2);
  * d = N+1: Σ‖Θ2‖² does not depend on the gate (U⊗U* is unitary on every block pair).
"""
import itertools

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth


def _theta2(case, theta=None):
    th = case.theta if theta is None else theta
    return oracle.theta2_sectors(case.N, case.d, case.q1_l, case.q2_l, case.q1_c, case.q2_c, case.q1_r, case.q2_r,
                                 case.gamma_k, case.lam_k, case.gamma_k1, case.lam_l, case.lam_r, th, case.phi)


def _rows_cols(case, perms, c1, c2):
    pl, _, pr = perms
    l1, l2 = case.q1_l[pl], case.q2_l[pl]
    r1, r2 = case.q1_r[pr], case.q2_r[pr]
    return (oracle.pair_sector_rows(l1, l2, case.d, c1, c2), oracle.pair_sector_cols(r1, r2, case.d, c1, c2))


def test_pair_sort_is_lexicographic_and_stable():
    q1 = [2, 0, 1, 0, 2, 1, 0]
    q2 = [1, 1, 0, 1, 0, 0, 0]
    perm = oracle.sort_pair_bonds(q1, q2)
    assert perm.tolist() == [6, 1, 3, 2, 5, 4, 0]


@pytest.mark.parametrize("seed,N,d,chi", [(0, 2, 3, 5), (3, 3, 4, 4), (7, 3, 2, 5)])
def test_vectorized_pure_state_factorises(seed, N, d, chi):
    base = synth.make_case(N, d, chi, chi, chi, seed=seed, charges="uniform", lam="random")
    vec = synth.vectorize_pure(base)
    s1, perms1, offs1, _ = oracle.theta_sectors(N, d, base.q_l, base.q_c, base.q_r, base.gamma_k, base.lam_k,
                                                base.gamma_k1, base.lam_l, base.lam_r, base.theta, base.phi)
    s2, perms2, _ = _theta2(vec)
    pl1, _, pr1 = perms1
    pl2, _, pr2 = perms2
    for c1, c2 in itertools.product(range(N + 1), repeat=2):
        rows, cols = _rows_cols(vec, perms2, c1, c2)
        got = s2[(c1, c2)]
        assert got.shape == (len(rows), len(cols))
        (a0, _), (b0, _) = oracle.sector_ranges(offs1[0], offs1[2], N, d, c1)
        (e0, _), (f0, _) = oracle.sector_ranges(offs1[0], offs1[2], N, d, c2)
        inv_l, inv_r = np.argsort(pl1), np.argsort(pr1)
        ref = np.zeros_like(got)
        for i, p in enumerate(rows):
            al, alp = divmod(int(pl2[p]), chi)             # bond (α, α') of the vectorized index
            for j, q in enumerate(cols):
                be, bep = divmod(int(pr2[q]), chi)
                ref[i, j] = s1[c1][inv_l[al] - a0, inv_r[be] - b0] * np.conj(s1[c2][inv_l[alp] - e0, inv_r[bep] - f0])
        nrm = np.linalg.norm(ref)
        assert np.linalg.norm(got - ref) <= 1e-13 * max(nrm, 1e-300), (c1, c2)


def _u4(theta, phi, d, N):
    D = min(N, 2 * d - 2) + 1
    a = np.diag(np.sqrt(np.arange(1, D)), 1)
    A, B = np.kron(a, np.eye(D)), np.kron(np.eye(D), a)
    G = theta * (np.exp(1j * phi) * A.conj().T @ B - np.exp(-1j * phi) * A @ B.conj().T)
    Uf = scipy.linalg.expm(G).reshape(D, D, D, D)
    U4 = np.zeros((d, d, d, d), dtype=np.complex128)
    m = min(d, D)
    for i, ip, j, jp in itertools.product(range(m), repeat=4):
        if i + ip == j + jp and i + ip <= D - 1:
            U4[i, ip, j, jp] = Uf[i, ip, j, jp]
    return U4


def _bruteforce2(case):
    """Eq. S5 for the vectorized site: doubled gate U8 = U⊗U*, explicit δ tensors per species."""
    N, d = case.N, case.d
    U4 = _u4(case.theta, case.phi, d, N)
    # U8[(i,i'),(k,k'),(j,j'),(l,l')] = U4[i,k,j,l]·conj(U4[i',k',j',l'])
    U8 = np.einsum("ikjl,pqrs->ipkqjrls", U4, np.conj(U4))
    L1, L2 = case.q1_l.astype(np.int64), case.q2_l.astype(np.int64)
    M1, M2 = case.q1_c.astype(np.int64), case.q2_c.astype(np.int64)
    R1, R2 = case.q1_r.astype(np.int64), case.q2_r.astype(np.int64)
    J = np.arange(d)
    dl = ((L1[:, None, None, None] - M1[None, None, None, :] == J[None, :, None, None]) &
          (L2[:, None, None, None] - M2[None, None, None, :] == J[None, None, :, None])).astype(float)   # [α,j,j',γ]
    dr = ((M1[:, None, None, None] - R1[None, None, None, :] == J[None, :, None, None]) &
          (M2[:, None, None, None] - R2[None, None, None, :] == J[None, None, :, None])).astype(float)   # [γ,l,l',β]
    A = case.lam_l[:, None, None, None] * case.gamma_k[:, None, None, :] * case.lam_k[None, None, None, :] * dl
    Bt = case.gamma_k1[:, None, None, :] * case.lam_r[None, None, None, :] * dr
    T = np.einsum("ajkg,glmb->ajklmb", A, Bt, optimize=True)
    full = np.einsum("ipkqjrls,ajrlsb->aipkqb", U8, T, optimize=True)   # [α, i, i', k, k', β]
    out = {}
    for c1, c2 in itertools.product(range(N + 1), repeat=2):
        i1, i2 = L1 - c1, L2 - c2
        k1, k2 = c1 - R1, c2 - R2
        rows = np.where((i1 >= 0) & (i1 <= d - 1) & (i2 >= 0) & (i2 <= d - 1))[0]
        cols = np.where((k1 >= 0) & (k1 <= d - 1) & (k2 >= 0) & (k2 <= d - 1))[0]
        sec = np.array([[full[a, i1[a], i2[a], k1[b], k2[b], b] for b in cols] for a in rows],
                       dtype=np.complex128).reshape(len(rows), len(cols))
        out[(c1, c2)] = (rows, cols, sec)
    return out


@pytest.mark.parametrize("args", [dict(N=2, d=3, chi=(7, 6, 8), seed=1), dict(N=3, d=2, chi=(6, 5, 7), seed=2),
                                  dict(N=2, d=4, chi=(5, 7, 6), seed=3)])
def test_theta2_bruteforce(args):
    case = synth.make_pair_case(args["N"], args["d"], *args["chi"], seed=args["seed"], charges="uniform",
                                lam="random", theta=0.83, phi=1.9)
    secs, perms, _ = _theta2(case)
    bf = _bruteforce2(case)
    pl, _, pr = perms
    for key, (rows, cols, ref) in bf.items():
        srows, scols = _rows_cols(case, perms, *key)
        assert sorted(pl[srows].tolist()) == rows.tolist() and sorted(pr[scols].tolist()) == cols.tolist()
        pos_r = {b: i for i, b in enumerate(rows.tolist())}
        pos_c = {b: i for i, b in enumerate(cols.tolist())}
        ref_sorted = ref[np.ix_([pos_r[int(x)] for x in pl[srows]], [pos_c[int(x)] for x in pr[scols]])]
        got = secs[key]
        nrm = np.linalg.norm(ref_sorted)
        if nrm == 0:
            assert np.all(got == 0)
        else:
            assert np.linalg.norm(got - ref_sorted) / nrm < 1e-13, key


@pytest.mark.parametrize("cfg", [0, 1])
def test_theta2_identity_gate_is_two_site_product(cfg):
    case = synth.make_pair_config(cfg)
    secs, perms, _ = _theta2(case, theta=0.0)
    pl, pc, pr = perms
    Gk, Gk1 = case.gamma_k[pl][:, pc], case.gamma_k1[pc][:, pr]
    m1, m2 = case.q1_c[pc], case.q2_c[pc]
    for (c1, c2), got in secs.items():
        rows, cols = _rows_cols(case, perms, c1, c2)
        lk = case.lam_k[pc] * ((m1 == c1) & (m2 == c2))
        ref = (case.lam_l[pl][rows, None] * Gk[rows]) @ (lk[:, None] * Gk1[:, cols]) * case.lam_r[pr][None, cols]
        assert np.linalg.norm(got - ref) <= 1e-13 * max(np.linalg.norm(ref), 1e-300)


@pytest.mark.parametrize("cfg", [0, 1])
def test_theta2_norm_invariance(cfg):
    case = synth.make_pair_config(cfg)
    assert case.d == case.N + 1
    su = sum(np.linalg.norm(x) ** 2 for x in _theta2(case)[0].values())
    si = sum(np.linalg.norm(x) ** 2 for x in _theta2(case, theta=0.0)[0].values())
    assert abs(su - si) / si < 1e-12


def test_flop_counts2_against_bruteforce_count():
    case = synth.make_pair_case(2, 3, 9, 8, 10, seed=4, charges="uniform", lam="random")
    fc, fm = oracle.flop_counts2(case.N, case.d, case.q1_l, case.q2_l, case.q1_c, case.q2_c, case.q1_r, case.q2_r)
    # brute force over bond triples: one complex MAC per allowed (α, α_k, β) — 8 flops each
    ok = lambda a, b: (a - b >= 0) & (a - b <= case.d - 1)
    al = ok(case.q1_l[:, None], case.q1_c[None, :]) & ok(case.q2_l[:, None], case.q2_c[None, :])
    ar = ok(case.q1_c[:, None], case.q1_r[None, :]) & ok(case.q2_c[:, None], case.q2_r[None, :])
    assert fc == 8 * int(al.astype(np.int64).sum(axis=0) @ ar.astype(np.int64).sum(axis=1))
    assert fm > 0


def test_theta2_element_matches_sectors():
    case = synth.make_pair_config(1)
    secs, perms, ub = _theta2(case)
    rng = np.random.default_rng(0)
    for key in [(0, 0), (2, 3), (4, 4), (1, 2)]:
        R, Cc = secs[key].shape
        for _ in range(5):
            a, b = int(rng.integers(R)), int(rng.integers(Cc))
            v = oracle.theta2_element(case.N, case.d, *key, a, b, case.q1_l, case.q2_l, case.q1_c, case.q2_c,
                                      case.q1_r, case.q2_r, case.gamma_k, case.lam_k, case.gamma_k1, case.lam_l,
                                      case.lam_r, ub, perms)
            assert abs(v - secs[key][a, b]) <= 1e-13 * max(abs(v), 1e-300)
