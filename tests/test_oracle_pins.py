"""Pins for the CPU oracle against things other than itself (runs without a GPU).

Each test names what fixes the expected value: the paper/SPEC worked examples, a textbook routine
(scipy expm of the ladder-operator generator, sympy Wigner small-d), a closed form, an invariant, or
brute force with explicit dense δ tensors (PAPER.md:70 describes exactly that contraction).
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- sorting
def test_sort_spec_examples():
    perm, off = oracle.sort_bonds([2, 0, 1, 0], N=2)
    assert perm.tolist() == [1, 3, 2, 0]
    assert off.tolist() == [0, 2, 3, 4]
    perm, off = oracle.sort_bonds([0, 1, 1, 3], N=3)
    assert perm.tolist() == [0, 1, 2, 3]                       # SPEC.md:57 idempotence
    assert off.tolist() == [0, 1, 3, 3, 4]


def test_sort_idempotent_and_stable_random():
    rng = np.random.default_rng(7)
    q = rng.integers(0, 6, size=200)
    perm, off = oracle.sort_bonds(q, N=5)
    qs = q[perm]
    assert np.all(np.diff(qs) >= 0)
    for v in range(6):                                          # stability: original order kept
        idx = perm[qs == v]
        assert np.all(np.diff(idx) > 0)
        assert off[v + 1] - off[v] == np.sum(q == v)
    perm2, _ = oracle.sort_bonds(qs, N=5)
    assert perm2.tolist() == list(range(200))


# ---------------------------------------------------------------- U (Eq. S4) against textbook routines
def _expm_block(n, theta, phi):
    """exp of θ(e^{iφ} a†b − e^{−iφ} a b†) on the (n+1)-dim fixed-n block, basis |i, n−i⟩, by scipy."""
    G = np.zeros((n + 1, n + 1), dtype=np.complex128)
    for i in range(n + 1):
        if i + 1 <= n:   # a†b |i, n−i⟩ = √((i+1)(n−i)) |i+1, n−i−1⟩
            G[i + 1, i] += theta * np.exp(1j * phi) * math.sqrt((i + 1) * (n - i))
        if i - 1 >= 0:   # a b† |i, n−i⟩ = √(i(n−i+1)) |i−1, n−i+1⟩
            G[i - 1, i] -= theta * np.exp(-1j * phi) * math.sqrt(i * (n - i + 1))
    return scipy.linalg.expm(G)


@pytest.mark.parametrize("d", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("theta,phi", [(0.3, 0.0), (0.7, 0.3), (1.3, 4.0), (math.pi / 2 - 1e-3, 2.2)])
def test_u_matches_expm(d, theta, phi):
    N = d - 1
    for n in range(0, min(N, 2 * d - 2) + 1, max(1, d // 8)):
        blk = oracle.bs_unitary_block(n, theta, phi, d)
        ref = _expm_block(n, theta, phi)
        lo, hi = max(0, n - d + 1), min(n, d - 1)
        tol = 2e-15 * max(1, n)                     # expm's own error grows ~ with the block norm
        assert np.max(np.abs(blk - ref[lo:hi + 1, lo:hi + 1])) < tol, n


def test_u_truncated_blocks_are_restricted_exact_elements():
    # DESIGN.md R6: for n >= d, the stored block is the untruncated exact block restricted
    d, N = 3, 5
    for n in range(0, min(N, 2 * d - 2) + 1):
        blk = oracle.bs_unitary_block(n, 0.9, 1.7, d)
        ref = _expm_block(n, 0.9, 1.7)
        lo, hi = max(0, n - d + 1), min(n, d - 1)
        assert blk.shape == (hi - lo + 1, hi - lo + 1)
        assert np.max(np.abs(blk - ref[lo:hi + 1, lo:hi + 1])) < 1e-14


def test_hom_dip_and_identity():
    g = json.load(open(os.path.join(GOLD, "hom_dip.json")))
    blk = oracle.bs_unitary_block(g["n"], g["theta"], g["phi"], d=4)
    assert abs(blk[g["i"], g["j"]] - g["value"]) <= g["abs_tol"]
    for n in range(6):
        assert np.array_equal(oracle.bs_unitary_block(n, 0.0, 0.77, d=6), np.eye(n + 1))


@pytest.mark.parametrize("phi", [0.0, 0.3, 4.0])
def test_u_half_pi_swap_closed_form(phi):
    # θ=π/2: B a† B† = −e^{−iφ} b†, B b† B† = e^{iφ} a†  ⇒  U|j, n−j⟩ = (−e^{−iφ})^j e^{iφ(n−j)} |n−j, j⟩
    d = 12
    for n in range(d):
        blk = oracle.bs_unitary_block(n, math.pi / 2, phi, d)
        ref = np.zeros_like(blk)
        for j in range(n + 1):
            ref[n - j, j] = (-np.exp(-1j * phi)) ** j * np.exp(1j * phi * (n - j))
        assert np.max(np.abs(blk - ref)) < 1e-15 * (n + 1)


def test_u_wigner_small_d():
    # U(θ,0) block n is the spin-n/2 rotation d^{n/2}_{i−n/2, j−n/2}(−2θ) (sympy, textbook routine)
    from sympy import Rational, N as sN
    from sympy.physics.quantum.spin import Rotation
    theta = 0.61
    for n in range(1, 5):
        blk = oracle.bs_unitary_block(n, theta, 0.0, d=n + 1)
        j = Rational(n, 2)
        for i in range(n + 1):
            for k in range(n + 1):
                ref = complex(sN(Rotation.d(j, i - j, k - j, -2 * theta).doit(), 30))
                assert abs(blk[i, k] - ref) < 3e-16, (n, i, k)


@pytest.mark.parametrize("d", [2, 4, 8, 16, 32, 48])
def test_u_block_unitarity(d):
    th, ph = 0.7, 0.3
    for n in range(0, d, max(1, d // 6)):             # blocks n <= d-1 are complete, hence unitary
        blk = oracle.bs_unitary_block(n, th, ph, d)
        assert np.max(np.abs(blk.conj().T @ blk - np.eye(n + 1))) < 1e-13


def test_u_phase_relation():
    for n in (3, 9, 20):
        b0 = oracle.bs_unitary_block(n, 1.1, 0.0, d=n + 1)
        b1 = oracle.bs_unitary_block(n, 1.1, 2.5, d=n + 1)
        assert np.all(b0.imag == 0)
        i = np.arange(n + 1)
        ph = np.exp(1j * 2.5 * (i[:, None] - i[None, :]))
        assert np.max(np.abs(b1 - ph * b0)) < 1e-15 * (n + 1)


def test_packed_u_layout():
    starts, tot = oracle.packed_u_offsets(32, 31)
    assert tot == 11440 and starts[5] == 5 * 6 * 11 // 6           # (N+1)(N+2)(2N+3)/6, n(n+1)(2n+1)/6
    assert oracle.packed_u_offsets(48, 47)[1] == 38024
    pu = oracle.packed_u(0.4, 0.2, 4, 3)
    assert pu.shape == (30,)
    s4, _ = oracle.packed_u_offsets(4, 3)
    assert s4 == [0, 1, 5, 14]
    assert np.array_equal(pu[5:14], oracle.bs_unitary_block(2, 0.4, 0.2, 4).ravel())


# ---------------------------------------------------------------- Θ (Eq. S5) against a dense δ-tensor brute force
def _u4_dense(theta, phi, d, N):
    """U4[i, i', j, j'] = ⟨i,i'|U|j,j'⟩ from expm of the two-mode generator on a Fock space big enough
    to hold every total n <= min(N, 2d-2) exactly, restricted to occupations < d (textbook route)."""
    D = min(N, 2 * d - 2) + 1
    a = np.diag(np.sqrt(np.arange(1, D)), 1)            # annihilation on one mode, truncated at D
    A = np.kron(a, np.eye(D))
    B = np.kron(np.eye(D), a)
    G = theta * (np.exp(1j * phi) * A.conj().T @ B - np.exp(-1j * phi) * A @ B.conj().T)
    Uf = scipy.linalg.expm(G).reshape(D, D, D, D)
    U4 = np.zeros((d, d, d, d), dtype=np.complex128)
    m = min(d, D)
    for i in range(m):
        for ip in range(m):
            for j in range(m):
                for jp in range(m):
                    if i + ip == j + jp and i + ip <= D - 1:   # blocks beyond D-1 cannot occur in Θ
                        U4[i, ip, j, jp] = Uf[i, ip, j, jp]
    return U4


def _theta_bruteforce(case):
    """Eq. S5 as written: dense δ tensors, sum over j_k, j_{k+1}, α_k, then read off sector c."""
    N, d = case.N, case.d
    U4 = _u4_dense(case.theta, case.phi, d, N)
    ql, qc, qr = (x.astype(np.int64) for x in (case.q_l, case.q_c, case.q_r))
    dl = (ql[:, None, None] - qc[None, None, :] == np.arange(d)[None, :, None]).astype(float)  # δ(c_l−c_c−j_k)
    dr = (qc[:, None, None] - qr[None, None, :] == np.arange(d)[None, :, None]).astype(float)  # δ(c_c−c_r−j_k+1)
    A = case.lam_l[:, None, None] * case.gamma_k[:, None, :] * case.lam_k[None, None, :] * dl  # [α, j, γ]
    Bt = case.gamma_k1[:, None, :] * case.lam_r[None, None, :] * dr                            # [γ, j', β]
    T = np.einsum("ajg,gkb->ajkb", A, Bt, optimize=True)
    full = np.einsum("ipjk,ajkb->aipb", U4, T, optimize=True)                                # [α, i, i', β]
    out = []
    for c in range(N + 1):
        il = ql - c                      # δ(c_l − c − i_k)
        ir = c - qr                      # δ(c − c_r − i_{k+1})
        rows = np.where((il >= 0) & (il <= d - 1))[0]
        cols = np.where((ir >= 0) & (ir <= d - 1))[0]
        sec = np.array([[full[a, il[a], ir[b], b] for b in cols] for a in rows],
                       dtype=np.complex128).reshape(len(rows), len(cols))
        out.append((rows, cols, sec))
    return out


def _check_vs_bruteforce(case, tol):
    secs, perms, offs, _ = oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k,
                                                case.lam_k, case.gamma_k1, case.lam_l, case.lam_r,
                                                case.theta, case.phi)
    bf = _theta_bruteforce(case)
    perm_l, _, perm_r = perms
    for c in range(case.N + 1):
        rows, cols, ref = bf[c]
        (r0, r1), (k0, k1) = oracle.sector_ranges(offs[0], offs[2], case.N, case.d, c)
        # oracle rows are sorted positions; map to original bonds and compare as sets + values
        assert sorted(perm_l[r0:r1].tolist()) == rows.tolist()
        assert sorted(perm_r[k0:k1].tolist()) == cols.tolist()
        pos_r = {b: i for i, b in enumerate(rows.tolist())}
        pos_c = {b: i for i, b in enumerate(cols.tolist())}
        ri = [pos_r[int(x)] for x in perm_l[r0:r1]]
        ci = [pos_c[int(x)] for x in perm_r[k0:k1]]
        ref_sorted = ref[np.ix_(ri, ci)] if ref.size else ref
        got = secs[c]
        assert got.shape == ref_sorted.shape
        nrm = np.linalg.norm(ref_sorted)
        if nrm == 0:
            assert np.all(got == 0)
        else:
            assert np.linalg.norm(got - ref_sorted) / nrm < tol, c


def test_theta_bruteforce_config0():
    _check_vs_bruteforce(synth.make_config(0), 1e-13)


def test_theta_bruteforce_config0_shuffled():
    _check_vs_bruteforce(synth.make_config(0, shuffled=True), 1e-13)


def test_theta_bruteforce_truncated_d():
    # d < N+1: U blocks with n >= d are truncated (R6); SURVEY.md T6 case N=5, d=3, χ=16
    case = synth.make_case(5, 3, 16, 16, 16, seed=11, charges="uniform", lam="random", theta=0.9, phi=1.1)
    _check_vs_bruteforce(case, 1e-13)


def test_theta_bruteforce_rect_and_gaps():
    # rectangular bonds, an empty center-charge segment, d = N+2 (> N+1)
    case = synth.make_case(4, 6, 12, 9, 14, seed=5, charges="uniform", lam="random", theta=0.4, phi=2.0)
    case.q_c[case.q_c == 2] = 1
    case.gamma_k *= ((case.q_l[:, None] - case.q_c[None, :] >= 0) & (case.q_l[:, None] - case.q_c[None, :] <= case.d - 1))
    case.gamma_k1 *= ((case.q_c[:, None] - case.q_r[None, :] >= 0) & (case.q_c[:, None] - case.q_r[None, :] <= case.d - 1))
    _check_vs_bruteforce(case, 1e-13)


@pytest.mark.slow
def test_theta_bruteforce_config1():
    _check_vs_bruteforce(synth.make_config(1), 1e-13)


# ---------------------------------------------------------------- invariants
def _oracle(case, theta=None):
    th = case.theta if theta is None else theta
    return oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                case.gamma_k1, case.lam_l, case.lam_r, th, case.phi)


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_norm_invariance_total(cfg):
    # d = N+1: every block U_n with n <= N is unitary, so Σ_c ‖Θ(c)‖² is independent of U (total only)
    case = synth.make_config(cfg)
    s_u = sum(np.linalg.norm(x) ** 2 for x in _oracle(case)[0])
    s_i = sum(np.linalg.norm(x) ** 2 for x in _oracle(case, theta=0.0)[0])
    assert abs(s_u - s_i) / s_i < 1e-12


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_identity_gate_is_two_site_product(cfg):
    # θ=0: U = I, so Θ(c) = λl Γk λk|_{c_c=c} Γk1 λr restricted to Θ(c)'s rows/cols
    case = synth.make_config(cfg)
    secs, perms, offs, _ = _oracle(case, theta=0.0)
    pl, pc, pr = perms
    Gk = case.gamma_k[pl][:, pc]
    Gk1 = case.gamma_k1[pc][:, pr]
    qc = case.q_c[pc]
    for c in range(case.N + 1):
        (r0, r1), (k0, k1) = oracle.sector_ranges(offs[0], offs[2], case.N, case.d, c)
        lk = case.lam_k[pc] * (qc == c)
        ref = (case.lam_l[pl][r0:r1, None] * Gk[r0:r1]) @ (lk[:, None] * Gk1[:, k0:k1]) * case.lam_r[pr][None, k0:k1]
        nrm = np.linalg.norm(ref)
        assert np.linalg.norm(secs[c] - ref) <= 1e-13 * max(nrm, 1e-300)


def test_single_photon_golden():
    g = json.load(open(os.path.join(GOLD, "single_photon_bs.json")))
    one = np.ones((1, 1), dtype=np.complex128)
    for cs in g["cases"]:
        secs, *_ = oracle.theta_sectors(g["N"], g["d"], np.array(g["q_l"]), np.array(g["q_c"]), np.array(g["q_r"]),
                                        one, np.ones(1), one, np.ones(1), np.ones(1), cs["theta"], cs["phi"])
        assert [s.shape for s in secs] == [(1, 1), (1, 1)]
        for c in range(2):
            assert abs(abs(secs[c][0, 0]) - cs["abs_theta"][c]) < 1e-15


def test_theta_element_matches_sectors():
    case = synth.make_config(1)
    secs, perms, offs, ub = _oracle(case)
    rng = np.random.default_rng(0)
    for _ in range(40):
        c = int(rng.integers(0, case.N + 1))
        if secs[c].size == 0:
            continue
        a, b = int(rng.integers(0, secs[c].shape[0])), int(rng.integers(0, secs[c].shape[1]))
        v = oracle.theta_element(case.N, case.d, c, a, b, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                 case.gamma_k1, case.lam_l, case.lam_r, ub, (perms, offs))
        assert abs(v - secs[c][a, b]) <= 1e-13 * (abs(secs[c][a, b]) + 1e-30) + 1e-300


def test_flop_counts_per_seed():
    # SURVEY.md §8(d) "Exact per-seed counts under this generator" (computed independently from the draws)
    want = {0: (14560, 10000, 458), 1: (34023872, 4867904, 132672),
            2: (1735597600, 142705608, 2626603), 3: (102206486240, 8615627728, 80079528)}
    for cfg, w in want.items():
        c = synth.make_config(cfg)
        assert oracle.flop_counts(c.N, c.d, c.q_l, c.q_c, c.q_r) == w
