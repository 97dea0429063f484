"""GPU parity of the SVD step (tn_svd_truncate) against the pinned oracle (oracle/svd.py).

Singular vectors are unique only up to a phase per value, so the comparison is on what is unique:
kept count, charges and values of the new bond (bit-exact charges; values ≤ 1e-12 relative), the
discarded weight, and — phase-free — every sector's truncated reconstruction
λl Γk_new diag(λ_new) Γk1_new λr (≤ 1e-10 relative Frobenius, the Θ bar) plus orthonormality of the
new factors (λl·Γk_new columns and Γk1_new·λr rows of each charge are orthonormal, ≤ 1e-12)."""
import numpy as np
import pytest
import torch

import oracle
import oracle.svd as osvd
import synth
from gpu_util import gpu_theta, oracle_theta

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


def _run(tn, case, chi_max, cutoff=1e-14):
    plan, U, got = gpu_theta(case)
    t = [torch.from_numpy(np.ascontiguousarray(g)).cuda() for g in got]
    ll = torch.from_numpy(case.lam_l).cuda()
    lr = torch.from_numpy(case.lam_r).cuda()
    res = tn.svd_truncate(plan, t, ll, lr, chi_max, cutoff)
    torch.cuda.synchronize()
    out = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in res.items()}
    return got, out


def _recon(case, res, c):
    perm_l, off_l = oracle.sort_bonds(case.q_l, case.N)
    perm_r, off_r = oracle.sort_bonds(case.q_r, case.N)
    (r0, r1), (k0, k1) = oracle.sector_ranges(off_l, off_r, case.N, case.d, c)
    rows, cols = perm_l[r0:r1], perm_r[k0:k1]
    a = np.nonzero(res["q_new"] == c)[0]
    A = case.lam_l[rows][:, None] * res["gamma_k_new"][np.ix_(rows, a)]
    B = res["gamma_k1_new"][np.ix_(a, cols)] * case.lam_r[cols][None, :]
    return (A * res["lam_new"][a][None, :]) @ B, A, B


ALGOS = ["gram", "gesvdp", "gesvdj"]   # TN_SVD_ALGO: Gram eigensolver + Rayleigh–Ritz (default), library SVDs


@pytest.mark.parametrize("algo", ALGOS + ["gram-tested", "gram-libritz"])
@pytest.mark.parametrize("cfg,chi", [(0, 5), (1, 64), (1, 100000), (2, 1024), (2, 300)])
def test_svd_truncate_parity(tn, cfg, chi, algo, monkeypatch):
    # "gram-tested": the trace-power sector test (normally only for n_g ≥ 256) applied to every candidate;
    # "gram-libritz": the Ritz step by a library SVD of Y instead of the default Ritz refinement
    monkeypatch.setenv("TN_SVD_ALGO", algo.split("-")[0])
    if algo == "gram-tested":
        monkeypatch.setenv("TN_SVD_TEST_MIN_NG", "1")
    if algo == "gram-libritz":
        monkeypatch.setenv("TN_RITZ_SVD", "1")
    case = synth.make_config(cfg)
    got, res = _run(tn, case, chi)
    ref_secs, *_ = oracle_theta(case)
    ref = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, ref_secs, case.lam_l, case.lam_r, chi)
    assert res["chi"] == ref["chi"]
    assert np.array_equal(res["q_new"], ref["q_new"])
    smax = max(float(s.max()) for s in ref["svals"] if s.size)
    assert np.max(np.abs(res["lam_new"] - ref["lam_new"]), initial=0.0) <= 1e-12 * smax
    tot = sum(np.linalg.norm(x) ** 2 for x in ref_secs)
    assert abs(res["discarded"] - ref["discarded"]) <= 1e-12 * tot
    for c in range(case.N + 1):
        if ref_secs[c].size == 0:
            continue
        rg, A, B = _recon(case, res, c)
        rr, *_ = _recon(case, ref, c)
        n = np.linalg.norm(rr)
        assert np.linalg.norm(rg - rr) <= 1e-10 * max(n, 1e-300), c
        if A.shape[1]:
            assert np.allclose(A.conj().T @ A, np.eye(A.shape[1]), atol=1e-12)
            assert np.allclose(B @ B.conj().T, np.eye(B.shape[0]), atol=1e-12)


def test_svd_truncate_parity_config3(tn):
    # the configuration whose SVD-step time is quoted (bench.py --svd): config 3, χ_max = 4096,
    # default algorithm; oracle SVD (numpy LAPACK) of the ORACLE's Θ, so nothing on the reference side comes
    # from the GPU
    case = synth.make_config(3)
    got, res = _run(tn, case, 4096)
    ref_secs, *_ = oracle_theta(case)
    ref = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, ref_secs, case.lam_l, case.lam_r, 4096)
    assert res["chi"] == ref["chi"] == 4096
    assert np.array_equal(res["q_new"], ref["q_new"])
    smax = max(float(s.max()) for s in ref["svals"] if s.size)
    assert np.max(np.abs(res["lam_new"] - ref["lam_new"])) <= 1e-12 * smax
    tot = sum(np.linalg.norm(x) ** 2 for x in ref_secs)
    assert abs(res["discarded"] - ref["discarded"]) <= 1e-12 * tot
    for c in range(case.N + 1):
        if ref_secs[c].size == 0:
            continue
        rg, A, B = _recon(case, res, c)
        rr, *_ = _recon(case, ref, c)
        assert np.linalg.norm(rg - rr) <= 1e-10 * max(np.linalg.norm(rr), 1e-300), c
        if A.shape[1]:
            assert np.abs(A.conj().T @ A - np.eye(A.shape[1])).max() <= 1e-12
            assert np.abs(B @ B.conj().T - np.eye(B.shape[0])).max() <= 1e-12


@pytest.mark.parametrize("algo", ALGOS + ["gram-tested", "gram-libritz"])
@pytest.mark.parametrize("chi", [40, 250, 100000])
def test_svd_wide_spectrum(tn, chi, algo, monkeypatch):
    # λ = 0.97^i on every bond: Θ's singular values span many decades, the regime where an eigen-
    # decomposition of the Gram matrix alone loses the small kept values (the Ritz step must recover them)
    monkeypatch.setenv("TN_SVD_ALGO", algo.split("-")[0])
    if algo == "gram-tested":
        monkeypatch.setenv("TN_SVD_TEST_MIN_NG", "1")
    if algo == "gram-libritz":
        monkeypatch.setenv("TN_RITZ_SVD", "1")
    case = synth.make_case(6, 7, 300, 280, 320, seed=44, charges="uniform", lam="steep")
    got, res = _run(tn, case, chi)
    ref_secs, *_ = oracle_theta(case)
    ref = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, ref_secs, case.lam_l, case.lam_r, chi)
    assert res["chi"] == ref["chi"]
    assert np.array_equal(res["q_new"], ref["q_new"])
    smax = max(float(s.max()) for s in ref["svals"] if s.size)
    assert np.max(np.abs(res["lam_new"] - ref["lam_new"])) <= 1e-12 * smax
    for c in range(case.N + 1):
        if ref_secs[c].size == 0:
            continue
        rg, A, B = _recon(case, res, c)
        rr, *_ = _recon(case, ref, c)
        assert np.linalg.norm(rg - rr) <= 1e-10 * max(np.linalg.norm(rr), 1e-300), c
        if A.shape[1]:
            assert np.allclose(A.conj().T @ A, np.eye(A.shape[1]), atol=1e-12)
            assert np.allclose(B @ B.conj().T, np.eye(B.shape[0]), atol=1e-12)


@pytest.mark.parametrize("algo", ALGOS)
def test_svd_no_truncation_reconstructs_theta(tn, algo, monkeypatch):
    monkeypatch.setenv("TN_SVD_ALGO", algo)
    case = synth.make_config(1)
    got, res = _run(tn, case, 10 ** 6)
    assert res["discarded"] <= 1e-24
    for c in range(case.N + 1):
        if got[c].size:
            rg, _, _ = _recon(case, res, c)
            assert np.linalg.norm(rg - got[c]) <= 1e-12 * np.linalg.norm(got[c])


def test_svd_errors(tn):
    case = synth.make_config(0)
    plan, U, got = gpu_theta(case)
    t = [torch.from_numpy(np.ascontiguousarray(g)).cuda() for g in got]
    ll, lr = torch.from_numpy(case.lam_l).cuda(), torch.from_numpy(case.lam_r).cuda()
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.svd_truncate(plan, t, ll, lr, 0)
    sharded = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, 2, 0)
    with pytest.raises(tn.TnError, match="UNSUPPORTED"):
        tn.svd_truncate(sharded, t, ll, lr, 4)


# ------------------------------------------------------------------ MPO pair plans (oracle.svd.truncate_update2)
def _recon2(c, res, c1, c2, key):
    pl, pr = oracle.sort_pair_bonds(c.q1_l, c.q2_l), oracle.sort_pair_bonds(c.q1_r, c.q2_r)
    rows = pl[oracle.pair_sector_rows(c.q1_l[pl], c.q2_l[pl], c.d, c1, c2)]
    cols = pr[oracle.pair_sector_cols(c.q1_r[pr], c.q2_r[pr], c.d, c1, c2)]
    a = np.nonzero(key == c1 * (c.N + 1) + c2)[0]
    A = c.lam_l[rows][:, None] * res["gamma_k_new"][np.ix_(rows, a)]
    B = res["gamma_k1_new"][np.ix_(a, cols)] * c.lam_r[cols][None, :]
    return (A * res["lam_new"][a][None, :]) @ B, A, B


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("cfg,chi", [(0, 10), (1, 200), (1, 10 ** 6)])
def test_pair_svd_truncate_parity(tn, cfg, chi, algo, monkeypatch):
    monkeypatch.setenv("TN_SVD_ALGO", algo)
    from test_gpu_pair import gpu_theta2
    c = synth.make_pair_config(cfg)
    plan, got = gpu_theta2(tn, c)
    N = c.N
    t = [torch.from_numpy(np.ascontiguousarray(got[(s // (N + 1), s % (N + 1))])).cuda() for s in range((N + 1) ** 2)]
    ll, lr = torch.from_numpy(c.lam_l).cuda(), torch.from_numpy(c.lam_r).cuda()
    res = tn.svd_truncate(plan, t, ll, lr, chi)
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in res.items()}
    ref = osvd.truncate_update2(N, c.d, c.q1_l, c.q2_l, c.q1_r, c.q2_r, got, c.lam_l, c.lam_r, chi)
    assert res["chi"] == ref["chi"]
    assert np.array_equal(res["q_new"], ref["q_new"])
    assert np.array_equal(res["q1_new"], ref["q1_new"]) and np.array_equal(res["q2_new"], ref["q2_new"])
    smax = max(float(s.max()) for s in ref["svals"] if s.size)
    assert np.max(np.abs(res["lam_new"] - ref["lam_new"]), initial=0.0) <= 1e-12 * smax
    tot = sum(np.linalg.norm(x) ** 2 for x in got.values())
    assert abs(res["discarded"] - ref["discarded"]) <= 1e-12 * tot
    for c1 in range(N + 1):
        for c2 in range(N + 1):
            if got[(c1, c2)].size == 0:
                continue
            rg, A, B = _recon2(c, res, c1, c2, res["q_new"])
            rr, *_ = _recon2(c, ref, c1, c2, ref["q_new"])
            assert np.linalg.norm(rg - rr) <= 1e-10 * max(np.linalg.norm(rr), 1e-300), (c1, c2)
            if A.shape[1]:
                assert np.allclose(A.conj().T @ A, np.eye(A.shape[1]), atol=1e-12)
                assert np.allclose(B @ B.conj().T, np.eye(B.shape[0]), atol=1e-12)


@pytest.mark.parametrize("algo", ALGOS)
def test_svd_leaves_theta_intact(tn, algo, monkeypatch):
    monkeypatch.setenv("TN_SVD_ALGO", algo)
    case = synth.make_config(1)
    plan, U, got = gpu_theta(case)
    t = [torch.from_numpy(np.ascontiguousarray(g)).cuda() for g in got]
    before = [x.clone() for x in t]
    tn.svd_truncate(plan, t, torch.from_numpy(case.lam_l).cuda(), torch.from_numpy(case.lam_r).cuda(), 50)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(t, before))


@pytest.mark.parametrize("name,N,d,chi,chi_max", [("N0", 0, 2, (5, 4, 6), 3), ("chi1", 2, 3, (20, 18, 22), 1),
                                                  ("ragged", 3, 2, (37, 29, 41), 25)])
def test_pair_svd_edge_cases(tn, name, N, d, chi, chi_max):
    from test_gpu_pair import gpu_theta2
    c = synth.make_pair_case(N, d, *chi, seed=17, charges="uniform", lam="random")
    plan, got = gpu_theta2(tn, c)
    t = [torch.from_numpy(np.ascontiguousarray(got[(s // (N + 1), s % (N + 1))])).cuda() for s in range((N + 1) ** 2)]
    res = tn.svd_truncate(plan, t, torch.from_numpy(c.lam_l).cuda(), torch.from_numpy(c.lam_r).cuda(), chi_max)
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in res.items()}
    ref = osvd.truncate_update2(N, c.d, c.q1_l, c.q2_l, c.q1_r, c.q2_r, got, c.lam_l, c.lam_r, chi_max)
    assert res["chi"] == ref["chi"] and np.array_equal(res["q_new"], ref["q_new"]), name
    smax = max((float(s.max()) for s in ref["svals"] if s.size), default=1.0)
    assert np.max(np.abs(res["lam_new"] - ref["lam_new"]), initial=0.0) <= 1e-12 * smax
    for c1 in range(N + 1):
        for c2 in range(N + 1):
            if got[(c1, c2)].size:
                rg, _, _ = _recon2(c, res, c1, c2, res["q_new"])
                rr, *_ = _recon2(c, ref, c1, c2, ref["q_new"])
                assert np.linalg.norm(rg - rr) <= 1e-10 * max(np.linalg.norm(rr), 1e-300), (name, c1, c2)


# ------------------------------------------------------------------ right-canonical (B) form, R22
def _recon_b(case, res, c):
    """λl·B^{[k]}_new·B^{[k+1]}_new restricted to Θ(c)'s rows / columns and charge c's new bonds = the truncated Θ(c)."""
    perm_l, off_l = oracle.sort_bonds(case.q_l, case.N)
    perm_r, off_r = oracle.sort_bonds(case.q_r, case.N)
    (r0, r1), (k0, k1) = oracle.sector_ranges(off_l, off_r, case.N, case.d, c)
    rows, cols = perm_l[r0:r1], perm_r[k0:k1]
    a = np.nonzero(res["q_new"] == c)[0]
    A = case.lam_l[rows][:, None] * res["gamma_k_new"][np.ix_(rows, a)]
    B = res["gamma_k1_new"][np.ix_(a, cols)]
    return A @ B, B


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("cfg,chi", [(0, 5), (1, 64), (1, 100000), (2, 300), ("steep", 250)])
def test_svd_truncate_bform_parity(tn, cfg, chi, algo, monkeypatch):
    monkeypatch.setenv("TN_SVD_ALGO", algo)
    case = (synth.make_case(6, 7, 300, 280, 320, seed=44, charges="uniform", lam="steep") if cfg == "steep"
            else synth.make_config(cfg))
    plan, U, got = gpu_theta(case)
    t = [torch.from_numpy(np.ascontiguousarray(g)).cuda() for g in got]
    res = tn.svd_truncate(plan, t, torch.from_numpy(case.lam_l).cuda(), None, chi, form="b")
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in res.items()}
    ref_secs, *_ = oracle_theta(case)
    ref = osvd.truncate_update(case.N, case.d, case.q_l, case.q_r, ref_secs, case.lam_l, case.lam_r, chi, form="b")
    assert res["chi"] == ref["chi"] and np.array_equal(res["q_new"], ref["q_new"])
    smax = max(float(s.max()) for s in ref["svals"] if s.size)
    assert np.max(np.abs(res["lam_new"] - ref["lam_new"]), initial=0.0) <= 1e-12 * smax
    for c in range(case.N + 1):
        if ref_secs[c].size == 0:
            continue
        rg, Bg = _recon_b(case, res, c)
        rr, _ = _recon_b(case, ref, c)
        assert np.linalg.norm(rg - rr) <= 1e-10 * max(np.linalg.norm(rr), 1e-300), c
        if Bg.shape[0]:
            assert np.abs(Bg @ Bg.conj().T - np.eye(Bg.shape[0])).max() <= 1e-12   # V_c† rows orthonormal


def test_ritz_refinement_is_the_default_path(tn, capfd, monkeypatch):
    # config 2 at χ_max 300 and 1024: every Ritz step converges in the refinement (no library SVD), and
    # TN_SVD_PROFILE reports it; the result is the one the parity tests above check
    monkeypatch.setenv("TN_SVD_PROFILE", "1")
    case = synth.make_config(2)
    for chi in (300, 1024):
        _run(tn, case, chi)
        err = capfd.readouterr().err
        line = [x for x in err.splitlines() if "[svd_gram] Ritz:" in x][-1]
        refined, fallbacks = int(line.split()[2]), int(line.split("),")[1].split()[0])
        assert refined > 0 and fallbacks == 0, line
