"""GPU parity of the MPO (doubled-charge) path Θ(c1, c2) (tn_theta2_plan + tn_theta_exec) against the
pinned pair oracle (oracle/theta2.py): bond tables bit-exact, sector shapes identical, Θ ≤ 1e-10 relative
Frobenius per sector (the north_star bar carried over), plus the vectorized-pure-state factorisation
against the single-charge GPU path at sizes the literal pair loop cannot reach."""
import functools
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_theta2(tn, case, contraction=None, plan=None, theta=None):
    if plan is None:
        plan = tn.Plan2(case.d, case.N, case.q1_l, case.q2_l, case.q1_c, case.q2_c, case.q1_r, case.q2_r)
    if contraction is not None:
        plan.set_contraction(*contraction)
    U = tn.build_bs_unitary(plan, case.theta if theta is None else theta, case.phi)
    out = tn.theta_exec(plan, _dev(case.gamma_k), _dev(case.lam_k), _dev(case.gamma_k1), _dev(case.lam_l),
                        _dev(case.lam_r), U)
    torch.cuda.synchronize()
    N = case.N
    return plan, {(c1, c2): out[c1 * (N + 1) + c2].cpu().numpy() for c1, c2 in itertools.product(range(N + 1), repeat=2)}


@functools.lru_cache(maxsize=None)
def _pair(cfg):
    return synth.make_pair_config(cfg)


@functools.lru_cache(maxsize=None)
def _oracle2(cfg):
    c = _pair(cfg)
    return oracle.theta2_sectors(c.N, c.d, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, c.gamma_k, c.lam_k,
                                 c.gamma_k1, c.lam_l, c.lam_r, c.theta, c.phi)


def _check(got, ref, tol, what):
    worst = 0.0
    for key, r in ref.items():
        g = got[key]
        assert g.shape == r.shape, (what, key, g.shape, r.shape)
        e = rel_err(g, r)
        assert e <= tol, f"{what} sector {key}: {e:.3e}"
        worst = max(worst, e)
    return worst


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_pair_tables_bit_exact(tn, cfg):
    c = _pair(cfg)
    plan = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)
    nk = c.N + 1
    for b, (q1, q2) in enumerate(((c.q1_l, c.q2_l), (c.q1_c, c.q2_c), (c.q1_r, c.q2_r))):
        assert np.array_equal(plan.perm(b), oracle.sort_pair_bonds(q1, q2))
        key = q1.astype(np.int64) * nk + q2
        ref = np.concatenate([[0], np.cumsum(np.bincount(key, minlength=nk * nk))]).astype(np.int32)
        assert np.array_equal(plan.offsets(b), ref)
    perms = tuple(oracle.sort_pair_bonds(*q) for q in ((c.q1_l, c.q2_l), (c.q1_c, c.q2_c), (c.q1_r, c.q2_r)))
    for c1, c2 in itertools.product(range(nk), repeat=2):
        rows = oracle.pair_sector_rows(c.q1_l[perms[0]], c.q2_l[perms[0]], c.d, c1, c2)
        cols = oracle.pair_sector_cols(c.q1_r[perms[2]], c.q2_r[perms[2]], c.d, c1, c2)
        assert plan.sector_shape(plan.sector(c1, c2)) == (len(rows), len(cols))
    fc, fm = oracle.flop_counts2(c.N, c.d, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)
    f = plan.flops()
    assert (f["f_contract"], f["f_mix"]) == (fc, fm)


@pytest.mark.parametrize("mix", ["default", "two_pass"])
@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_pair_parity(tn, cfg, mix, monkeypatch):
    # default: these small-d configs are mixed by K5F (one pass, both species); two_pass: TN_PAIR_TWO_PASS=1 sends
    # every block through the two K5P passes instead — both against the oracle
    if mix == "two_pass":
        monkeypatch.setenv("TN_PAIR_TWO_PASS", "1")
    ref, *_ = _oracle2(cfg)
    plan, got = gpu_theta2(tn, _pair(cfg))
    # set + K3 a/b + K4, then one K5F launch, or at least one launch per K5P pass
    assert plan.exec_launches() == 5 if mix == "default" else plan.exec_launches() >= 6
    _check(got, ref, TOL, f"pair config {cfg} ({mix})")


@pytest.mark.parametrize("cfg", [1, 2])
def test_pair_parity_int8(tn, cfg):
    ref, *_ = _oracle2(cfg)
    _, got = gpu_theta2(tn, _pair(cfg), contraction=("int8", 6))
    _check(got, ref, TOL, f"pair config {cfg} int8")


def test_pair_config3_sampled(tn):
    c = _pair(3)
    plan, got = gpu_theta2(tn, c)
    ub = [oracle.bs_unitary_block(n, c.theta, c.phi, c.d) for n in range(min(c.N, 2 * c.d - 2) + 1)]
    perms = tuple(oracle.sort_pair_bonds(*q) for q in ((c.q1_l, c.q2_l), (c.q1_c, c.q2_c), (c.q1_r, c.q2_r)))
    rng = np.random.default_rng(5)
    for key in [(0, 0), (2, 3), (3, 2), (5, 5), (1, 4)]:
        g = got[key]
        if g.size == 0:
            continue
        for _ in range(6):
            a, b = int(rng.integers(g.shape[0])), int(rng.integers(g.shape[1]))
            v = oracle.theta2_element(c.N, c.d, *key, a, b, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r,
                                      c.gamma_k, c.lam_k, c.gamma_k1, c.lam_l, c.lam_r, ub, perms)
            scale = np.linalg.norm(g) / np.sqrt(g.size)       # element error relative to the sector's rms
            assert abs(g[a, b] - v) <= 1e-10 * max(scale, abs(v)), (key, a, b)


@pytest.mark.parametrize("cfg", [4, 5])
def test_pair_paper_charge_ranges_sampled(tn, cfg):
    # PAIR_CONFIGS 4/5: d = 14 and d = 18, N = 13 / 17 — 196 / 324 pair keys, beyond
    # round 1's by-value sector tables (N ≤ 9). Pair-key tables bit-exact; every sector shape as the oracle's row /
    # column rule; 40 sectors sampled element-wise against the literal pair sum (≤ 1e-10 of the sector's RMS).
    c = _pair(cfg)
    nk = c.N + 1
    plan, got = gpu_theta2(tn, c)
    perms = tuple(oracle.sort_pair_bonds(*q) for q in ((c.q1_l, c.q2_l), (c.q1_c, c.q2_c), (c.q1_r, c.q2_r)))
    for b, (q1, q2) in enumerate(((c.q1_l, c.q2_l), (c.q1_c, c.q2_c), (c.q1_r, c.q2_r))):
        assert np.array_equal(plan.perm(b), perms[b])
        key = q1.astype(np.int64) * nk + q2
        ref = np.concatenate([[0], np.cumsum(np.bincount(key, minlength=nk * nk))]).astype(np.int32)
        assert np.array_equal(plan.offsets(b), ref)
    ub = [oracle.bs_unitary_block(n, c.theta, c.phi, c.d) for n in range(min(c.N, 2 * c.d - 2) + 1)]
    rng = np.random.default_rng(50 + cfg)
    keys = [k for k, g in got.items() if g.size > 0]
    assert len(keys) > 100
    for i in rng.permutation(len(keys))[:40]:
        key = keys[int(i)]
        g = got[key]
        rows = oracle.pair_sector_rows(c.q1_l[perms[0]], c.q2_l[perms[0]], c.d, *key)
        cols = oracle.pair_sector_cols(c.q1_r[perms[2]], c.q2_r[perms[2]], c.d, *key)
        assert g.shape == (len(rows), len(cols))
        scale = np.linalg.norm(g) / np.sqrt(g.size)
        for _ in range(3):
            a, b = int(rng.integers(g.shape[0])), int(rng.integers(g.shape[1]))
            v = oracle.theta2_element(c.N, c.d, *key, a, b, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r,
                                      c.gamma_k, c.lam_k, c.gamma_k1, c.lam_l, c.lam_r, ub, perms)
            assert abs(g[a, b] - v) <= 1e-10 * max(scale, abs(v)), (key, a, b)
    # U⊗U* is unitary on every pair block: Σ‖Θ‖² with the gate equals Σ‖Θ‖² with the identity (d = N+1)
    s_u = sum(np.linalg.norm(g) ** 2 for g in got.values())
    _, got_i = gpu_theta2(tn, c, plan=plan, theta=0.0)
    s_i = sum(np.linalg.norm(g) ** 2 for g in got_i.values())
    assert abs(s_u - s_i) <= 1e-11 * s_i


def test_pair_vectorized_pure_state_matches_single_path(tn):
    # Θ2(c1,c2)[(α,α'),(β,β')] = Θ(c1)[α,β]·conj(Θ(c2)[α',β']) — both sides on the GPU, at χ = 24 → 576 pairs
    base = synth.make_case(4, 5, 24, 24, 24, seed=21, charges="uniform", lam="random")
    vec = synth.vectorize_pure(base)
    from gpu_util import gpu_theta
    p1, _, s1 = gpu_theta(base)
    p2, s2 = gpu_theta2(tn, vec)
    pl1, pr1, pl2, pr2 = p1.perm(0), p1.perm(2), p2.perm(0), p2.perm(2)
    inv_l, inv_r = np.argsort(pl1), np.argsort(pr1)
    off_l, off_r = p1.offsets(0), p1.offsets(2)
    N, d, chi = base.N, base.d, 24
    for c1, c2 in itertools.product(range(N + 1), repeat=2):
        rows = oracle.pair_sector_rows(vec.q1_l[pl2], vec.q2_l[pl2], d, c1, c2)
        cols = oracle.pair_sector_cols(vec.q1_r[pr2], vec.q2_r[pr2], d, c1, c2)
        g = s2[(c1, c2)]
        assert g.shape == (len(rows), len(cols))
        if g.size == 0:
            continue
        (a0, _), (b0, _) = oracle.sector_ranges(off_l, off_r, N, d, c1)
        (e0, _), (f0, _) = oracle.sector_ranges(off_l, off_r, N, d, c2)
        al, alp = np.divmod(pl2[rows].astype(np.int64), chi)
        be, bep = np.divmod(pr2[cols].astype(np.int64), chi)
        ref = s1[c1][np.ix_(inv_l[al] - a0, inv_r[be] - b0)] * np.conj(s1[c2][np.ix_(inv_l[alp] - e0, inv_r[bep] - f0)])
        assert rel_err(g, ref) < 1e-12, (c1, c2)


@pytest.mark.parametrize("name,N,d,chi", [("N0", 0, 2, (3, 4, 5)), ("d_lt_N1", 3, 2, (40, 33, 29)),
                                          ("d_gt_N1", 2, 5, (30, 31, 32)), ("ragged", 3, 4, (77, 65, 90))])
def test_pair_edge_cases(tn, name, N, d, chi):
    case = synth.make_pair_case(N, d, *chi, seed=31, charges="uniform", lam="random")
    ref, *_ = oracle.theta2_sectors(case.N, case.d, case.q1_l, case.q2_l, case.q1_c, case.q2_c, case.q1_r,
                                    case.q2_r, case.gamma_k, case.lam_k, case.gamma_k1, case.lam_l, case.lam_r,
                                    case.theta, case.phi)
    _, got = gpu_theta2(tn, case)
    _check(got, ref, 1e-12, name)


def test_pair_errors(tn):
    with pytest.raises(tn.TnError, match="UNSUPPORTED"):
        tn.Plan2(33, 32, [0], [0], [0], [0], [0], [0])        # (N+1)^2 = 1089 sectors beyond this build (≤ 1024)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.Plan2(4, 3, [0, 4], [0, 0], [0], [0], [0], [0])    # charge outside [0, N]
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.Plan2(4, 3, [0], [-1], [0], [0], [0], [0])
    plan = tn.Plan2(4, 3, [0, 1], [1, 0], [0, 1], [0, 1], [0, 1], [1, 1])
    with pytest.raises(tn.TnError, match="DOMAIN"):
        plan.sector_shape(16)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_pair_sharded_equals_unsharded(tn, world):
    # each rank's row slab of every Θ(c1,c2) (its plan run in turn on this one GPU, no collective needed):
    # the slabs tile the sector rows and reproduce the unsharded Θ bit for bit
    c = _pair(2)
    _, full = gpu_theta2(tn, c)
    dv = lambda a: _dev(a)
    slabs = {k: [] for k in full}
    f_loc = 0
    for r in range(world):
        pr = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, world, r)
        U = tn.build_bs_unitary(pr, c.theta, c.phi)
        out = tn.theta_exec(pr, dv(c.gamma_k), dv(c.lam_k), dv(c.gamma_k1), dv(c.lam_l), dv(c.lam_r), U)
        torch.cuda.synchronize()
        f_loc += pr.flops()["f_contract_local"]
        for (c1, c2) in full:
            s = pr.sector(c1, c2)
            R, Cc, row0 = pr.local_sector_shape(s)
            assert tuple(out[s].shape) == (R, Cc)
            slabs[(c1, c2)].append((row0, out[s].cpu().numpy()))
    assert f_loc == pr.flops()["f_contract"]
    for key, parts in slabs.items():
        parts = sorted((p for p in parts if p[1].shape[0] > 0), key=lambda x: x[0])
        pos = 0
        for b, blk in parts:
            assert b == pos
            pos += blk.shape[0]
        assert pos == full[key].shape[0]
        if parts:
            assert np.array_equal(np.concatenate([p for _, p in parts], axis=0), full[key]), key


@pytest.mark.parametrize("world", [2, 3, 5])
def test_gather_placement_and_owners(tn, world):
    # what tn_theta_exec_sharded's ROOT / SECTOR_OWNER gathers use for every source rank: tn_plan_slab_rows
    # must place rank r's slab exactly where rank r's own plan says it starts (tn_plan_local_sector_shape),
    # for MPO pair plans and single-charge plans; pair-plan owners follow the LPT rule over (N+1)² sectors
    c = _pair(2)
    plans = [tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, world, r) for r in range(world)]
    s1 = synth.make_config(2)
    singles = [tn.Plan(s1.d, s1.N, s1.q_l, s1.q_c, s1.q_r, world, r) for r in range(world)]
    for ps in (plans, singles):
        for s in range(ps[0].nsec):
            R, _ = ps[0].sector_shape(s)
            pos = 0
            for r in range(world):
                Rl, _, b = ps[r].local_sector_shape(s)
                got = ps[0].slab_rows(s, r)
                if Rl:
                    assert got == (b, Rl), (s, r)
                    assert b == pos
                    pos += Rl
                else:
                    assert got[1] == 0
            assert pos == R, s
    sizes = [int(np.prod(plans[0].sector_shape(s))) for s in range(plans[0].nsec)]
    want = tn.sector_owners_host(sizes, world)
    assert [plans[0].sector_owner(s) for s in range(plans[0].nsec)] == list(want)
