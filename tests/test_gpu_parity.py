"""GPU parity: libtn_theta.so (through the C ABI) against the CPU oracle (SURVEY.md §8(c) T1–T14).

Tolerances: bond tables bit-exact; U max-abs ≤ 1e-14 vs 50-digit mpmath; Θ ≤ 1e-10 relative Frobenius
per sector (BASELINE.json north_star), oracle-zero sectors exactly zero, identical (R_c, C_c).
"""
import functools
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_sectors_close, gpu_theta, oracle_theta, rel_err, to_dev

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


@functools.lru_cache(maxsize=None)
def _case(cfg, shuffled=False, flat=False):
    return synth.make_config(cfg, shuffled=shuffled, flat=flat)


@functools.lru_cache(maxsize=None)
def _oracle(cfg, shuffled=False, flat=False):
    return oracle_theta(_case(cfg, shuffled, flat))


# ------------------------------------------------------------------ T1/T2: K1 bond tables, bit-exact
@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("shuffled", [False, True])
def test_k1_tables_bit_exact(tn, cfg, shuffled):
    N, d, ql, qc, qr = synth.make_charges(cfg, shuffled=shuffled)
    plan = tn.Plan(d, N, ql, qc, qr)
    for b, q in enumerate((ql, qc, qr)):
        perm, off = oracle.sort_bonds(q, N)
        assert np.array_equal(plan.perm(b), perm)
        assert np.array_equal(plan.offsets(b), off)


def test_k1_spec_examples_and_device_charges(tn):
    import torch
    plan = tn.Plan(3, 2, [2, 0, 1, 0], torch.tensor([0, 1, 1, 2], dtype=torch.int32, device="cuda"), [0, 1, 1, 2])
    assert plan.perm(0).tolist() == [1, 3, 2, 0]
    assert plan.offsets(0).tolist() == [0, 2, 3, 4]
    assert plan.perm(1).tolist() == [0, 1, 2, 3]                  # SPEC.md:57 (device-resident charges)


def test_k1_large_chi_multi_chunk(tn):
    rng = np.random.default_rng(3)
    q = rng.integers(0, 9, size=100_003).astype(np.int32)
    plan = tn.Plan(9, 8, q, q[:777], q[:5])
    perm, off = oracle.sort_bonds(q, 8)
    assert np.array_equal(plan.perm(0), perm) and np.array_equal(plan.offsets(0), off)


def test_plan_flop_counts_exact(tn):
    want = {0: (14560, 10000), 1: (34023872, 4867904), 2: (1735597600, 142705608),
            3: (102206486240, 8615627728)}
    for cfg, (fc, fm) in want.items():
        N, d, ql, qc, qr = synth.make_charges(cfg)
        f = tn.Plan(d, N, ql, qc, qr).flops()
        assert (f["f_contract"], f["f_mix"]) == (fc, fm)
        assert fc <= f["f_exec"]
        if cfg == 3:                               # executed/useful DMMA flops incl. tile padding
            assert f["f_exec"] <= 1.3 * fc


# ------------------------------------------------------------------ T3/T4: K2 U builder
@functools.lru_cache(maxsize=None)
def _oracle_u(theta, phi, d, N):
    return oracle.packed_u(theta, phi, d, N)


@pytest.mark.parametrize("d", [2, 4, 8, 16])
@pytest.mark.parametrize("theta", [0.0, 0.3, math.pi / 4, 1.3, math.pi / 2 - 1e-3, math.pi / 2])
@pytest.mark.parametrize("phi", [0.0, 0.3, 4.0])
def test_k2_u_vs_mpmath(tn, d, theta, phi):
    N = d - 1
    plan = tn.Plan(d, N, [0], [0], [0])
    U = tn.build_bs_unitary(plan, theta, phi).cpu().numpy()
    ref = _oracle_u(theta, phi, d, N)
    assert U.shape == ref.shape
    assert np.max(np.abs(U - ref)) <= 1e-14


@pytest.mark.parametrize("d,theta,phi", [(32, 0.7, 0.3), (32, 1.3, 4.0), (48, 0.7, 0.3), (48, math.pi / 2 - 1e-3, 4.0),
                                         (48, 0.3, 2.2), (6, 0.9, 1.1)])
def test_k2_u_large_d(tn, d, theta, phi):
    N = d - 1 if d > 6 else 9            # d=6 with N=9: truncated blocks n ≥ d (R6)
    plan = tn.Plan(d, N, [0], [0], [0])
    U = tn.build_bs_unitary(plan, theta, phi).cpu().numpy()
    ref = _oracle_u(theta, phi, d, N)
    assert np.max(np.abs(U - ref)) <= 1e-14
    starts, _ = oracle.packed_u_offsets(d, N)
    for n in range(0, min(N, d - 1) + 1, 7):  # complete blocks are unitary
        s = n + 1
        B = U[starts[n]:starts[n] + s * s].reshape(s, s)
        assert np.max(np.abs(B.conj().T @ B - np.eye(s))) <= 1e-13


def test_k2_rejects_nonfinite(tn):
    plan = tn.Plan(4, 3, [0], [0], [0])
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.build_bs_unitary(plan, float("nan"), 0.0)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.build_bs_unitary(plan, 0.1, float("inf"))


# ------------------------------------------------------------------ T9/T9b: Θ parity
@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
@pytest.mark.parametrize("variant", ["plain", "flat", "shuffled"])
def test_theta_parity(tn, cfg, variant):
    kw = dict(shuffled=variant == "shuffled", flat=variant == "flat")
    case = _case(cfg, **kw)
    ref, perms, offs, _ = _oracle(cfg, **kw)
    plan, U, got = gpu_theta(case)
    for c in range(case.N + 1):
        assert plan.sector_shape(c) == ref[c].shape
    assert_sectors_close(got, ref, TOL, f"config{cfg}-{variant}")


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_theta_parity_flat_per_block(tn, cfg):
    # G12 / T9b: error per (c, c_l, c_r) block with flat λ, so no charge block can hide behind λ decay
    case = _case(cfg, flat=True)
    ref, perms, offs, _ = _oracle(cfg, flat=True)
    _, _, got = gpu_theta(case)
    off_l, _, off_r = offs
    for c in range(case.N + 1):
        (r0, r1), (k0, k1) = oracle.sector_ranges(off_l, off_r, case.N, case.d, c)
        for cl in range(c, min(case.N, c + case.d - 1) + 1):
            for cr in range(max(0, c - case.d + 1), c + 1):
                rs = slice(off_l[cl] - r0, off_l[cl + 1] - r0)
                cs = slice(off_r[cr] - k0, off_r[cr + 1] - k0)
                assert rel_err(got[c][rs, cs], ref[c][rs, cs]) <= TOL, (c, cl, cr)


@pytest.mark.parametrize("gate", [0, 15, 31])
def test_theta_parity_config4_sectors(tn, gate):
    """T9 at config 4 ("config 4 on gates {0, 15, 31}"): the full Θ is built on the GPU at the
    north_star shape, and three whole sectors per gate — the largest R·C sector and one low-c and one high-c
    sector of very different aspect — are compared with the oracle's literal triple loop at ≤ 1e-10 relative
    Frobenius (oracle.theta_sectors(sectors=…), ~30 s of host BLAS per gate); every other sector is sampled
    element-wise (≤ 1e-10 of the sector's RMS), and Σ_c‖Θ(c)‖² is checked against the identity gate at full
    size (d = N+1)."""
    case = synth.make_config(4, gate=gate)
    N, d = case.N, case.d
    plan = tn.Plan(d, N, case.q_l, case.q_c, case.q_r)
    U = tn.build_bs_unitary(plan, case.theta, case.phi)
    t = to_dev(case)
    out = tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)
    torch.cuda.synchronize()
    sizes = [o.numel() for o in out]
    cmax = int(np.argmax(sizes))
    picks = sorted({cmax, N // 6, N - N // 6})
    ub = [oracle.bs_unitary_block(n, case.theta, case.phi, d) for n in range(min(N, 2 * d - 2) + 1)]
    ref, *_ = oracle.theta_sectors(N, d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k, case.gamma_k1,
                                   case.lam_l, case.lam_r, case.theta, case.phi, u_blocks=ub, sectors=picks)
    for c in picks:
        g = out[c].cpu().numpy()
        assert g.shape == ref[c].shape and g.size > 0
        e = rel_err(g, ref[c])
        assert e <= TOL, f"config 4 gate {gate} sector {c}: rel err {e:.3e}"
    # every sector, sampled element-wise against the oracle's single-element sum
    pl = plan.perm(0), plan.perm(1), plan.perm(2)
    of = plan.offsets(0), plan.offsets(1), plan.offsets(2)
    rng = np.random.default_rng(gate)
    for c in range(N + 1):
        R, Cc = out[c].shape
        if R * Cc == 0:
            continue
        scale = float(torch.linalg.norm(out[c])) / math.sqrt(R * Cc)
        for _ in range(4):
            a, b = int(rng.integers(0, R)), int(rng.integers(0, Cc))
            v = oracle.theta_element(N, d, c, a, b, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                     case.gamma_k1, case.lam_l, case.lam_r, ub, (pl, of))
            assert abs(complex(out[c][a, b]) - v) <= TOL * max(scale, 1e-300), (c, a, b)
    s_u = sum(float(torch.linalg.norm(o)) ** 2 for o in out)
    del out
    out_i = tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], tn.build_bs_unitary(plan, 0.0, 0.0))
    s_i = sum(float(torch.linalg.norm(o)) ** 2 for o in out_i)
    assert abs(s_u - s_i) / s_i < 1e-11


# ------------------------------------------------------------------ T10: metamorphic checks
def test_metamorphic_linearity_and_norm(tn):
    case = _case(2)
    plan, U, got = gpu_theta(case)
    c2 = synth.make_config(2)
    c2.gamma_k = c2.gamma_k * (0.5 - 2j)
    _, _, got2 = gpu_theta(c2, plan=plan, U=U)
    for g, h in zip(got, got2):
        assert rel_err(h, g * (0.5 - 2j)) < 1e-13
    _, _, gi = gpu_theta(case, plan=plan, U=tn.build_bs_unitary(plan, 0.0, 0.0))
    su, si = (sum(np.linalg.norm(x) ** 2 for x in v) for v in (got, gi))
    assert abs(su - si) / si < 1e-11


def test_metamorphic_half_pi_swap(tn):
    # θ=π/2: Θ(c)[α,β] = λlλr (−1)^{c−c_r} e^{iφ(c_l+c_r−2c)} P_{c_l+c_r−c}[α,β]
    case = _case(2)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    phi = 0.9
    _, _, sw = gpu_theta(case, plan=plan, U=tn.build_bs_unitary(plan, math.pi / 2, phi))
    _, _, ident = gpu_theta(case, plan=plan, U=tn.build_bs_unitary(plan, 0.0, 0.0))  # P scaled by λlλr
    off_l, off_r, N, d = plan.offsets(0), plan.offsets(2), case.N, case.d
    for c in range(N + 1):
        (r0, r1), (k0, k1) = oracle.sector_ranges(off_l, off_r, N, d, c)
        for cl in range(c, N + 1):
            for cr in range(0, c + 1):
                cc = cl + cr - c
                (q0, _), (p0, _) = oracle.sector_ranges(off_l, off_r, N, d, cc)
                blk = sw[c][off_l[cl] - r0:off_l[cl + 1] - r0, off_r[cr] - k0:off_r[cr + 1] - k0]
                src = ident[cc][off_l[cl] - q0:off_l[cl + 1] - q0, off_r[cr] - p0:off_r[cr + 1] - p0]
                ref = (-1) ** (c - cr) * np.exp(1j * phi * (cl + cr - 2 * c)) * src
                assert rel_err(blk, ref) < 1e-12 or np.linalg.norm(ref) < 1e-300


def test_metamorphic_shuffle_invariance(tn):
    case, cs = _case(1), _case(1, shuffled=True)
    _, _, a = gpu_theta(case)
    _, _, b = gpu_theta(cs)
    # both are in sorted order; the shuffle only permutes equal-charge bonds → compare per sector after
    # mapping each sorted position back to its original generator index
    pa = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    pb = tn.Plan(cs.d, cs.N, cs.q_l, cs.q_c, cs.q_r)
    rng2 = np.random.default_rng(1000 + 1)
    perm_l, perm_c, perm_r = rng2.permutation(cs.chi_l), rng2.permutation(cs.chi_c), rng2.permutation(cs.chi_r)
    orig_l, orig_r = perm_l[pb.perm(0)], perm_r[pb.perm(2)]
    inv_l, inv_r = np.argsort(pa.perm(0)), np.argsort(pa.perm(2))
    for c in range(case.N + 1):
        (r0, _), (k0, _) = oracle.sector_ranges(pa.offsets(0), pa.offsets(2), case.N, case.d, c)
        R, Cc = a[c].shape
        ri = inv_l[orig_l[r0:r0 + R]] - r0
        ci = inv_r[orig_r[k0:k0 + Cc]] - k0
        assert rel_err(b[c], a[c][np.ix_(ri, ci)]) < 1e-13


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_equals_unsharded(tn, world):
    # T12: each rank's plan run on this one GPU in turn (no collective needed for the compute);
    # stacking the slabs reproduces the unsharded Θ bit for bit (same K order per element).
    case = _case(2)
    plan, U, full = gpu_theta(case)
    slabs = [[] for _ in range(case.N + 1)]
    for r in range(world):
        pr = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, r)
        assert pr.shard_rows(r) == tuple(tn.shard_rows_host(
            case.d, case.N, *(np.bincount(q, minlength=case.N + 1) for q in (case.q_l, case.q_c, case.q_r)),
            world)[r:r + 2])
        _, _, loc = gpu_theta(case, world, r, plan=pr)
        for c in range(case.N + 1):
            R, Cc, row0 = pr.local_sector_shape(c)
            assert loc[c].shape == (R, Cc)
            slabs[c].append((row0, loc[c]))
    for c in range(case.N + 1):
        parts = sorted(slabs[c], key=lambda x: x[0])
        stacked = np.concatenate([p for _, p in parts], axis=0)
        assert np.array_equal(stacked, full[c])


# ------------------------------------------------------------------ T13: edge cases
EDGE = {
    "N0": dict(N=0, d=2, chi=(3, 2, 4)),
    "chi1": dict(N=3, d=4, chi=(1, 1, 1)),
    "d_gt_N1": dict(N=4, d=7, chi=(20, 15, 18)),
    "d_lt_N1": dict(N=6, d=3, chi=(40, 33, 29)),
    "ragged": dict(N=5, d=6, chi=(131, 67, 190)),
}


@pytest.mark.parametrize("name", list(EDGE))
def test_edge_cases(tn, name):
    e = EDGE[name]
    case = synth.make_case(e["N"], e["d"], *e["chi"], seed=hash(name) % 1000, charges="uniform", lam="random")
    ref, *_ = oracle_theta(case)
    _, _, got = gpu_theta(case)
    assert_sectors_close(got, ref, 1e-12, name)


def test_edge_single_charge_and_empty_segments(tn):
    case = synth.make_case(6, 7, 50, 40, 45, seed=9, charges="uniform", lam="random")
    case.q_c[:] = np.where(case.q_c == 3, 2, case.q_c)        # empty middle segment c_c = 3
    case.q_c[case.q_c == 5] = 4
    m = lambda a, b: ((a[:, None] - b[None, :] >= 0) & (a[:, None] - b[None, :] <= case.d - 1))
    case.gamma_k *= m(case.q_l, case.q_c)
    case.gamma_k1 *= m(case.q_c, case.q_r)
    case.lam_k[::7] = 0.0                                      # λ containing zeros
    ref, *_ = oracle_theta(case)
    _, _, got = gpu_theta(case)
    assert_sectors_close(got, ref, 1e-12, "empty-segments")
    one = synth.make_case(5, 6, 30, 30, 30, seed=4, charges="single", lam="random")
    ref, *_ = oracle_theta(one)
    _, _, got = gpu_theta(one)
    assert_sectors_close(got, ref, 1e-12, "single-charge")


# ------------------------------------------------------------------ T14: error codes
def test_error_codes(tn):
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.Plan(1, 3, [0], [0], [0])                       # d < 2
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.Plan(4, 3, [0, 4], [0], [0])                    # charge ∉ [0, N]
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.Plan(4, 3, [0, -1], [0], [0])
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.Plan(4, 3, [0], [0], [0], world_size=2, rank=2)
    with pytest.raises(tn.TnError, match="UNSUPPORTED"):
        tn.Plan(70, 69, [0], [0], [0])                     # min(N+1, d) > TN_MAX_MIX
    plan = tn.Plan(4, 3, [0, 1], [0, 1], [0, 1])
    with pytest.raises(tn.TnError, match="DOMAIN"):
        plan.sector_shape(4)                               # c ∉ [0, N]
    with pytest.raises(tn.TnError, match="DOMAIN"):
        plan.sector_shape(-1)
    case = _case(0)
    t = to_dev(case)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    U = tn.build_bs_unitary(plan, case.theta, case.phi)
    outs = tn.alloc_theta(plan)
    outs[1] = None                                         # NULL for a non-empty sector
    with pytest.raises(tn.TnError, match="DIMENSION"):
        tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, out=outs)


# ------------------------------------------------------------------ T10: φ shift; T11: padding invariance
@pytest.mark.parametrize("cfg", [2, 3])
def test_metamorphic_phi_shift(tn, cfg):
    # U_n[i][j] = e^{iφ(i−j)} U_n(θ,0)[i][j] with i − j = c_c − c, so
    # Θ(c; θ, φ) = e^{−iφc} Θ'(c; θ, 0) where Γk1' has row α_k multiplied by e^{iφ q_c[α_k]}.
    case = _case(cfg)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    _, _, got = gpu_theta(case, plan=plan)
    shifted = synth.make_config(cfg)
    shifted.gamma_k1 = shifted.gamma_k1 * np.exp(1j * case.phi * case.q_c)[:, None]
    _, _, got0 = gpu_theta(shifted, plan=plan, U=tn.build_bs_unitary(plan, case.theta, 0.0))
    for c in range(case.N + 1):
        assert rel_err(got[c], np.exp(-1j * case.phi * c) * got0[c]) < 1e-11, c


@pytest.mark.parametrize("cfg,extra", [(1, (37, 61, 45)), (2, (129, 3, 200))])
def test_padding_invariance(tn, cfg, extra):
    # T11: extra bonds move every tile and segment boundary but must not change Θ on the
    # original (α, β). Extra left/right bonds carry random Γ (their rows/cols are new rows/cols of Θ);
    # extra centre bonds carry random Γ but λk = 0, so they add exact zeros to every contraction.
    case = _case(cfg)
    rng = np.random.default_rng(77)
    el, ec, er = extra
    N, d = case.N, case.d
    q = [np.concatenate([qq, rng.integers(0, N + 1, e).astype(np.int32)]) for qq, e in
         zip((case.q_l, case.q_c, case.q_r), extra)]
    allowed = lambda a, b: ((a[:, None] - b[None, :] >= 0) & (a[:, None] - b[None, :] <= d - 1))
    cn = lambda *s: (rng.standard_normal(s) + 1j * rng.standard_normal(s)) / math.sqrt(2)
    gk = cn(case.chi_l + el, case.chi_c + ec)
    gk[:case.chi_l, :case.chi_c] = case.gamma_k
    gk1 = cn(case.chi_c + ec, case.chi_r + er)
    gk1[:case.chi_c, :case.chi_r] = case.gamma_k1
    big = synth.Case("padded", N, d, q[0], q[1], q[2], gk * allowed(q[0], q[1]), gk1 * allowed(q[1], q[2]),
                     np.concatenate([case.lam_l, rng.random(el)]), np.concatenate([case.lam_k, np.zeros(ec)]),
                     np.concatenate([case.lam_r, rng.random(er)]), case.theta, case.phi)
    pa = tn.Plan(d, N, case.q_l, case.q_c, case.q_r)
    pb = tn.Plan(d, N, big.q_l, big.q_c, big.q_r)
    _, _, a = gpu_theta(case, plan=pa)
    _, _, b = gpu_theta(big, plan=pb)
    inv_l, inv_r = np.argsort(pa.perm(0)), np.argsort(pa.perm(2))
    for c in range(N + 1):
        (r0, r1), (k0, k1) = oracle.sector_ranges(pa.offsets(0), pa.offsets(2), N, d, c)
        (s0, s1), (m0, m1) = oracle.sector_ranges(pb.offsets(0), pb.offsets(2), N, d, c)
        bl, br = pb.perm(0)[s0:s1], pb.perm(2)[m0:m1]
        rows = np.nonzero(bl < case.chi_l)[0]
        cols = np.nonzero(br < case.chi_r)[0]
        sub = b[c][np.ix_(rows, cols)]
        ra = inv_l[bl[rows]] - r0
        ca = inv_r[br[cols]] - k0
        assert sub.shape == a[c].shape
        assert rel_err(sub, a[c][np.ix_(ra, ca)]) < 1e-13, c


# ------------------------------------------------------------------ paper-literal ablation engine
@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_paper_literal_engine_parity(tn, cfg):
    # one GEMM per Θ(c) with the per-element U lookup: the same Θ, so the same bar
    case = _case(cfg)
    ref, *_ = _oracle(cfg)
    plan, _, got = gpu_theta(case, contraction=("literal", 0))
    assert plan.contraction()[0] == "literal"
    assert_sectors_close(got, ref, TOL, f"literal config{cfg}")
    f = plan.flops()
    assert f["f_exec"] > f["f_contract"] + f["f_mix"]     # it executes more work than the useful count


def test_paper_literal_engine_edge_cases(tn):
    for name in ("N0", "d_lt_N1", "ragged"):
        e = EDGE[name]
        case = synth.make_case(e["N"], e["d"], *e["chi"], seed=5, charges="uniform", lam="random")
        ref, *_ = oracle_theta(case)
        _, _, got = gpu_theta(case, contraction=("literal", 0))
        assert_sectors_close(got, ref, 1e-12, f"literal {name}")


def test_theta_parity_config4_flat_per_block_sampled(tn):
    # T9b for config 4 (gate 0, flat λ): elements sampled in random (c, c_l, c_r) blocks,
    # each checked against the literal sum relative to its own block's RMS — with flat λ no block's
    # contribution is hidden under the geometric decay
    case = synth.flat_lambda(synth.make_config(4, gate=0))
    plan, U, got = gpu_theta(case)
    pl = plan.perm(0), plan.perm(1), plan.perm(2)
    of = plan.offsets(0), plan.offsets(1), plan.offsets(2)
    ub = [oracle.bs_unitary_block(n, case.theta, case.phi, case.d) for n in range(min(case.N, 2 * case.d - 2) + 1)]
    rng = np.random.default_rng(44)
    N, d = case.N, case.d
    checked, worst = 0, 0.0
    while checked < 200:
        c = int(rng.integers(0, N + 1))
        cl = int(rng.integers(c, min(N, c + d - 1) + 1))
        cr = int(rng.integers(max(0, c - d + 1), c + 1))
        (r0, _), (k0, _) = oracle.sector_ranges(of[0], of[2], N, d, c)
        a0, a1 = int(of[0][cl]) - r0, int(of[0][cl + 1]) - r0
        b0, b1 = int(of[2][cr]) - k0, int(of[2][cr + 1]) - k0
        if a1 <= a0 or b1 <= b0:
            continue
        blk = got[c][a0:a1, b0:b1]
        rms = np.linalg.norm(blk) / math.sqrt(blk.size)
        if rms == 0.0:
            continue
        a, b = int(rng.integers(a0, a1)), int(rng.integers(b0, b1))
        v = oracle.theta_element(N, d, c, a, b, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                 case.gamma_k1, case.lam_l, case.lam_r, ub, (pl, of))
        worst = max(worst, abs(got[c][a, b] - v) / rms)
        checked += 1
    assert worst <= 1e-10, worst
    # and the largest sector in full, block by block (every (c_l, c_r) block ≤ 1e-10 of its own norm)
    cmax = int(np.argmax([g.size for g in got]))
    ref, *_ = oracle.theta_sectors(N, d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k, case.gamma_k1,
                                   case.lam_l, case.lam_r, case.theta, case.phi, u_blocks=ub, sectors=[cmax])
    (r0, _), (k0, _) = oracle.sector_ranges(of[0], of[2], N, d, cmax)
    assert got[cmax].shape == ref[cmax].shape
    for cl in range(cmax, min(N, cmax + d - 1) + 1):
        for cr in range(max(0, cmax - d + 1), cmax + 1):
            rs = slice(int(of[0][cl]) - r0, int(of[0][cl + 1]) - r0)
            cs = slice(int(of[2][cr]) - k0, int(of[2][cr + 1]) - k0)
            assert rel_err(got[cmax][rs, cs], ref[cmax][rs, cs]) <= TOL, (cmax, cl, cr)


def test_exec_launch_count(tn):
    # tn_plan_exec_launches (bench.py's gpu_launches): k_set_sectors + K3 a/b + K4 + one K5 launch per non-empty
    # L class; config 3 has blocks in the L ≤ 8, ≤ 16 and ≤ 32 classes (the ncu launch list of bench.py shows the
    # same 9 launches per step with K1 and K2: profiles/r02_launches.csv)
    N, d, ql, qc, qr = synth.make_charges(3)
    plan = tn.Plan(d, N, ql, qc, qr)
    assert plan.exec_launches() == 7
    plan.set_contraction("int8", 6)
    assert plan.exec_launches() == 9                 # set, K3O ×4, K4O, K5 ×3
    plan.set_contraction("literal")
    assert plan.exec_launches() == 4                 # set, K3L a/b, K4L (no mix)
    c = synth.make_pair_config(1)
    p2 = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)
    # set, K3 a/b, K4 and one K5F launch: at d = 5 every (l, r) block has L1, L2 ≤ 8, so both species are mixed in
    # one pass (no two-pass K5P launches)
    assert p2.exec_launches() == 5


def test_exec_captured_in_cuda_graph(tn):
    # tn_theta_exec is stream-ordered, so it can be captured into a CUDA graph (its K3/K5 launches fork onto
    # auxiliary streams and join back, which capture records as graph branches) and replayed bit-identically
    case = _case(2)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    U = tn.build_bs_unitary(plan, case.theta, case.phi)
    t = to_dev(case)
    ref = [x.clone() for x in tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)]
    out = tn.alloc_theta(plan)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):          # warm-up outside capture (lazy per-thread stream creation)
        tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, out=out, stream=s)
    torch.cuda.synchronize()
    for o in out:
        o.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, out=out, stream=s)
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(out, ref):
        assert torch.equal(a, b)
