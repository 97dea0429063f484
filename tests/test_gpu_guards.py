"""Out-of-bounds write checks (stand-in for SURVEY T15: compute-sanitizer is not available on this GPU pool).

Every output buffer the library writes — each Θ(c) slab, the SVD step's q/λ/Γ outputs — is carved out of one
allocation with guard zones before and after it, all filled with a sentinel bit pattern; after the call
every guard must still hold the sentinel, and the read-only inputs (Γ, λ, U) must be unchanged. The
inputs themselves sit between NaN guard zones, and the result must equal a run on plain buffers bit for
bit (an out-of-bounds READ reaching a guard would turn it into NaN). Covers the
FP64 DMMA, INT8-emulation and paper-literal engines, MPO pair plans, sharded slabs, edge shapes and the SVD
step."""
import ctypes as C

import numpy as np
import pytest
import torch

import synth
from gpu_util import to_dev

pytestmark = pytest.mark.gpu
GUARD = 4099                                  # complex entries per guard zone (odd, so misalignment shows)
SENT = complex(1.2345678901234567e300, -7.654321e-300)


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


def _guarded(shapes, dtype=torch.complex128, sent=SENT):
    """One device allocation: guard, buf0, guard, buf1, …, guard; returns (big, views, guard slices)."""
    n = [int(np.prod(s)) for s in shapes]
    total = GUARD * (len(shapes) + 1) + sum(n)
    big = torch.full((total,), sent, dtype=dtype, device="cuda")
    views, guards, off = [], [(0, GUARD)], GUARD
    for s, k in zip(shapes, n):
        views.append(big[off:off + k].view(*s) if k else None)
        off += k
        guards.append((off, off + GUARD))
        off += GUARD
    return big, views, guards


def _check_guards(big, guards, sent=SENT, what=""):
    for a, b in guards:
        assert bool((big[a:b] == sent).all().item()), f"{what}: guard [{a}, {b}) overwritten"


def _nan_guarded(t):
    """A copy of device tensor t inside an allocation whose guard zones hold NaN (an out-of-bounds READ
    that reaches them turns the result into NaN)."""
    nan = complex("nan+nanj") if t.is_complex() else float("nan")
    big, (v,), _ = _guarded([tuple(t.shape)], dtype=t.dtype, sent=nan)
    v.copy_(t)
    return big, v


def _exec_guarded(tn, plan, case, U):
    shapes = [plan.local_sector_shape(c)[:2] for c in range(plan.nsec)]
    big, views, guards = _guarded(shapes)
    t = to_dev(case)
    ref = tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)   # plain buffers
    keep, g = [], {}
    for k, v in t.items():
        b, g[k] = _nan_guarded(v)
        keep.append(b)
    bu, Ug = _nan_guarded(U)
    out = [v if v is not None else torch.empty((0, 0), dtype=torch.complex128, device="cuda") for v in views]
    tn.theta_exec(plan, g["gk"], g["lk"], g["gk1"], g["ll"], g["lr"], Ug, out=out)
    torch.cuda.synchronize()
    _check_guards(big, guards, what="Θ slabs")
    for k, v in t.items():
        assert torch.equal(g[k], v), f"input {k} modified"
    assert torch.equal(Ug, U), "U modified"
    for c, (a, r) in enumerate(zip(out, ref)):   # NaN guards never reached: identical results
        if a.numel() or r.numel():
            assert torch.equal(a, r), f"sector {c} differs with NaN-guarded inputs"
    return out


@pytest.mark.parametrize("cfg,engine", [(0, None), (1, None), (2, None), (3, None), (1, ("int8", 6)), (2, ("int8", 6)),
                                        (3, ("int8", 6)), (1, ("literal",)), (2, ("literal",))])
def test_theta_exec_writes_stay_in_bounds(tn, cfg, engine):
    case = synth.make_config(cfg)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    if engine:
        plan.set_contraction(*engine)
    _exec_guarded(tn, plan, case, tn.build_bs_unitary(plan, case.theta, case.phi))


@pytest.mark.parametrize("N,d,chi", [(0, 2, (3, 4, 5)), (3, 2, (40, 33, 29)), (2, 5, (30, 31, 32)), (5, 3, (61, 1, 47))])
def test_edge_shapes_write_in_bounds(tn, N, d, chi):
    case = synth.make_case(N, d, *chi, seed=41, charges="uniform", lam="random")
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    _exec_guarded(tn, plan, case, tn.build_bs_unitary(plan, case.theta, case.phi))


@pytest.mark.parametrize("world,rank", [(3, 0), (3, 1), (3, 2)])
def test_sharded_slabs_write_in_bounds(tn, world, rank):
    case = synth.make_config(2)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, rank)
    _exec_guarded(tn, plan, case, tn.build_bs_unitary(plan, case.theta, case.phi))


@pytest.mark.parametrize("cfg", [0, 1])
def test_pair_plan_writes_in_bounds(tn, cfg):
    c = synth.make_pair_config(cfg)
    plan = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)
    shapes = [plan.local_sector_shape(s)[:2] for s in range(plan.nsec)]
    big, views, guards = _guarded(shapes)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    U = tn.build_bs_unitary(plan, c.theta, c.phi)
    out = [v if v is not None else torch.empty((0, 0), dtype=torch.complex128, device="cuda") for v in views]
    tn.theta_exec(plan, dv(c.gamma_k), dv(c.lam_k), dv(c.gamma_k1), dv(c.lam_l), dv(c.lam_r), U, out=out)
    torch.cuda.synchronize()
    _check_guards(big, guards, what="pair Θ slabs")


@pytest.mark.parametrize("algo", ["gram", "gesvdp", "gesvdj"])
@pytest.mark.parametrize("chi_max", [7, 64, 100000])
def test_svd_outputs_write_in_bounds(tn, algo, chi_max, monkeypatch):
    monkeypatch.setenv("TN_SVD_ALGO", algo)
    case = synth.make_config(1)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    theta = _exec_guarded(tn, plan, case, tn.build_bs_unitary(plan, case.theta, case.phi))
    chi_l, _, chi_r = plan.chi
    cap = min(chi_max, sum(min(plan.sector_shape(c)) for c in range(plan.nsec)))
    bigc, (gk, gk1), gc = _guarded([(chi_l, cap), (cap, chi_r)])
    bigd, (lam,), gd = _guarded([(cap,)], dtype=torch.float64, sent=1.5e300)
    bigi, (q,), gi = _guarded([(cap,)], dtype=torch.int32, sent=-123456789)
    ll, lr = torch.from_numpy(case.lam_l).cuda(), torch.from_numpy(case.lam_r).cuda()
    chi_out, disc = C.c_int64(), C.c_double()
    tn.check(tn.lib.tn_svd_truncate(plan.handle, tn._stream_ptr(None), tn._theta_ptrs(theta), tn._ptr(ll), tn._ptr(lr),
                                    int(cap), 1e-14, tn._ptr(q), tn._ptr(lam), tn._ptr(gk), tn._ptr(gk1),
                                    C.byref(chi_out), C.byref(disc)), "tn_svd_truncate")
    torch.cuda.synchronize()
    assert 0 < chi_out.value <= cap
    _check_guards(bigc, gc, what="Γ_new")
    _check_guards(bigd, gd, sent=1.5e300, what="λ_new")
    _check_guards(bigi, gi, sent=-123456789, what="q_new")
