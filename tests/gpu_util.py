"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI and compare with the oracle."""
import numpy as np
import torch

import oracle


def to_dev(case):
    dv = "cuda"
    return dict(gk=torch.from_numpy(np.ascontiguousarray(case.gamma_k)).to(dv),
                gk1=torch.from_numpy(np.ascontiguousarray(case.gamma_k1)).to(dv),
                lk=torch.from_numpy(np.ascontiguousarray(case.lam_k)).to(dv),
                ll=torch.from_numpy(np.ascontiguousarray(case.lam_l)).to(dv),
                lr=torch.from_numpy(np.ascontiguousarray(case.lam_r)).to(dv))


def gpu_theta(case, world_size=1, rank=0, U=None, plan=None, contraction=None):
    """(plan, U, list of numpy sector slabs) computed entirely by libtn_theta.so.
    `contraction` = None (plan default, FP64 DMMA) or ("int8", slices) for the tcgen05 INT8 emulation."""
    import paper_2301_12814_b200 as tn
    if plan is None:
        plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world_size, rank)
    if contraction is not None:
        plan.set_contraction(*contraction)
    if U is None:
        U = tn.build_bs_unitary(plan, case.theta, case.phi)
    t = to_dev(case)
    out = tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)
    torch.cuda.synchronize()
    return plan, U, [o.cpu().numpy() for o in out]


def oracle_theta(case, theta=None):
    th = case.theta if theta is None else theta
    return oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                case.gamma_k1, case.lam_l, case.lam_r, th, case.phi)


def rel_err(got, ref):
    """Relative Frobenius error per sector; an oracle-zero sector must be exactly zero."""
    n = np.linalg.norm(ref)
    if n == 0:
        return 0.0 if np.all(got == 0) else np.inf
    return float(np.linalg.norm(got - ref) / n)


def assert_sectors_close(got, ref, tol, what=""):
    assert len(got) == len(ref)
    worst = 0.0
    for c, (g, r) in enumerate(zip(got, ref)):
        assert g.shape == r.shape, (what, c, g.shape, r.shape)
        e = rel_err(g, r)
        assert e <= tol, f"{what} sector {c}: rel err {e:.3e} > {tol}"
        worst = max(worst, e)
    return worst
