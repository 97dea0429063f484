"""Worst per-sector relative Frobenius error of the GPU Θ against the oracle, per config:
configs 0–3 in full (plain, flat λ), config 4 gate 0 on its largest sector plus one low-c and one high-c sector,
MPO pair configs 0–2 in full. One JSON line per case on stdout; --pair-only runs just the pair configs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle
import paper_2301_12814_b200 as tn
import synth
from gpu_util import gpu_theta, oracle_theta, rel_err, to_dev

ONLY_PAIR = "--pair-only" in sys.argv
for cfg in ((0, 1, 2, 3) if not ONLY_PAIR else ()):
    for flat in (False, True):
        case = synth.make_config(cfg, flat=flat)
        ref = oracle_theta(case)[0]
        for eng in (None, ("int8", 6)):
            _, _, got = gpu_theta(case, contraction=eng)
            errs = [rel_err(g, r) for g, r in zip(got, ref)]
            print(json.dumps({"config": cfg, "lambda": "flat" if flat else "as specified",
                              "engine": "dmma" if eng is None else "int8 S=6", "sectors": len(errs),
                              "worst_rel_err": max(errs), "median_rel_err": float(np.median(errs))}), flush=True)


def config4():
    case = synth.make_config(4, gate=0)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    U = tn.build_bs_unitary(plan, case.theta, case.phi)
    t = to_dev(case)
    out = tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)
    torch.cuda.synchronize()
    sizes = [o.numel() for o in out]
    picks = sorted({int(np.argmax(sizes)), case.N // 6, case.N - case.N // 6})
    ref, *_ = oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                   case.gamma_k1, case.lam_l, case.lam_r, case.theta, case.phi, sectors=picks)
    errs = {c: rel_err(out[c].cpu().numpy(), ref[c]) for c in picks}
    print(json.dumps({"config": 4, "gate": 0, "engine": "dmma", "sectors_checked": picks,
                      "rel_err": {str(k): v for k, v in errs.items()}, "worst_rel_err": max(errs.values())}), flush=True)


if not ONLY_PAIR:
    config4()
# MPO pair plans (pair configs 0–2 in full against oracle.theta2_sectors): the K5F one-pass mix (blocks with both
# vectors ≤ 8) and the two-pass K5P mix both run here
import itertools  # noqa: E402
for pcfg in (0, 1, 2):
    c = synth.make_pair_config(pcfg)
    p2 = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)
    U2 = tn.build_bs_unitary(p2, c.theta, c.phi)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    out2 = tn.theta_exec(p2, dv(c.gamma_k), dv(c.lam_k), dv(c.gamma_k1), dv(c.lam_l), dv(c.lam_r), U2)
    torch.cuda.synchronize()
    ref2, *_ = oracle.theta2_sectors(c.N, c.d, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, c.gamma_k, c.lam_k,
                                     c.gamma_k1, c.lam_l, c.lam_r, c.theta, c.phi)
    errs = [rel_err(out2[c1 * (c.N + 1) + c2].cpu().numpy(), ref2[(c1, c2)])
            for c1, c2 in itertools.product(range(c.N + 1), repeat=2) if ref2[(c1, c2)].size]
    print(json.dumps({"pair_config": pcfg, "N": c.N, "d": c.d, "engine": "dmma", "exec_launches": p2.exec_launches(),
                      "sectors": len(errs), "worst_rel_err": max(errs), "median_rel_err": float(np.median(errs))}),
          flush=True)
