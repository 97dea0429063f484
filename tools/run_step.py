"""Run `--reps` full Θ steps (plan + U + exec) of a BASELINE config on cuda:0 — the command profiled by
ncu (launch list and --set full captures under profiles/). Prints per-kernel CUDA-event times."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2301_12814_b200 as tn
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--gate", type=int, default=0)
ap.add_argument("--contraction", default="dmma")
ap.add_argument("--slices", type=int, default=7)
a = ap.parse_args()

case = synth.make_config(a.config, gate=a.gate)
h = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
gk, gk1, lk, ll, lr = h(case.gamma_k), h(case.gamma_k1), h(case.lam_k), h(case.lam_l), h(case.lam_r)
ql, qc, qr = h(case.q_l), h(case.q_c), h(case.q_r)
outs = None
U = None
import time
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = tn.Plan(case.d, case.N, ql, qc, qr)
    plan.set_contraction(a.contraction, a.slices)
    t_plan = (time.perf_counter() - t0) * 1e3
    if outs is None:
        outs = tn.alloc_theta(plan)
        U = torch.empty(plan.u_size(), dtype=torch.complex128, device="cuda")
    tn.build_bs_unitary(plan, case.theta, case.phi, out=U)
    tn.theta_exec(plan, gk, lk, gk1, ll, lr, U, out=outs)
    torch.cuda.synchronize()
    print(json.dumps({"rep": r, "config": a.config, "plan_wall_ms": round(t_plan, 3), **{k: round(v, 4) for k, v in plan.kernel_times().items()},
                      "flops": plan.flops()}))
    plan.destroy()
