"""Time the SVD step (tn_svd_truncate) after one Θ build of a BASELINE config on cuda:0."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2301_12814_b200 as tn
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--chi", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
case = synth.make_config(a.config)
h = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
gk, gk1, lk, ll, lr = h(case.gamma_k), h(case.gamma_k1), h(case.lam_k), h(case.lam_l), h(case.lam_r)
plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
U = tn.build_bs_unitary(plan, case.theta, case.phi)
for r in range(a.reps):
    out = tn.theta_exec(plan, gk, lk, gk1, ll, lr, U)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = tn.svd_truncate(plan, out, ll, lr, a.chi)
    e1.record()
    torch.cuda.synchronize()
    shapes = [plan.sector_shape(c) for c in range(case.N + 1)]
    print(json.dumps({"rep": r, "config": a.config, "chi_max": a.chi, "svd_ms": round(e0.elapsed_time(e1), 2),
                      "wall_ms": round((time.perf_counter() - t0) * 1e3, 2), "chi_kept": res["chi"],
                      "discarded": res["discarded"], "largest_sector": max(shapes, key=lambda s: s[0] * s[1]),
                      "sum_min_dim": int(sum(min(s) for s in shapes))}), flush=True)
