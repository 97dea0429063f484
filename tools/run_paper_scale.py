"""The paper's largest run size (d = 18, χ = 16384) on one B200: one Θ build (plan + U +
exec, both K4 engines), timed with CUDA events, and checked element-wise against the oracle's
literal sum (oracle.theta_element) on sampled outputs of every sector. Inputs: Gaussian charges
(N = 17 = d − 1), 0.995^i λ, complex-normal Γ masked to the δ-allowed blocks (synth's recipe)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2301_12814_b200 as tn
import synth

N, d, chi = 17, 18, 16384
t0 = time.time()
case = synth.make_case(N, d, chi, chi, chi, seed=408, charges="gauss", lam="geometric", name="paper-scale")
gen_s = time.time() - t0
h = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
gk, gk1, lk, ll, lr = h(case.gamma_k), h(case.gamma_k1), h(case.lam_k), h(case.lam_l), h(case.lam_r)
res = {"N": N, "d": d, "chi": chi, "host_generation_s": round(gen_s, 1)}
for mode in ("dmma", "int8"):
    times = []
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan = tn.Plan(d, N, case.q_l, case.q_c, case.q_r)
        if mode == "int8":
            plan.set_contraction("int8", 6)
        U = tn.build_bs_unitary(plan, case.theta, case.phi)
        out = tn.theta_exec(plan, gk, lk, gk1, ll, lr, U) if rep == 0 else tn.theta_exec(plan, gk, lk, gk1, ll, lr, U, out=out)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        kt = plan.kernel_times()
        f = plan.flops()
        if rep < 2:
            plan.destroy()
    res[mode] = {"ms_per_gate": round(min(times[1:]), 2), "kernels_ms": {k: round(v, 3) for k, v in kt.items()},
                 "useful_tflops": round((f["f_contract"] + f["f_mix"]) / (min(times[1:]) * 1e-3) / 1e12, 2),
                 "theta_elements": int(sum(o.numel() for o in out)), "workspace_gb": round(plan.workspace_bytes() / 1e9, 2)}
    # sampled parity against the literal sum
    ub = [oracle.bs_unitary_block(n, case.theta, case.phi, d) for n in range(min(N, 2 * d - 2) + 1)]
    tables = (tuple(oracle.sort_bonds(q, N)[0] for q in (case.q_l, case.q_c, case.q_r)),
              tuple(oracle.sort_bonds(q, N)[1] for q in (case.q_l, case.q_c, case.q_r)))
    rng = np.random.default_rng(7)
    worst = 0.0
    for c in range(N + 1):
        o = out[c]
        if o.numel() == 0:
            continue
        rms = float(torch.linalg.vector_norm(o)) / np.sqrt(o.numel())
        for _ in range(4):
            a, b = int(rng.integers(o.shape[0])), int(rng.integers(o.shape[1]))
            v = oracle.theta_element(N, d, c, a, b, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                     case.gamma_k1, case.lam_l, case.lam_r, ub, tables)
            worst = max(worst, abs(complex(o[a, b].item()) - v) / max(rms, abs(v)))
    res[mode]["sampled_worst_err_rel_to_sector_rms"] = worst
    plan.destroy()
    del out
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
