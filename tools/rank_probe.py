"""Where a world-R rank's step time goes (bench.py's multi_gpu_projection): for each rank r of a world-R row
sharding of config 3, the steady-state step (a) with a fresh tn_theta_plan per gate and (b) re-using one plan
(U + exec only), timed with CUDA events on the exec stream; host time of each call. One GPU, ranks in turn."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2301_12814_b200 as tn
import synth

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
STEPS = 30
case = synth.make_config(3)
h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
gk, gk1, lk, ll, lr = (h(x) for x in (case.gamma_k, case.gamma_k1, case.lam_k, case.lam_l, case.lam_r))
hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
s = torch.cuda.current_stream()
U = torch.empty(20000, dtype=torch.complex128, device="cuda")
for r in range(R):
    probe = tn.Plan(case.d, case.N, *hq, R, r)
    outs = tn.alloc_theta(probe)
    res = {"rank": r}
    for mode in ("fresh_plan", "reused_plan"):
        hp, hu, he, hd = [], [], [], []
        keep = []
        for it in range(STEPS + 5):
            if it == 5:
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
            t0 = time.perf_counter()
            p = tn.Plan(case.d, case.N, *hq, R, r) if mode == "fresh_plan" else probe
            t1 = time.perf_counter()
            tn.build_bs_unitary(p, case.theta, case.phi, out=U)
            t2 = time.perf_counter()
            tn.theta_exec(p, gk, lk, gk1, ll, lr, U, out=outs)
            t3 = time.perf_counter()
            if mode == "fresh_plan":
                keep.append(p)
                if len(keep) > 2:
                    keep.pop(0).destroy()
            t4 = time.perf_counter()
            if it >= 5:
                hp.append(t1 - t0); hu.append(t2 - t1); he.append(t3 - t2); hd.append(t4 - t3)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(s)
        torch.cuda.synchronize()
        for p in keep:
            p.destroy()
        kt = probe.kernel_times() if mode == "reused_plan" else None
        med = lambda v: round(statistics.median(v) * 1e3, 4)
        res[mode] = {"device_ms_per_step": round(e0.elapsed_time(e1) / STEPS, 4), "host_plan_ms": med(hp),
                     "host_U_ms": med(hu), "host_exec_ms": med(he), "host_destroy_ms": med(hd),
                     "kernels": {k: round(v, 4) for k, v in kt.items()} if kt else None}
    res["rows"] = probe.shard_rows(r)
    res["exec_launches"] = probe.exec_launches()
    print(json.dumps(res), flush=True)
    probe.destroy()
    del outs
