"""Gates in flight: time K config-3 gates (plan + U + exec each) with 1, 2 or 3 streams in rotation
(independent gates, as within a brick-wall layer) — does K5 of gate g overlap K4 of gate g+1?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2301_12814_b200 as tn
import synth

case = synth.make_config(int(os.environ.get("CFG", "3")))
h = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
gk, gk1, lk, ll, lr = h(case.gamma_k), h(case.gamma_k1), h(case.lam_k), h(case.lam_l), h(case.lam_r)
ql, qc, qr = h(case.q_l), h(case.q_c), h(case.q_r)
probe = tn.Plan(case.d, case.N, ql, qc, qr)
f = probe.flops()
K = 20
for ns in (1, 2, 3):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    outs = [tn.alloc_theta(probe) for _ in range(ns)]
    Us = [torch.empty(probe.u_size(), dtype=torch.complex128, device="cuda") for _ in range(ns)]
    keep = []
    main = torch.cuda.current_stream()
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for st in streams:
            st.wait_stream(main)
        for g in range(K):
            i = g % ns
            with torch.cuda.stream(streams[i]):
                p = tn.Plan(case.d, case.N, ql, qc, qr)
                tn.build_bs_unitary(p, case.theta, case.phi, out=Us[i], stream=streams[i])
                tn.theta_exec(p, gk, lk, gk1, ll, lr, Us[i], out=outs[i], stream=streams[i])
            keep.append(p)
            if len(keep) > 2 * ns:
                keep.pop(0).destroy()
        for st in streams:
            main.wait_stream(st)
        e1.record(main)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
    for p in keep:
        p.destroy()
    print(json.dumps({"streams": ns, "ms_per_gate": round(ms, 4),
                      "useful_tflops": round((f["f_contract"] + f["f_mix"]) / (ms * 1e-3) / 1e12, 2)}), flush=True)
