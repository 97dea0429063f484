"""Host wall time of tn_theta_plan (Plan()) at config 3 for world sizes 1 and 8 (rank 0): the per-step host
cost that bounds strong scaling once the per-rank GPU work shrinks."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2301_12814_b200 as tn
import synth

case = synth.make_config(3)
qd = [torch.from_numpy(x).cuda() for x in (case.q_l, case.q_c, case.q_r)]
for world in (1, 8):
    for src in ("host", "device"):
        qs = (case.q_l, case.q_c, case.q_r) if src == "host" else qd
        ts = []
        for it in range(12):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p = tn.Plan(case.d, case.N, *qs, world, 0)
            ts.append((time.perf_counter() - t0) * 1e3)
            p.destroy()
        print(json.dumps({"world": world, "charges": src, "plan_ms_median": round(float(np.median(ts[2:])), 3),
                          "plan_ms_min": round(min(ts[2:]), 3)}), flush=True)
