"""Run `--reps` MPO pair-charge Θ steps (plan + U + exec) of a pair config on cuda:0 — the command profiled by
ncu for the pair path (K5F / K5P mixes). Prints the per-kernel CUDA-event times of the last step."""
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
ap.add_argument("--pair", type=int, default=5)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
c = synth.make_pair_config(a.pair)
h = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
ops = [h(x) for x in (c.gamma_k, c.lam_k, c.gamma_k1, c.lam_l, c.lam_r)]
qs = [np.ascontiguousarray(q) for q in (c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)]
for r in range(a.reps):
    p = tn.Plan2(c.d, c.N, *qs)
    U = tn.build_bs_unitary(p, c.theta, c.phi)
    out = tn.theta_exec(p, *ops, U)
    torch.cuda.synchronize()
    kt = p.kernel_times()
    p.destroy()
print(json.dumps({"pair_config": a.pair, "kernels_ms": {k: round(v, 4) for k, v in kt.items()},
                  "theta_bytes": int(sum(o.numel() for o in out) * 16)}))
