"""Accuracy of the INT8 Ozaki contraction vs slice count: worst per-sector relative Frobenius error of
Θ against the FP64-DMMA Θ (itself ≤1e-15 from the oracle) for configs 1–3, plain and flat λ."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth  # noqa: E402
from gpu_util import gpu_theta, rel_err  # noqa: E402

for cfg in (1, 2, 3):
    for flat in (False, True):
        case = synth.make_config(cfg, flat=flat)
        plan, U, ref = gpu_theta(case)
        for S in (4, 5, 6, 7, 8):
            _, _, got = gpu_theta(case, plan=plan, U=U, contraction=("int8", S))
            errs = [rel_err(g, r) for g, r in zip(got, ref)]
            print(json.dumps({"config": cfg, "flat": flat, "slices": S, "worst": max(errs),
                              "median": sorted(errs)[len(errs) // 2]}), flush=True)
            plan.set_contraction("dmma")
