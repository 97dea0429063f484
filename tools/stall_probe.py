"""Hunts the occasional multi-ms stall in bench.py's multi_gpu_projection: the world-8 rank loop of config 3 with
3 gates in flight (same slot streams, keep depth and plan turnover as bench.emulate_ranks), repeated TRIALS
times; for every rank trial it prints the device ms/step and, for any step whose host enqueue took > 1 ms, which
call took it; Python GC pauses are logged through gc.callbacks. One GPU."""
import gc
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

R, TRIALS, STEPS, NSLOT = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 4, 40, 3
GC_OFF = len(sys.argv) > 2 and sys.argv[2] == "gcoff"
gcl = []


def _gc_cb(phase, info, t=[0.0]):
    if phase == "start":
        t[0] = time.perf_counter()
    else:
        gcl.append((info["generation"], (time.perf_counter() - t[0]) * 1e3))


gc.callbacks.append(_gc_cb)
case = synth.make_config(3)
h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
gk, gk1, lk, ll, lr = (h(x) for x in (case.gamma_k, case.gamma_k1, case.lam_k, case.lam_l, case.lam_r))
hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
stream = torch.cuda.current_stream()
slots = [torch.cuda.Stream() for _ in range(NSLOT)]
Us = [torch.empty(20000, dtype=torch.complex128, device="cuda") for _ in range(NSLOT)]
for trial in range(TRIALS):
    for r in range(R):
        probe = tn.Plan(case.d, case.N, *hq, R, r)
        outs = [tn.alloc_theta(probe) for _ in range(NSLOT)]
        probe.destroy()
        keep, slow = [], []
        cnt = [0]

        def step():
            i = cnt[0] % NSLOT
            cnt[0] += 1
            st = slots[i]
            t = [time.perf_counter()]
            with torch.cuda.stream(st):
                p = tn.Plan(case.d, case.N, *hq, R, r)
                t.append(time.perf_counter())
                tn.build_bs_unitary(p, case.theta, case.phi, out=Us[i], stream=st)
                t.append(time.perf_counter())
                tn.theta_exec(p, gk, lk, gk1, ll, lr, Us[i], out=outs[i], stream=st)
                t.append(time.perf_counter())
            keep.append(p)
            return t

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        for p in keep:
            p.destroy()
        keep.clear()
        gcl.clear()
        if GC_OFF:
            gc.disable()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in slots:
            st.wait_stream(stream)
        for k in range(STEPS):
            t = step()
            if len(keep) > 1 + 2 * NSLOT:
                old = keep.pop(0)
                old.kernel_times()
                td = time.perf_counter()
                old.destroy()
                t.append(time.perf_counter())
                t.insert(4, td)
            if t[-1] - t[0] > 1e-3:
                names = ["plan", "U", "exec", "kernel_times", "destroy"]
                slow.append((k, {n: round((b - a) * 1e3, 3) for n, a, b in zip(names, t, t[1:])}))
        for st in slots:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize()
        gc.enable()
        for p in keep:
            p.destroy()
        print(json.dumps({"trial": trial, "rank": r, "ms_per_step": round(e0.elapsed_time(e1) / STEPS, 4),
                          "slow_steps": slow, "gc": [(g, round(ms, 2)) for g, ms in gcl if ms > 0.5]}), flush=True)
        del outs
