#!/usr/bin/env python
"""Benchmark of the Θ(c) hot path (BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl tn|reference]
  (N > 1: launched by torchrun, one rank per GPU; Θ rows are sharded flop-balanced across ranks)

One STEP = one gate = every row of SURVEY.md §8(a): tn_theta_plan (K1 bond sort + work decomposition)
→ tn_build_bs_unitary (K2) → tn_theta_exec (K3 staging → K4 DMMA contraction → K5 U-mix). Inputs
(Γk, Γk1 268 MB each, Θ 1.28 GB at config 3) are resident in HBM and larger than the 126 MB L2.
`value` = useful complex-FP64 GFLOP/s of the whole gate (F_contract + F_mix) over the
max-over-ranks device time. `e2e` = the same metric through the same public calls with HOST buffers
(pinned H2D of Γ/λ/charges and D2H of every Θ(c) inside the timed region). `--impl reference` times the
CPU oracle (oracle/, the literal triple charge loop of PAPER.md:72) on host cores instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Θ-build useful complex FP64 GFLOP/s & gates/s at d=32,χ=4096; % FP64 TC peak"
FP64_TC_PEAK_TFLOPS = 37.2   # measured: DMMA.8x8x4 loop, 148 SMs @ 1965 MHz (profiles/r01_fp64_peaks.jsonl)
# kernel launches per step = K1 (plan) + K2 (U) + tn_plan_exec_launches (K3, K4, one K5 launch per register
# class of the mix; INT8 engine: 4 K3O launches + K4O), counted from the plan
INT8_UMMA_PEAK_TOPS = 4347.9  # measured tcgen05 kind::i8 M=128 N=256 (profiles/r01_umma_i8_test.log)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="tn", choices=["tn", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--streams", type=int, default=1,
                    help="independent gates in flight (each on its own stream with its own U and Θ buffers); 1 = serial")
    ap.add_argument("--projection-streams", type=int, default=3,
                    help="gates in flight for the multi-GPU projection (its wall(1) is re-measured with the same count)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt-engine", action="store_true", help="skip timing the INT8 emulation engine")
    ap.add_argument("--cpu-sectors", default="0,6,12,18,24,30")
    ap.add_argument("--contraction", default="dmma", choices=["dmma", "int8", "literal"],
                    help="K4 engine: FP64 DMMA (default) or the INT8 tcgen05 Ozaki emulation")
    ap.add_argument("--slices", type=int, default=6, help="INT8 emulation slice count (6: ≤1e-11 rel error)")
    ap.add_argument("--gates", type=int, default=32, help="config 4: gates of the brick-wall layer to time")
    ap.add_argument("--layer", type=int, default=None, metavar="M",
                    help="time brick-wall layers (Θ + SVD per gate) on an M-site MPS with config-N bonds")
    ap.add_argument("--chi-max", type=int, default=None, help="layer mode: truncation χ (default: the config's χ)")
    ap.add_argument("--mpo", type=int, default=None, metavar="K",
                    help="layer mode on an MPO (vectorized density matrix, pair charges) shaped like synth.PAIR_CONFIGS[K]")
    ap.add_argument("--emulate-ranks", type=int, default=8, metavar="R",
                    help="N=1 only: run every rank's row-sharded step of a world-R job in turn on this GPU and "
                         "report per-rank device times and the projected strong-scaling speedup (0: skip)")
    ap.add_argument("--pair", type=int, default=None,
                    help="time the MPO doubled-charge path on synth.PAIR_CONFIGS[k] instead (tn_theta2_plan)")
    return ap.parse_args()


# --------------------------------------------------------------------------------------------- helpers
def sector_useful_flops(N, d, nl, nc, nr):
    """F_useful split by output sector c: contraction of P_c (group c_c = c) plus the
    mix into Θ(c). Σ_c equals F_contract + F_mix exactly (bookkeeping only)."""
    out = []
    for c in range(N + 1):
        f = 0
        if nc[c]:
            for cl in range(c, min(N, c + d - 1) + 1):
                for cr in range(max(0, c - d + 1), c + 1):
                    f += 8 * nl[cl] * nc[c] * nr[cr]
        for cl in range(c, min(N, c + d - 1) + 1):
            for cr in range(max(0, c - d + 1), c + 1):
                ncc = sum(1 for x in range(max(cr, cl - d + 1), min(cl, cr + d - 1) + 1) if nc[x])
                f += 8 * nl[cl] * nr[cr] * ncc
        out.append(f)
    return out


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every ~5 ms during the timed region
    (B200_PROFILING.md clocks line; nvidia-smi is too slow to sample a ~0.1 s region)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.period = float(os.environ.get("TN_BENCH_NVML_PERIOD_S", "0.005"))
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.rows.append((sm, mx, pw, rs))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[3] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "power_w_max": round(max(r[2] for r in self.rows), 1),
                "source": "NVML, 5 ms period, timed region"}


def ncu_traffic(cfg):
    """dram bytes per K4 launch from the committed `ncu --set full` capture, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_k4_summary.json")
    try:
        d = json.load(open(p))
        return d.get(f"config{cfg}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


_UB_CACHE = {}


def cpu_oracle_run(case, sectors):
    """Time the oracle (as it stands) on the given sectors of `case`; returns (seconds, flops)."""
    import numpy as np
    import oracle
    nq = case.N + 1
    nl, nc, nr = (np.bincount(q, minlength=nq).tolist() for q in (case.q_l, case.q_c, case.q_r))
    per = sector_useful_flops(case.N, case.d, nl, nc, nr)
    key = (case.theta, case.phi, case.d, case.N)
    if key not in _UB_CACHE:
        _UB_CACHE[key] = [oracle.bs_unitary_block(n, case.theta, case.phi, case.d)
                          for n in range(min(case.N, 2 * case.d - 2) + 1)]
    ub = _UB_CACHE[key]
    t0 = time.perf_counter()
    oracle.theta_sectors(case.N, case.d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k, case.gamma_k1,
                         case.lam_l, case.lam_r, case.theta, case.phi, u_blocks=ub, sectors=sectors)
    dt = time.perf_counter() - t0
    return dt, sum(per[c] for c in sectors)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# --------------------------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    import synth
    case = synth.make_config(args.config)
    nq = case.N + 1
    order = [(7 * i + 3) % nq for i in range(args.warmup + args.steps)]
    for i in range(args.warmup):
        cpu_oracle_run(case, [order[i]])
    tot_t, tot_f = 0.0, 0
    for i in range(args.steps):
        dt, f = cpu_oracle_run(case, [order[args.warmup + i]])
        tot_t += dt
        tot_f += f
    value = tot_f / tot_t / 1e9
    ms = tot_t / args.steps * 1e3
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(case, args.config),
            "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": host_cores(), "kind": "oracle",
                             "sample": f"one Θ(c) sector per step (c = (7i+3) mod {nq}) of config {args.config}, "
                                       "useful flops of that sector / oracle wall time; U prebuilt (mpmath)"},
            "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(case, cfg):
    return {"workload": f"BASELINE.json config {cfg}: single gate N={case.N}, d={case.d}, chi={case.chi_l} on all "
                        f"three bonds, {case.meta.get('charges')} charges, {case.meta.get('lam')} lambda, seed "
                        f"{case.meta.get('seed')}",
            "N": case.N, "d": case.d, "chi": case.chi_l, "theta": case.theta, "phi": case.phi,
            "l2": "inputs larger than L2 (Γk, Γk1 268 MB each at config 3; Θ 1.28 GB; staging 0.3 GB)"}


# --------------------------------------------------------------------------------------------- our arm
def run_tn(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2301_12814_b200 as tn
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    case = synth.make_config(args.config)
    nq = case.N + 1
    h = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    gk, gk1 = h(case.gamma_k).to(dev), h(case.gamma_k1).to(dev)
    lk, ll, lr = h(case.lam_k).to(dev), h(case.lam_l).to(dev), h(case.lam_r).to(dev)
    # bond charges stay on the host (48 KB of plan metadata): tn_theta_plan counts them there and uploads them
    # for K1 (which sorts on the device), so planning never waits for the GPU (include/tn_theta.h)
    hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
    ql, qc, qr = hq

    torch.cuda.synchronize()
    tn.Plan(case.d, case.N, ql, qc, qr, world, rank).destroy()   # warm the module / pool
    torch.cuda.synchronize()
    probe = tn.Plan(case.d, case.N, ql, qc, qr, world, rank)
    int8 = args.contraction == "int8"
    if int8:
        probe.set_contraction("int8", args.slices)
    k1_isolated_ms = probe.kernel_times()["k1_sort"]   # K1 on an idle GPU (in the timed loop it overlaps)
    launches_per_step = 2 + probe.exec_launches()
    flops = probe.flops()
    f_useful = flops["f_contract"] + flops["f_mix"]
    int8_ops = 0   # INT8 tensor ops (2 per MAC) one K4O launch executes, incl. tile padding
    if int8:
        offc = probe.offsets(1)
        for cc in range(case.N + 1):
            K = int(offc[cc + 1] - offc[cc])
            R, Cc, _ = probe.local_sector_shape(cc)
            if K and R and Cc:
                int8_ops += 2 * (-(-R // 128) * 128) * (-(-Cc // 64) * 64) * (-(-K // 32) * 32) * 4 * (
                    args.slices * (args.slices + 1) // 2)
    # `--streams` independent gates in flight (a brick-wall layer's gates are independent): gate i runs
    # plan + U + exec on stream i mod S with its own U and Θ buffers, so one gate's staging / tails overlap another's
    nslot = max(1, args.streams)
    outs = tn.alloc_theta(probe, device=dev)
    slot_outs = [outs] + [tn.alloc_theta(probe, device=dev) for _ in range(nslot - 1)]
    slot_U = [torch.empty(probe.u_size(), dtype=torch.complex128, device=dev) for _ in range(nslot)]
    U = slot_U[0]
    del probe
    stream = torch.cuda.current_stream(dev)
    slot_streams = [stream] if nslot == 1 else [torch.cuda.Stream(dev) for _ in range(nslot)]

    plan_host_ms = []
    step_i = [0]

    def step(keep):
        i = step_i[0] % nslot
        step_i[0] += 1
        st = slot_streams[i]
        with torch.cuda.stream(st):
            t_p = time.perf_counter()
            plan = tn.Plan(case.d, case.N, ql, qc, qr, world, rank)          # K1 + decomposition
            plan_host_ms.append((time.perf_counter() - t_p) * 1e3)
            if int8:
                plan.set_contraction("int8", args.slices)                      # slice layout (K3O/K4O)
            tn.build_bs_unitary(plan, case.theta, case.phi, out=slot_U[i], stream=st)          # K2
            tn.theta_exec(plan, gk, lk, gk1, ll, lr, slot_U[i], out=slot_outs[i], stream=st)  # K3 → K4 → K5
        keep.append(plan)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up; then the pool is sized for every plan the timed loop keeps alive (tn_plan_reserve), so that no
    # step pays a cudaMalloc on its enqueue path
    keep = []
    for _ in range(args.warmup):
        step(keep)
    keep[-1].reserve(3 * nslot + 3)
    torch.cuda.synchronize()
    keep.clear()

    # timed region: K steps, per-kernel times read from plans two steps behind (already complete)
    ktimes = {k: [] for k in ("k1_sort", "k2_unitary", "k3_stage", "k4_contract", "k5_mix")}

    def harvest(plan):
        for k, v in plan.kernel_times().items():
            ktimes[k].append(v)
        plan.destroy()

    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for st in slot_streams:
            st.wait_stream(stream)
        for i in range(args.steps):
            step(keep)
            if len(keep) > 1 + 2 * nslot:
                harvest(keep.pop(0))
        for st in slot_streams:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    for p in keep:
        harvest(p)
    keep.clear()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = f_useful / (ms_step * 1e-3) / 1e9

    # ---- the optional INT8 tcgen05 emulation engine on the same gates (reported beside the FP64 line)
    alt = None
    if not int8 and not args.no_alt_engine:
        try:
            a_ms = []
            for it in range(args.warmup + 5):
                ap = tn.Plan(case.d, case.N, ql, qc, qr, world, rank)
                ap.set_contraction("int8", args.slices)
                barrier()
                torch.cuda.synchronize()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                tn.build_bs_unitary(ap, case.theta, case.phi, out=U)
                tn.theta_exec(ap, gk, lk, gk1, ll, lr, U, out=outs)
                a1.record(stream)
                torch.cuda.synchronize()
                if it >= args.warmup:
                    a_ms.append(a0.elapsed_time(a1))
                kt8 = ap.kernel_times()
                ap.destroy()
            am = torch.tensor([statistics.mean(a_ms)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(am, op=dist.ReduceOp.MAX)
            am = float(am.item())
            alt = {"engine": f"INT8 tcgen05 Ozaki emulation, {args.slices} slices (≤1e-11 rel. error vs oracle)",
                   "ms_per_gate_excl_plan": round(am, 4), "useful_gflops": round(f_useful / (am * 1e-3) / 1e9, 1),
                   "pct_fp64_tc_peak": round(100.0 * f_useful / (am * 1e-3) / (FP64_TC_PEAK_TFLOPS * 1e12 * world), 2),
                   "kernels_ms": {k: round(v, 4) for k, v in kt8.items() if k != "k1_sort"},
                   "note": "U build + exec on resident inputs, plan excluded (it includes a host sync for the "
                           "slice layout); the headline value above stays on FP64 DMMA"}
        except Exception as e:
            alt = {"error": repr(e)[:300]}

    # ---- multi-GPU communication variants: exec only, then + operand broadcast,
    # + SECTOR_OWNER gather, + ROOT gather, each timed on the device as the max over ranks
    comm_variants = None
    if world > 1:
        try:
            comm = tn.Comm(rank, world)
            vplan = tn.Plan(case.d, case.N, ql, qc, qr, world, rank)
            gk_scratch = torch.empty_like(gk)
            tn.build_bs_unitary(vplan, case.theta, case.phi, out=U)
            comm_variants = {}
            for name, bc, gm in (("exec_only", tn.TN_BCAST_NONE, tn.TN_GATHER_NONE),
                                 ("bcast_slabs", tn.TN_BCAST_SLABS, tn.TN_GATHER_NONE),
                                 ("bcast_full", tn.TN_BCAST_FULL, tn.TN_GATHER_NONE),
                                 ("gather_sector_owner", tn.TN_BCAST_NONE, tn.TN_GATHER_SECTOR_OWNER),
                                 ("gather_root", tn.TN_BCAST_NONE, tn.TN_GATHER_ROOT)):
                vout = None
                for it in range(4):                       # 1 warm-up + 3 timed
                    barrier()
                    torch.cuda.synchronize()
                    v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    v0.record(stream)
                    # TN_BCAST_SLABS overwrites a rank > 0's gk with its packed slab: use a scratch copy
                    g_in = gk if bc != tn.TN_BCAST_SLABS or rank == 0 else gk_scratch
                    vout = tn.theta_exec_sharded(vplan, comm, g_in, lk, gk1, ll, lr, U, out=vout, bcast_operands=bc,
                                                 gather_mode=gm)
                    v1.record(stream)
                    torch.cuda.synchronize()
                    if it:
                        comm_variants.setdefault(name, []).append(v0.elapsed_time(v1))
                tv = torch.tensor([statistics.mean(comm_variants[name])], dtype=torch.float64, device=dev)
                dist.all_reduce(tv, op=dist.ReduceOp.MAX)
                comm_variants[name] = round(float(tv.item()), 4)
                del vout
            # the SECTOR_OWNER exchange fused into K5 (peer-memory stores over NVLink, tn_theta_exec_remote)
            fx = []
            for it in range(4):
                barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                tn.theta_exec_to_owners(vplan, gk, lk, gk1, ll, lr, U)
                if it:
                    fx.append((time.perf_counter() - t0) * 1e3)
            tv = torch.tensor([statistics.mean(fx)], dtype=torch.float64, device=dev)
            dist.all_reduce(tv, op=dist.ReduceOp.MAX)
            comm_variants["fused_sector_owner_wall"] = round(float(tv.item()), 4)
            vplan.destroy()
            comm.destroy()
        except Exception as e:  # keep the headline line even if a variant fails
            comm_variants = {"error": repr(e)[:300]}

    # ---- end to end through the public API with host buffers (pinned H2D + Θ D2H inside the region).
    # Two slots on two streams: gate g+1's H2D and compute overlap gate g's D2H (independent gates, as in
    # a layer); every step still moves its full inputs in and its full Θ out.
    pin = lambda a: h(a).pin_memory()
    host_in = dict(gk=pin(case.gamma_k), gk1=pin(case.gamma_k1), lk=pin(case.lam_k), ll=pin(case.lam_l),
                   lr=pin(case.lam_r))
    host_q = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
    NSLOT = 2
    streams = [torch.cuda.Stream(dev) for _ in range(NSLOT)]
    slots = []
    for i in range(NSLOT):
        slots.append(dict(d_in={k: torch.empty_like(v, device=dev) for k, v in host_in.items()},
                          U=torch.empty_like(U), outs=outs if i == 0 else tn.alloc_theta(tn.Plan(
                              case.d, case.N, ql, qc, qr, world, rank), device=dev),
                          host_out=[torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]))
    h2d = sum(v.numel() * v.element_size() for v in host_in.values()) + sum(q.nbytes for q in host_q)
    d2h = sum(o.numel() * o.element_size() for o in outs)

    def e2e_step(g):
        sl, st = slots[g % NSLOT], streams[g % NSLOT]
        with torch.cuda.stream(st):
            for k, v in host_in.items():
                sl["d_in"][k].copy_(v, non_blocking=True)
            plan = tn.Plan(case.d, case.N, *host_q, world, rank)          # host charges → H2D inside
            tn.build_bs_unitary(plan, case.theta, case.phi, out=sl["U"], stream=st)
            tn.theta_exec(plan, sl["d_in"]["gk"], sl["d_in"]["lk"], sl["d_in"]["gk1"], sl["d_in"]["ll"],
                          sl["d_in"]["lr"], sl["U"], out=sl["outs"], stream=st)
            for o, ho in zip(sl["outs"], sl["host_out"]):
                ho.copy_(o, non_blocking=True)
        return plan

    for g in range(NSLOT):
        p_ = e2e_step(g)
        p_.reserve(2 * NSLOT + 2)
        p_.destroy()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for st in streams:
        st.wait_stream(stream)
    live = []
    for g in range(args.e2e_steps):
        live.append(e2e_step(g))
        if len(live) > NSLOT:
            live.pop(0).destroy()
    for st in streams:
        stream.wait_stream(st)
    f1.record(stream)
    torch.cuda.synchronize()
    for p_ in live:
        p_.destroy()
    e2e_ms = f0.elapsed_time(f1)
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_step_ms = float(te.item()) / args.e2e_steps
    e2e_value = f_useful / (e2e_step_ms * 1e-3) / 1e9

    projection = None
    if world == 1 and args.emulate_ranks > 1 and not int8:
        # the projection runs every rank's step with `--projection-streams` gates in flight and divides a world-1
        # step measured the same way (like with like); the headline line above keeps `--streams`
        ps = max(1, args.projection_streams)
        pstreams = [torch.cuda.Stream(dev) for _ in range(ps)] if ps > 1 else [stream]
        pU = [torch.empty_like(U) for _ in range(ps)]
        wall1_same = emulate_ranks(tn, case, 1, args.steps, args.warmup, dev, stream, hq, (gk, lk, gk1, ll, lr), pU,
                                   0.0, pstreams)["max_ms"] if ps != nslot else ms_step
        # the speedup divides the BEST world-1 step of this run (with three gates in flight one GPU is slower
        # than with one: L2 contention), so the projection never gains from a slowed baseline
        wall1 = min(wall1_same, ms_step)
        projection = emulate_ranks(tn, case, args.emulate_ranks, args.steps, args.warmup, dev, stream, hq,
                                   (gk, lk, gk1, ll, lr), pU, wall1, pstreams)
        projection["gates_in_flight"] = ps
        projection["wall1_same_streams_ms"] = round(wall1_same, 4)
        projection["projected_speedup_same_streams"] = round(wall1_same / projection["max_ms"], 3)
        projection["wall1_def"] = (f"the best world-1 step of this run: min(headline ms_per_step with {nslot} gate(s) "
                                   f"in flight, the world-1 step with the ranks' {ps} gates in flight = "
                                   f"wall1_same_streams_ms)")

    if rank != 0:
        return
    kmean = {k: (statistics.mean(v) if v else None) for k, v in ktimes.items()}
    kmean["k1_sort"] = k1_isolated_ms
    k4_ms = kmean["k4_contract"]
    achieved = flops["f_contract_local"] / (k4_ms * 1e-3) / 1e12
    step_kernel_ms = sum(v for v in kmean.values() if v is not None)
    kernels = {k: {"ms": round(v, 4), "share_of_step": round(v / ms_step, 4)} for k, v in kmean.items()}
    kernels["k5_mix"]["hbm_gbs"] = round(2 * 16 * sum(o.numel() for o in outs) / (kmean["k5_mix"] * 1e-3) / 1e9, 1)
    kernels["k4_contract"]["useful_tflops"] = round(achieved, 3)
    kernels["k4_contract"]["executed_tflops"] = round(flops["f_exec"] / (k4_ms * 1e-3) / 1e12, 3)
    # the 3M (Gauss) product executes 3 real DMMA MACs per complex MAC: 6 real flops instead of 8
    dmma_real_tflops = flops["f_exec"] * 6 / 8 / (k4_ms * 1e-3) / 1e12
    kernels["k4_contract"]["dmma_real_tflops"] = round(dmma_real_tflops, 3)
    kernels["k1_sort"]["note"] = "isolated (plan on an idle GPU); in the timed loop K1 overlaps the previous exec"
    kernels["k1_sort"]["share_of_step"] = round(kmean["k1_sort"] / ms_step, 4)

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        secs = [int(x) for x in args.cpu_sectors.split(",") if x.strip() != "" and int(x) <= case.N]
        dt, f = cpu_oracle_run(case, secs)
        cpu = {"value": round(f / dt / 1e9, 4), "unit": "GFLOP/s", "cores": host_cores(), "kind": "oracle",
               "sample": f"sectors {secs} of config {args.config} (oracle triple charge loop, numpy/OpenBLAS "
                         f"threads = host cores), useful flops of those sectors {f / 1e9:.2f} GFLOP in {dt:.1f} s; "
                         "U prebuilt with mpmath (not timed)"}

    roofline = {"bound": "tensor", "kernel": "k4_contract", "achieved": round(achieved, 3),
                "peak": FP64_TC_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": round(achieved / FP64_TC_PEAK_TFLOPS, 4),
                "traffic": ncu_traffic(args.config),
                "peak_source": "measured FP64 DMMA.8x8x4 rate (profiles/r01_fp64_peaks.jsonl; "
                               "MEASURED_PEAKS.json has no FP64 entry)",
                "achieved_def": "F_contract of this rank (useful complex FP64 flops, 8/CMAC) / mean K4 "
                                "launch time (CUDA events on the exec stream, timed region)",
                "note": "K4 forms complex products with 3 real DMMAs (Gauss), so useful 8-flop/CMAC throughput "
                        "can exceed the 4-multiplication peak; dmma_pipe_frac is the real-DMMA utilisation",
                "dmma_pipe_frac": round(dmma_real_tflops / FP64_TC_PEAK_TFLOPS, 4)}
    if int8:
        i8 = int8_ops / (k4_ms * 1e-3) / 1e12
        roofline = {"bound": "tensor", "kernel": "k4o_contract (INT8 tcgen05, Ozaki S=%d)" % args.slices,
                    "achieved": round(i8, 1), "peak": INT8_UMMA_PEAK_TOPS, "unit": "TOPS (int8)",
                    "frac": round(i8 / INT8_UMMA_PEAK_TOPS, 4), "traffic": None,
                    "peak_source": "measured tcgen05.mma kind::i8 M=128 N=256 rate (profiles/r01_umma_i8_test.log)",
                    "achieved_def": "INT8 ops (2/MAC) of the slice products incl. 128x64x32 tile padding / mean "
                                    "K4O launch time (CUDA events, timed region)",
                    "useful_fp64_tflops": round(achieved, 3),
                    "useful_frac_of_fp64_tc_peak": round(achieved / FP64_TC_PEAK_TFLOPS, 4)}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator synth/, BASELINE.json config recipe)",
        "gates_per_s": round(1000.0 / ms_step, 3),
        "pct_fp64_tc_peak": round(100.0 * value / (FP64_TC_PEAK_TFLOPS * 1e3 * world), 2),
        "config": dict(workload_config(case, args.config), parallelism=f"rows{world}" if world > 1 else "single",
                       gates_in_flight=nslot,
                       contraction="dmma (FP64 tensor cores)" if not int8 else
                       f"int8 tcgen05 Ozaki emulation, {args.slices} slices (≤1e-11 rel. error vs oracle)",
                       f_contract=flops["f_contract"], f_mix=flops["f_mix"], f_exec_rank0=flops["f_exec"],
                       step="tn_theta_plan + tn_build_bs_unitary + tn_theta_exec (all SURVEY §8(a) rows)"),
        "roofline": roofline,
        "kernels": kernels,
        "e2e": {"value": round(e2e_value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_step_ms, 3),
                "note": "pinned H2D of Γk, Γk1, λ's and charges + D2H of every Θ(c) per gate, 2 gates in flight"},
        "comm_variants_ms": comm_variants,
        "plan_host_ms": round(statistics.median(plan_host_ms), 4) if plan_host_ms else None,
        "multi_gpu_projection": projection,
        "alt_engine": alt,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def emulate_ranks(tn, case, R, steps, warmup, dev, stream, hq, ops, slot_U, wall1_ms, slot_streams):
    """A PROJECTION of the world-R row-sharded step (compute only, operands
    pre-replicated, Θ left sharded), measured on this one GPU: every rank's own step — tn_theta_plan(R, r) with
    host charges + U + tn_theta_exec of its flop-balanced row shard — runs back to back `steps` times in turn,
    timed with CUDA events exactly like the N=1 line (same gates in flight); a rank on its own B200 would see this
    device time (same SM count and HBM), while the host-side plan time per rank is what could keep it from staying
    GPU-bound. projected_speedup = wall(1) / max_r wall(r)."""
    import torch
    gk, lk, gk1, ll, lr = ops
    nslot = len(slot_streams)
    per, host, kern, slow = [], [], [], []
    for r in range(R):
        probe = tn.Plan(case.d, case.N, *hq, R, r)
        outs = [tn.alloc_theta(probe, device=dev) for _ in range(nslot)]
        probe.destroy()
        hms = []
        cnt = [0]

        def step(keep):
            i = cnt[0] % nslot
            cnt[0] += 1
            st = slot_streams[i]
            with torch.cuda.stream(st):
                t0 = time.perf_counter()
                p = tn.Plan(case.d, case.N, *hq, R, r)
                t1 = time.perf_counter()
                hms.append((t1 - t0) * 1e3)
                tn.build_bs_unitary(p, case.theta, case.phi, out=slot_U[i], stream=st)
                t2 = time.perf_counter()
                tn.theta_exec(p, gk, lk, gk1, ll, lr, slot_U[i], out=outs[i], stream=st)
                t3 = time.perf_counter()
            keep.append(p)
            return t0, t1, t2, t3
        keep = []
        for _ in range(warmup):
            step(keep)
        keep[-1].reserve(3 * nslot + 3)
        torch.cuda.synchronize()
        for p in keep:
            p.destroy()
        keep.clear()
        hms.clear()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kt = []
        e0.record(stream)
        for st in slot_streams:
            st.wait_stream(stream)
        for k in range(steps):
            t = step(keep)
            if len(keep) > 1 + 2 * nslot:
                old = keep.pop(0)
                kt.append(old.kernel_times())
                t = t + (time.perf_counter(),)
                old.destroy()
                t = t + (time.perf_counter(),)
            if t[-1] - t[0] > 2e-3:   # diagnostics: which host call held the enqueue (backpressure waits are < 2 ms)
                slow.append([r, k] + [round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])])
        for st in slot_streams:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize()
        for p in keep:
            kt.append(p.kernel_times())
            p.destroy()
        per.append(e0.elapsed_time(e1) / steps)
        host.append(statistics.median(hms))
        kern.append({k: round(statistics.mean(x[k] for x in kt), 4) for k in ("k3_stage", "k4_contract", "k5_mix")})
        del outs
    mx, mean = max(per), statistics.mean(per)
    comm = comm_model(tn, case, hq, R, per, wall1_ms) if R > 1 else None
    return {"kind": "projection (not a multi-GPU measurement): each rank's step timed alone on this GPU",
            "comm_model": comm,
            "ranks": R, "per_rank_ms": [round(x, 4) for x in per], "max_ms": round(mx, 4),
            "imbalance_max_over_mean": round(mx / mean, 4), "wall1_ms": round(wall1_ms, 4),
            "projected_speedup": round(wall1_ms / mx, 3) if wall1_ms > 0 else None,
            "plan_host_ms_per_rank": [round(x, 4) for x in host],
            "kernels_ms_rank0": kern[0], "kernels_ms_slowest": kern[per.index(mx)],
            "excludes": "operand distribution and Θ gathers (modelled in comm_model; comm_variants_ms at N>1 "
                        "measures them)",
            "slow_host_steps": slow[:16],
            "slow_host_steps_def": "[rank, step, plan ms, U ms, exec ms, kernel_times ms, destroy ms] of steps whose "
                                   "host enqueue took > 2 ms"}


NVLINK_GBS = 900.0   # NVLink 5 per GPU per direction, nominal (B200_PROFILING.md); NCCL reaches less


def comm_model(tn, case, hq, R, per_ms, wall1_ms):
    """A MODEL (bytes from the library's own schedules, time at the nominal NVLink rate) of the exchange steps the
    compute projection leaves out: the Γk row-slab scatter from rank 0 (TN_BCAST_SLABS) and the Θ gather to the
    sector owners (TN_GATHER_SECTOR_OWNER, tn_plan_gather_schedule). Per rank, t = max(bytes sent, bytes
    received) / NVLINK_GBS; "serial" adds it to the rank's compute, "overlapped" takes the max of the two (gates
    in flight: gate g's exchange under gate g+1's kernels, which touch other buffers)."""
    import numpy as np
    N = case.N
    cnt = [np.bincount(np.asarray(q), minlength=N + 1).astype(np.int64) for q in hq]
    off = [np.concatenate([[0], np.cumsum(c)]).astype(np.int32) for c in cnt]
    bounds = tn.shard_rows_host(case.d, N, cnt[0], cnt[1], cnt[2], R)        # the plan's own row shards
    sched = tn.gather_schedule_host(case.d, N, off[0], off[2], bounds, tn.TN_GATHER_SECTOR_OWNER)
    sched_root = tn.gather_schedule_host(case.d, N, off[0], off[2], bounds, tn.TN_GATHER_ROOT)
    chi_c = int(len(hq[1]))
    rows = [(int(bounds[r]), int(bounds[r + 1])) for r in range(R)]
    sent, recv = [0] * R, [0] * R
    for r in range(1, R):                       # Γk slabs: rank 0 → r
        b = (rows[r][1] - rows[r][0]) * chi_c * 16
        sent[0] += b
        recv[r] += b
    gsent, grecv = [0] * R, [0] * R
    for t in sched:                             # Θ slabs: src → owner
        if t["src"] == t["dst"]:
            continue
        b = t["rows"] * t["cols"] * 16
        gsent[t["src"]] += b
        grecv[t["dst"]] += b
    rsent, rrecv = [0] * R, [0] * R
    for t in sched_root:                        # Θ slabs: every rank → rank 0
        if t["src"] == t["dst"]:
            continue
        b = t["rows"] * t["cols"] * 16
        rsent[t["src"]] += b
        rrecv[t["dst"]] += b
    ms = lambda b: b / (NVLINK_GBS * 1e9) * 1e3
    t_slab = [ms(max(a, b)) for a, b in zip(sent, recv)]
    t_gath = [ms(max(a, b)) for a, b in zip(gsent, grecv)]
    t_root = [ms(max(a, b)) for a, b in zip(rsent, rrecv)]
    # full Γk broadcast (TN_BCAST_FULL): every rank receives all of Γk (a pipelined broadcast costs ≈ one copy)
    t_full = [ms(len(hq[0]) * chi_c * 16) if R > 1 else 0.0] * R
    out = {"kind": "model: library schedules' bytes at the nominal NVLink 5 rate (not measured)",
           "nvlink_gbs": NVLINK_GBS,
           "slab_scatter_mb_rank0_sent": round(sent[0] / 1e6, 1),
           "gather_owner_mb_max_sent": round(max(gsent) / 1e6, 1),
           "gather_owner_mb_max_recv": round(max(grecv) / 1e6, 1),
           "gather_root_mb_recv": round(rrecv[0] / 1e6, 1),
           "t_slab_ms": [round(x, 4) for x in t_slab], "t_gather_ms": [round(x, 4) for x in t_gath],
           "t_root_gather_ms": round(max(t_root), 4), "t_full_bcast_ms": round(t_full[0], 4)}
    if wall1_ms > 0:
        # SURVEY.md §8(e) reporting items 2–4: + operand distribution, + sector-owner gather, + root gather
        for name, extra in (("slabs", t_slab), ("full_bcast", t_full),
                            ("slabs_and_owner_gather", [a + b for a, b in zip(t_slab, t_gath)]),
                            ("slabs_and_root_gather", [a + b for a, b in zip(t_slab, t_root)])):
            serial = max(c + e for c, e in zip(per_ms, extra))
            over = max(max(c, e) for c, e in zip(per_ms, extra))
            out[f"projected_speedup_{name}_serial"] = round(wall1_ms / serial, 3)
            out[f"projected_speedup_{name}_overlapped"] = round(wall1_ms / over, 3)
    return out


# --------------------------------------------------------------------------------------------- brick-wall layer
def run_layer(args, rank, world, local_rank):
    """Two brick-wall layers (even, then odd site pairs) of real TEBD gates on an M-site MPS whose inner bonds
    have the shape of BASELINE.json config `--config` (N, d, χ, Gaussian charges, 0.995^i λ): each gate is
    tn_theta_plan + U + tn_theta_exec + tn_svd_truncate, the next gate consuming the previous one's output.
    Γ is drawn on the device (same distribution, δ-masked). Reports gates/s (host wall clock: the SVD step
    synchronises once per gate to learn the kept bond dimension). Under torchrun every rank builds the same
    replica and the gates of each layer are dealt to the ranks (mps.MPS.apply_layer(group=…)),
    results broadcast over NCCL; the time is the max over ranks."""
    import numpy as np
    import torch

    import synth
    from paper_2301_12814_b200.mps import MPO, MPS

    import torch.distributed as dist
    mpo = args.mpo is not None
    group = dist.group.WORLD if world > 1 else None
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.PAIR_CONFIGS[args.mpo] if mpo else synth.CONFIGS[args.config]
    N, d, chi, M = cfg["N"], cfg["d"], cfg["chi"], args.layer
    chi_max = args.chi_max or chi
    rng = np.random.default_rng(cfg["seed"] + 77)
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg["seed"] + 77)

    def bond_charges(k):   # Gaussian charges in bond k's reachable window (photons to the right)
        lo, hi = max(0, N - k * (d - 1)), min(N, (M - k) * (d - 1))
        return np.clip(np.rint(rng.normal(N / 2, N / 4, chi)), lo, hi).astype(np.int32)

    def ends():
        return np.array([N], np.int32), np.array([0], np.int32)
    if mpo:   # two independent species per bond, lexicographic order (synth's pair recipe)
        q1, q2 = [ends()[0]], [ends()[0]]
        for k in range(1, M):
            a, b = bond_charges(k), bond_charges(k)
            o = np.lexsort((b, a))
            q1.append(a[o])
            q2.append(b[o])
        q1.append(ends()[1])
        q2.append(ends()[1])
        qs = [[torch.from_numpy(x).to(dev) for x in q1], [torch.from_numpy(x).to(dev) for x in q2]]
    else:
        q = [ends()[0]] + [np.sort(bond_charges(k)) for k in range(1, M)] + [ends()[1]]
        qs = [[torch.from_numpy(x).to(dev) for x in q]]
    gam = []
    for k in range(M):
        m = None
        for qq in qs:
            a, b = qq[k].long(), qq[k + 1].long()
            mk = ((a[:, None] - b[None, :]) >= 0) & ((a[:, None] - b[None, :]) <= d - 1)
            m = mk if m is None else m & mk
        x = torch.randn(tuple(m.shape), generator=gen, device=dev, dtype=torch.float64)
        y = torch.randn(tuple(m.shape), generator=gen, device=dev, dtype=torch.float64)
        gam.append(torch.complex(x, y) / math.sqrt(2) * m)
    lam = [torch.ones(1, dtype=torch.float64, device=dev)]
    for k in range(1, M):
        v = torch.from_numpy(0.995 ** np.arange(chi)).to(dev)
        lam.append(v / torch.linalg.vector_norm(v))
    lam.append(torch.ones(1, dtype=torch.float64, device=dev))

    def make_state(clone=False):
        cp = (lambda xs: [x.clone() for x in xs]) if clone else (lambda xs: xs)
        if mpo:
            return MPO(N, d, cp(qs[0]), cp(qs[1]), cp(gam), cp(lam), device=dev)
        return MPS(N, d, cp(qs[0]), cp(gam), cp(lam), device=dev)
    mps = make_state()
    th = rng.uniform(0, math.pi / 2, M)
    ph = rng.uniform(0, 2 * math.pi, M)
    # warm-up: `--warmup` full-size gates on a throw-away copy (library handles, SVD scratch, memory pool)
    kw = M // 2 - 1
    for _ in range(args.warmup):
        w = make_state(clone=True)
        w.apply_gate(kw, th[0], ph[0], chi_max)
        del w
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    t0 = time.perf_counter()
    gate_ms = []
    if group is None:   # one GPU: the same gates as apply_layer, timed one by one
        disc = []
        for parity in (0, 1):
            for g, k in enumerate(range(parity, M - 1, 2)):
                tg = time.perf_counter()
                disc.append(mps.apply_gate(k, th[g], ph[g], chi_max))
                torch.cuda.synchronize()
                gate_ms.append(round((time.perf_counter() - tg) * 1e3, 1))
    else:
        disc = mps.apply_layer(0, th, ph, chi_max, group=group) + mps.apply_layer(1, th, ph, chi_max, group=group)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if group is not None:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        if rank != 0:
            return
    ngates = len(disc)
    line = {"metric": ("MPO " if mpo else "") + "brick-wall TEBD gates/s (Θ + per-sector SVD + truncation per gate)",
            "value": round(ngates / dt, 4), "unit": "gates/s", "n_gpus": world if group is not None else 1, "steps": ngates,
            "warmup": args.warmup,
            "ms_per_step": round(dt / ngates * 1e3, 2), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-drawn Γ, config-shaped bonds)",
            "config": {"workload": (f"{M}-site MPO (vectorized density matrix, pair charges, U⊗U*), two brick-wall layers, "
                                    f"inner bonds shaped like synth.PAIR_CONFIGS[{args.mpo}]" if mpo else
                                    f"{M}-site MPS, two brick-wall layers, inner bonds of BASELINE.json config {args.config}")
                                   + f" (N={N}, d={d}, chi={chi}), chi_max={chi_max}",
                       "timing": "host wall clock around whole layers (tn_svd_truncate synchronises per gate), max over ranks",
                       "parallelism": "single GPU" if group is None else
                       f"layer-parallel over {world} GPU(s): gates dealt by LPT, results broadcast (NCCL)"},
            "bond_dims_after": [int(x.numel()) for x in mps.lam], "discarded": [float(x) for x in disc],
            "gate_ms": gate_ms}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------- MPO pair path
def run_pair(args, rank, world, local_rank):
    """One step = tn_theta2_plan (K1 on pair keys + tables) + tn_build_bs_unitary (K2) + tn_theta_exec
    (K3 → K4 → two-pass K5P) on synth.PAIR_CONFIGS[k] (PAPER.md:101/:107 MPO workload; single GPU)."""
    import numpy as np
    import torch

    import paper_2301_12814_b200 as tn
    import synth

    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c = synth.make_pair_config(args.pair)
    h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    gk, gk1, lk, ll, lr = h(c.gamma_k), h(c.gamma_k1), h(c.lam_k), h(c.lam_l), h(c.lam_r)
    # pair charges stay on the host (plan metadata): the plan counts them there, no per-gate host sync
    qs = [np.ascontiguousarray(q) for q in (c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)]
    int8 = args.contraction == "int8"

    def mk():
        p = tn.Plan2(c.d, c.N, *qs, world, rank)   # row-sharded over the ranks (slabs stay local)
        if int8:
            p.set_contraction("int8", args.slices)
        return p

    probe = mk()
    launches_per_step = 2 + probe.exec_launches()
    flops = probe.flops()
    f_useful = flops["f_contract"] + flops["f_mix"]
    outs = tn.alloc_theta(probe, device=dev)
    U = torch.empty(probe.u_size(), dtype=torch.complex128, device=dev)
    probe.destroy()
    stream = torch.cuda.current_stream(dev)
    keep, kt = [], []

    def step():
        p = mk()
        tn.build_bs_unitary(p, c.theta, c.phi, out=U)
        tn.theta_exec(p, gk, lk, gk1, ll, lr, U, out=outs)
        keep.append(p)
        if len(keep) > 2:
            old = keep.pop(0)
            kt.append(old.kernel_times())
            old.destroy()

    for _ in range(args.warmup):
        step()
    keep[-1].reserve(5)
    torch.cuda.synchronize()
    kt.clear()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for p in keep:
        kt.append(p.kernel_times())
        p.destroy()
    tms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
    ms = float(tms.item()) / args.steps
    if rank != 0:
        return
    km = {k: statistics.mean(x[k] for x in kt[-args.steps:]) for k in kt[0]}
    k4 = km["k4_contract"]
    achieved = flops["f_contract_local"] / (k4 * 1e-3) / 1e12
    line = {"metric": "Θ(c1,c2) MPO build useful complex FP64 GFLOP/s", "value": round(f_useful / (ms * 1e-3) / 1e9, 3),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (synth.PAIR_CONFIGS, seeded)",
            "gates_per_s": round(1000.0 / ms, 3),
            "config": {"workload": f"MPO pair config {args.pair}: N={c.N}, d={c.d}, chi={c.chi_l}, "
                                   f"{c.meta['charges']} charge pairs", "f_contract": flops["f_contract"],
                       "f_mix": flops["f_mix"], "contraction": args.contraction,
                       "parallelism": f"rows{world}" if world > 1 else "single",
                       "step": "tn_theta2_plan + tn_build_bs_unitary + tn_theta_exec"},
            "roofline": {"bound": "tensor", "kernel": "k4_contract", "achieved": round(achieved, 3),
                         "peak": FP64_TC_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": round(achieved / FP64_TC_PEAK_TFLOPS, 4),
                         "achieved_def": "F_contract (useful, 8/CMAC) / mean K4 launch time"},
            "kernels_ms": {k: round(v, 4) for k, v in km.items()},
            "mix_hbm_gbs": round(2 * 2 * 16 * sum(o.numel() for o in outs) / (km["k5_mix"] * 1e-3) / 1e9, 1),
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------- config 4 sweep
def run_sweep(args, rank, world, local_rank):
    """BASELINE.json config 4: a brick-wall layer of `--gates` beam-splitter gates (N=47, d=48, χ=8192),
    each with its own bond charges (synth.make_charges(4, g), identical to the parity inputs) and its own
    Γ. Γ is drawn ON THE DEVICE (torch generator seeded per gate; same complex-normal distribution and
    δ-allowed mask as synth/, different values) because 32 × 2 × 8192² host draws take minutes; timing
    does not depend on the values, parity on config 4 is checked separately with synth/'s inputs.
    Gate-parallel across ranks (the paper's first-level parallelism): rank r runs gates
    r, r+N, …; no collective. One step = one gate: plan (K1) + U (K2) + exec (K3–K5), Θ buffers reused."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2301_12814_b200 as tn
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.CONFIGS[4]
    N, d, chi = cfg["N"], cfg["d"], cfg["chi"]
    mine = list(range(rank, args.gates, world))
    lam = torch.from_numpy(0.995 ** np.arange(chi)).to(dev)
    lam /= torch.linalg.vector_norm(lam)
    gates = []
    for g in mine:
        _, _, ql, qc, qr = synth.make_charges(4, g)
        gen = torch.Generator(device=dev)
        gen.manual_seed(4_000_000 + g)
        qd = [torch.from_numpy(q).to(dev) for q in (ql, qc, qr)]   # device copies draw the δ masks below

        def gamma(a, b):
            m = ((a[:, None] - b[None, :]) >= 0) & ((a[:, None] - b[None, :]) <= d - 1)
            x = torch.randn((chi, chi), generator=gen, device=dev, dtype=torch.float64)
            y = torch.randn((chi, chi), generator=gen, device=dev, dtype=torch.float64)
            return (torch.complex(x, y) / math.sqrt(2)) * m

        rng = np.random.default_rng([4, g, 7])
        gates.append(dict(q=[np.ascontiguousarray(q) for q in (ql, qc, qr)], gk=gamma(qd[0], qd[1]), gk1=gamma(qd[1], qd[2]),
                          theta=float(rng.uniform(0, math.pi / 2)), phi=float(rng.uniform(0, 2 * math.pi))))
    # Θ buffers: per sector the largest slab over this rank's gates, reused by every gate
    plans = [tn.Plan(d, N, *gt["q"]) for gt in gates]
    for pl in plans:
        pl.set_contraction(args.contraction, args.slices)
    cap = [max(pl.sector_shape(c)[0] * pl.sector_shape(c)[1] for pl in plans) for c in range(N + 1)]
    flops = [pl.flops() for pl in plans]
    for pl in plans:
        pl.destroy()
    pool = [torch.empty(max(1, n), dtype=torch.complex128, device=dev) for n in cap]
    U = torch.empty(38_024, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(gt, keep):
        plan = tn.Plan(d, N, *gt["q"])
        plan.set_contraction(args.contraction, args.slices)
        outs = [pool[c][:plan.sector_shape(c)[0] * plan.sector_shape(c)[1]].view(*plan.sector_shape(c))
                for c in range(N + 1)]
        tn.build_bs_unitary(plan, gt["theta"], gt["phi"], out=U)
        tn.theta_exec(plan, gt["gk"], lam, gt["gk1"], lam, lam, U, out=outs)
        launches.append(2 + plan.exec_launches())
        keep.append(plan)

    keep, launches = [], []
    for i in range(args.warmup):
        step(gates[i % len(gates)], keep)
    torch.cuda.synchronize()
    for p_ in keep:
        p_.destroy()
    keep.clear()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ktimes = []
    launches.clear()
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for gt in gates:
            step(gt, keep)
            if len(keep) > 2:
                old = keep.pop(0)
                ktimes.append(old.kernel_times())
                old.destroy()
        e1.record(stream)
        torch.cuda.synchronize()
    for p_ in keep:
        ktimes.append(p_.kernel_times())
        p_.destroy()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    f_all = sum(f["f_contract"] + f["f_mix"] for f in flops)
    if world > 1:
        ft = torch.tensor([float(f_all)], dtype=torch.float64, device=dev)
        dist.all_reduce(ft)
        f_all = ft.item()
    if rank != 0:
        return
    exec_ms = sum(sum(v for k, v in kt.items() if k != "k1_sort") for kt in ktimes)
    line = {"metric": "Θ-build gates/s (brick-wall layer, config 4) & useful complex FP64 GFLOP/s", "value":
            round(args.gates / (ms_max * 1e-3), 3), "unit": "gates/s", "n_gpus": world, "steps": args.gates,
            "warmup": args.warmup, "ms_per_step": round(ms_max / len(mine), 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: synth/ charges per gate, Γ drawn on device (same distribution and δ mask)",
            "useful_gflops": round(f_all / (ms_max * 1e-3) / 1e9, 1),
            "pct_fp64_tc_peak": round(100 * f_all / (ms_max * 1e-3) / (FP64_TC_PEAK_TFLOPS * 1e12 * world), 2),
            "exec_only_gates_per_s": round(len(mine) / (exec_ms * 1e-3), 3),
            "config": {"workload": f"BASELINE.json config 4: {args.gates} gates of a brick-wall layer, N={N}, d={d}, "
                                   f"chi={chi}, per-gate Gaussian charges", "parallelism": f"gates{world}",
                       "contraction": args.contraction if args.contraction == "dmma" else f"int8x{args.slices}",
                       "step": "per gate: tn_theta_plan + tn_build_bs_unitary + tn_theta_exec",
                       "l2": "inputs larger than L2 (Γ 1.07 GB each per gate; Θ up to 7.5 GB)"},
            "kernels_mean_ms": {k: round(statistics.mean(kt[k] for kt in ktimes), 4) for k in ktimes[0]},
            "gpu_launches": sum(launches),
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.layer is not None:
            run_layer(args, rank, world, local_rank)
        elif args.pair is not None:
            run_pair(args, rank, world, local_rank)
        elif args.config == 4:
            run_sweep(args, rank, world, local_rank)
        else:
            run_tn(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
