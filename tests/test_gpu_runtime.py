"""The plan runtime under concurrency (DESIGN.md §4 "Runtime pieces"): several gates in flight on different streams,
plans destroyed while their exec is still running (the pool's last-use fences), a host that plans far ahead of the
GPU (backpressure), device charges produced asynchronously on another stream, and host vs device charges giving the
same plan. Every result is compared bit for bit with the same gate run alone."""
import functools

import numpy as np
import pytest
import torch

import synth
from gpu_util import gpu_theta, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


@functools.lru_cache(maxsize=None)
def _alone(cfg):
    return gpu_theta(synth.make_config(cfg))[2]


def test_gates_in_flight_on_three_streams(tn):
    # configs 1, 2, 3 as three independent gates, each on its own stream, all enqueued before any completes
    cfgs = (1, 2, 3)
    streams = [torch.cuda.Stream() for _ in cfgs]
    outs, keep = [], []
    for cfg, st in zip(cfgs, streams):
        case = synth.make_config(cfg)
        t = to_dev(case)
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            plan = tn.Plan(case.d, case.N, *[np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)])
            U = tn.build_bs_unitary(plan, case.theta, case.phi, stream=st)
            outs.append(tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, stream=st))
        keep.append((plan, t, U))
    torch.cuda.synchronize()
    for cfg, o in zip(cfgs, outs):
        for g, ref in zip(o, _alone(cfg)):
            assert np.array_equal(g.cpu().numpy(), ref)


def test_plan_destroyed_while_exec_runs(tn):
    # plan A is destroyed right after its exec is enqueued; plans B.. of the same shape created immediately after may
    # only reuse A's pool blocks once A's exec is done (last-use fence) — A's result must still be exact
    case = synth.make_config(3)
    t = to_dev(case)
    hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        pa = tn.Plan(case.d, case.N, *hq)
        Ua = tn.build_bs_unitary(pa, case.theta, case.phi, stream=s1)
        oa = tn.theta_exec(pa, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], Ua, stream=s1)
        pa.destroy()
    others = []
    with torch.cuda.stream(s2):
        for _ in range(3):
            pb = tn.Plan(case.d, case.N, *hq)
            Ub = tn.build_bs_unitary(pb, 0.3, 1.1, stream=s2)
            others.append(tn.theta_exec(pb, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], Ub, stream=s2))
            pb.destroy()
    torch.cuda.synchronize()
    for g, ref in zip(oa, _alone(3)):
        assert np.array_equal(g.cpu().numpy(), ref)


def test_host_far_ahead_of_the_gpu(tn):
    # 40 gates planned and enqueued without any synchronisation, plans dropped two gates later: the pool waits for
    # a released block instead of growing without bound, and every gate's Θ is exact
    case = synth.make_config(2)
    t = to_dev(case)
    hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
    torch.cuda.synchronize()
    tn.release_cached_memory()
    keep, outs = [], []
    U = None
    for i in range(40):
        p = tn.Plan(case.d, case.N, *hq)
        U = tn.build_bs_unitary(p, case.theta, case.phi)
        outs.append(tn.theta_exec(p, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U))
        keep.append(p)
        if len(keep) > 2:
            keep.pop(0).destroy()
    _, cached = tn.release_cached_memory()
    ws = keep[-1].workspace_bytes()
    torch.cuda.synchronize()
    assert cached <= 8 * ws, (cached, ws)   # bounded: a few plans' worth, not 40
    ref = _alone(2)
    for o in outs[::13]:
        for g, r in zip(o, ref):
            assert np.array_equal(g.cpu().numpy(), r)


def test_device_charges_from_another_stream(tn):
    # charges computed by kernels on a side stream and handed to the plan straight away (the binding orders the
    # plan's reads after the producer); the tables equal those of a host-charge plan
    case = synth.make_config(2)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        qd = [(torch.from_numpy(q.astype(np.int64)).cuda(non_blocking=True) * 3 - 2 * torch.from_numpy(
            q.astype(np.int64)).cuda(non_blocking=True)).to(torch.int32) for q in (case.q_l, case.q_c, case.q_r)]
        pd = tn.Plan(case.d, case.N, *qd)
    ph = tn.Plan(case.d, case.N, *[np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)])
    for b in range(3):
        assert np.array_equal(pd.perm(b), ph.perm(b)) and np.array_equal(pd.offsets(b), ph.offsets(b))
    assert pd.flops() == ph.flops()


def test_host_and_device_charges_same_plan(tn):
    case = synth.make_config(3, shuffled=True)
    ph = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    pd = tn.Plan(case.d, case.N, *[torch.from_numpy(q).cuda() for q in (case.q_l, case.q_c, case.q_r)])
    for b in range(3):
        assert np.array_equal(pd.perm(b), ph.perm(b)) and np.array_equal(pd.offsets(b), ph.offsets(b))
    for c in range(case.N + 1):
        assert pd.sector_shape(c) == ph.sector_shape(c)
    with pytest.raises(tn.TnError, match="DOMAIN"):      # host charges are validated on the host
        tn.Plan(case.d, case.N, np.full(5, case.N + 1, np.int32), case.q_c, case.q_r)


def test_reserve_covers_pipelined_plans(tn):
    # tn_plan_reserve(6): five more plans of the same shape kept alive take the reserved blocks (no new
    # cudaMalloc), so with all six alive the pool holds no idle block; their gates are exact
    case = synth.make_config(2)
    t = to_dev(case)
    hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
    torch.cuda.synchronize()
    tn.release_cached_memory()
    plans = [tn.Plan(case.d, case.N, *hq)]
    plans[0].reserve(6)
    for _ in range(5):
        plans.append(tn.Plan(case.d, case.N, *hq))
    outs = []
    for p in plans:
        U = tn.build_bs_unitary(p, case.theta, case.phi)
        outs.append(tn.theta_exec(p, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U))
    torch.cuda.synchronize()
    freed, held = tn.release_cached_memory()
    assert freed == 0, freed                  # every reserved block is in use by one of the six plans
    assert held >= 6 * plans[0].workspace_bytes() * 0.9
    for o in outs[::5]:
        for g, r in zip(o, _alone(2)):
            assert np.array_equal(g.cpu().numpy(), r)
    with pytest.raises(tn.TnError, match="NULL"):
        tn.check(tn.lib.tn_plan_reserve(None, 2), "tn_plan_reserve")


def test_failed_call_does_not_poison_the_next(tn):
    # a CUDA-level failure (opening a garbage IPC handle) is reported by its own status and cleared from the
    # runtime's last-error slot: the next plan / exec must not report it again as its own
    import ctypes as C
    junk = (C.c_char * 64).from_buffer_copy(bytes(range(64)))
    ptr = C.c_void_p()
    with pytest.raises(tn.TnError, match="CUDA"):
        tn.check(tn.lib.tn_ipc_open(junk, C.byref(ptr)), "tn_ipc_open")
    out = gpu_theta(synth.make_config(1))[2]
    for g, r in zip(out, _alone(1)):
        assert np.array_equal(g, r)


def test_plans_from_several_host_threads(tn):
    # four host threads plan and execute gates concurrently, each on its own stream: the plan shells, the memory
    # pool and the pinned upload ring are shared; every gate's Θ must equal the same gate run alone
    import threading
    cfgs = [1, 2, 1, 2]
    results, errors = [None] * len(cfgs), []

    def work(i, cfg):
        try:
            case = synth.make_config(cfg)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                t = to_dev(case)
                outs = []
                for _ in range(5):
                    p = tn.Plan(case.d, case.N, *[np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)])
                    U = tn.build_bs_unitary(p, case.theta, case.phi, stream=st)
                    outs.append(tn.theta_exec(p, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, stream=st))
                    p.destroy()
            st.synchronize()
            results[i] = [[o.cpu().numpy() for o in out] for out in outs]
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(i, c)) for i, c in enumerate(cfgs)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    for cfg, res in zip(cfgs, results):
        ref = _alone(cfg)
        for out in res:
            for g, r in zip(out, ref):
                assert np.array_equal(g, r)
