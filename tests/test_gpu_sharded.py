"""Row a6: the row-sharded exec and its exchange steps, through the C ABI.

* tn_theta_exec_sharded with a real NCCL communicator (one rank: this pool has one GPU per box, and NCCL refuses
  two ranks on one device) for every operand-distribution mode (none, Γk row slabs, full broadcast) and every
  gather mode (none, root, sector owner), against the oracle at ≤ 1e-10 per sector and bit-identical to
  tn_theta_exec;
* the Γk row-slab path on every rank of world 2/3/8 (tn_pack_row_slab + tn_theta_exec_slab — what a rank > 0
  runs after receiving its slab), bit-identical to the full-Γk exec, single-charge and MPO pair plans, DMMA and
  INT8 engines;
* the gather schedule (tn_plan_gather_schedule): identical on every rank and equal to the host-only
  tn_gather_schedule_host, and executed over gloo by two processes on KERNEL OUTPUT — every receiving rank ends
  with the full oracle sectors. The two processes only exchange host copies after their streams drained, so no
  kernel waits on another rank's kernel.
"""
import functools
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from gpu_util import assert_sectors_close, gpu_theta, oracle_theta, to_dev

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-10


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


@pytest.fixture(scope="module")
def comm1(tn):
    c = tn.Comm(0, 1)
    yield c
    c.destroy()


@functools.lru_cache(maxsize=None)
def _case(cfg):
    return synth.make_config(cfg)


@functools.lru_cache(maxsize=None)
def _ref(cfg):
    return oracle_theta(_case(cfg))[0]


@functools.lru_cache(maxsize=None)
def _plain(cfg):
    return gpu_theta(_case(cfg))[2]


# ------------------------------------------------------------------ NCCL communicator, every mode
@pytest.mark.parametrize("cfg", [0, 1, 2])
@pytest.mark.parametrize("bcast", [0, 1, 2])   # TN_BCAST_NONE / _SLABS / _FULL
@pytest.mark.parametrize("gather", [0, 1, 2])  # TN_GATHER_NONE / _ROOT / _SECTOR_OWNER
def test_exec_sharded_nccl_one_rank(tn, comm1, cfg, bcast, gather):
    case = _case(cfg)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, 1, 0)
    U = tn.build_bs_unitary(plan, case.theta, case.phi)
    t = to_dev(case)
    out = tn.theta_exec_sharded(plan, comm1, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U,
                                bcast_operands=bcast, gather_mode=gather)
    torch.cuda.synchronize()
    comm1.async_error()
    got = [o.cpu().numpy() for o in out]
    assert_sectors_close(got, _ref(cfg), TOL, f"sharded cfg{cfg} bcast{bcast} gather{gather}")
    for g, p in zip(got, _plain(cfg)):
        assert np.array_equal(g, p)
    # the operands a broadcast touched are unchanged on the root
    assert np.array_equal(t["gk"].cpu().numpy(), case.gamma_k)
    assert np.array_equal(t["gk1"].cpu().numpy(), case.gamma_k1)


def test_exec_sharded_errors(tn, comm1):
    case = _case(1)
    t = to_dev(case)
    p2 = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, 2, 0)
    U = tn.build_bs_unitary(p2, case.theta, case.phi)
    with pytest.raises(tn.TnError, match="CONSISTENCY"):   # plan world 2, communicator world 1
        tn.theta_exec_sharded(p2, comm1, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)
    p1 = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.theta_exec_sharded(p1, comm1, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, gather_mode=5)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.theta_exec_sharded(p1, comm1, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, bcast_operands=7)
    p1.set_contraction("literal", 0)
    with pytest.raises(tn.TnError, match="UNSUPPORTED"):
        tn.theta_exec_sharded(p1, comm1, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U, bcast_operands=1)


# ------------------------------------------------------------------ Γk row slabs on every rank
@pytest.mark.parametrize("cfg,world", [(1, 2), (2, 3), (2, 8), (3, 8)])
@pytest.mark.parametrize("engine", [None, ("int8", 6)])
def test_exec_slab_every_rank(tn, cfg, world, engine):
    case = _case(cfg)
    t = to_dev(case)
    _, _, full = gpu_theta(case, contraction=engine)
    slabs = [[] for _ in range(case.N + 1)]
    for r in range(world):
        pr = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, r)
        if engine:
            pr.set_contraction(*engine)
        U = tn.build_bs_unitary(pr, case.theta, case.phi)
        slab = tn.pack_row_slab(pr, t["gk"], r)
        r0, r1 = pr.shard_rows(r)
        perm_l = pr.perm(0)
        assert np.array_equal(slab.cpu().numpy(), case.gamma_k[perm_l[r0:r1]])
        out = tn.theta_exec_slab(pr, slab, t["lk"], t["gk1"], t["ll"], t["lr"], U)
        ref_loc = tn.theta_exec(pr, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)
        torch.cuda.synchronize()
        for c in range(case.N + 1):
            assert torch.equal(out[c], ref_loc[c]), (r, c)
            slabs[c].append((pr.local_sector_shape(c)[2], out[c].cpu().numpy()))
    for c in range(case.N + 1):
        stacked = np.concatenate([p for _, p in sorted(slabs[c], key=lambda x: x[0])], axis=0)
        assert np.array_equal(stacked, full[c])


@pytest.mark.parametrize("pcfg,world", [(1, 2), (2, 3)])
def test_exec_slab_pair_plans(tn, pcfg, world):
    c = synth.make_pair_config(pcfg)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    gk, lk, gk1, ll, lr = (dv(x) for x in (c.gamma_k, c.lam_k, c.gamma_k1, c.lam_l, c.lam_r))
    for r in range(world):
        pr = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, world, r)
        U = tn.build_bs_unitary(pr, c.theta, c.phi)
        slab = tn.pack_row_slab(pr, gk, r)
        out = tn.theta_exec_slab(pr, slab, lk, gk1, ll, lr, U)
        ref = tn.theta_exec(pr, gk, lk, gk1, ll, lr, U)
        torch.cuda.synchronize()
        for s in range(pr.nsec):
            assert torch.equal(out[s], ref[s]), (r, s)


# ------------------------------------------------------------------ the gather schedule
@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_plan_schedule_matches_host_schedule(tn, cfg, world):
    case = _case(cfg)
    counts = [np.bincount(q, minlength=case.N + 1) for q in (case.q_l, case.q_c, case.q_r)]
    bounds = tn.shard_rows_host(case.d, case.N, *counts, world)
    for mode in (tn.TN_GATHER_NONE, tn.TN_GATHER_ROOT, tn.TN_GATHER_SECTOR_OWNER):
        scheds = []
        for r in (0, world - 1):
            pr = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, r)
            scheds.append(pr.gather_schedule(mode))
            for tr in scheds[-1]:
                assert (tr["row_begin"], tr["rows"]) == pr.slab_rows(tr["sector"], tr["src"])
        assert scheds[0] == scheds[1]
        host = tn.gather_schedule_host(case.d, case.N, pr.offsets(0), pr.offsets(2), bounds, mode)
        assert scheds[0] == host


def test_plan_schedule_pair_covers_rows(tn):
    c = synth.make_pair_config(2)
    world = 3
    pr = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, world, 1)
    for mode in (tn.TN_GATHER_ROOT, tn.TN_GATHER_SECTOR_OWNER):
        sched = pr.gather_schedule(mode)
        for s in range(pr.nsec):
            R, Cc = pr.sector_shape(s)
            ent = [t for t in sched if t["sector"] == s]
            if R * Cc == 0:
                assert not ent
                continue
            assert sum(t["rows"] for t in ent) == R
            pos = 0
            for t in ent:
                assert t["row_begin"] == pos and t["cols"] == Cc
                assert t["dst"] == (0 if mode == tn.TN_GATHER_ROOT else pr.sector_owner(s))
                pos += t["rows"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_worker(rank, world, port, cfg, mode, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2301_12814_b200 as tn
        import synth as sy
        from gpu_util import oracle_theta as oth, to_dev as tdev, rel_err
        torch.cuda.set_device(0)
        case = sy.make_config(cfg)
        plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, rank)
        U = tn.build_bs_unitary(plan, case.theta, case.phi)
        t = tdev(case)
        loc = tn.theta_exec(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)   # this rank's kernel output
        torch.cuda.synchronize()
        loc = [x.cpu() for x in loc]
        sched = plan.gather_schedule(mode)
        full = {}
        for tr in sched:
            c, src, dst, b, rows = tr["sector"], tr["src"], tr["dst"], tr["row_begin"], tr["rows"]
            if dst == rank and c not in full:
                full[c] = torch.zeros(plan.sector_shape(c), dtype=torch.complex128)
            if src == rank and dst == rank:
                full[c][b:b + rows] = loc[c]
            elif src == rank:
                dist.send(loc[c].contiguous(), dst=dst)
            elif dst == rank:
                buf = torch.empty((rows, tr["cols"]), dtype=torch.complex128)
                dist.recv(buf, src=src)
                full[c][b:b + rows] = buf
        ref = oth(case)[0]
        worst = 0.0
        for c, v in full.items():
            e = rel_err(v.numpy(), ref[c])
            worst = max(worst, e)
            assert e <= 1e-10, (c, e)
        n = [None] * world
        dist.all_gather_object(n, sorted(full))
        got = sorted(x for lst in n for x in lst)
        want = sorted(c for c in range(case.N + 1) if ref[c].size > 0)
        assert got == want, (got, want)
        q.put((rank, "ok", worst))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [1, 2])
@pytest.mark.parametrize("mode", [1, 2])
def test_gather_schedule_on_kernel_output_two_processes(tn, cfg, mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, cfg, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[1] == "ok", f"rank {r[0]}:\n{r[1]}"


def test_sharded_equals_unsharded_config3(tn):
    # T12 at config 3: every rank's slab of world 8, run in turn on this GPU, stacks into the
    # unsharded Θ bit for bit
    case = _case(3)
    _, _, full = gpu_theta(case)
    world = 8
    slabs = [[] for _ in range(case.N + 1)]
    for r in range(world):
        _, _, loc = gpu_theta(case, world, r)
        pr = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, r)
        for c in range(case.N + 1):
            slabs[c].append((pr.local_sector_shape(c)[2], loc[c]))
    for c in range(case.N + 1):
        stacked = np.concatenate([p for _, p in sorted(slabs[c], key=lambda x: x[0])], axis=0)
        assert np.array_equal(stacked, full[c])
