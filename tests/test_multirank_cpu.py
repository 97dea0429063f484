"""Multi-process `gloo` tests (CPU, world 2 and 4) of the N>1 host logic: every rank derives the same
flop-balanced row shards from the C library's host routine (tn_shard_rows_host, the rule tn_theta_plan uses)
and the same gather schedule (tn_gather_schedule_host, the transfer list tn_theta_exec_sharded executes over
NCCL), executes that schedule point to point, and every receiving rank (rank 0, or each sector's owner) ends
with the full Θ(c) (oracle values stand in for each rank's kernel output on this GPU-less host; the GPU
variant, tests/test_gpu_sharded.py, executes the plan's schedule on kernel output)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _execute_schedule(sched, rank, slab_of, full_shapes):
    """Run a gather transfer list (tn_gather_schedule_host / tn_plan_gather_schedule) over the default
    torch.distributed group: every rank walks the same list; a destination rank receives into (or, for its
    own slab, copies into) the full sector at the entry's row. Returns {sector: full array} for the sectors
    this rank receives."""
    import torch
    full = {}
    for t in sched:
        c, src, dst, b, rows, cols = (t[k] for k in ("sector", "src", "dst", "row_begin", "rows", "cols"))
        if dst == rank and c not in full:
            full[c] = np.zeros(full_shapes[c], dtype=np.complex128)
        if src == rank and dst == rank:
            full[c][b:b + rows] = slab_of(c)
        elif src == rank:
            blk = slab_of(c)
            assert blk.shape == (rows, cols), (c, blk.shape, rows, cols)
            dist.send(torch.from_numpy(np.ascontiguousarray(blk)), dst=dst)
        elif dst == rank:
            buf = torch.empty((rows, cols), dtype=torch.complex128)
            dist.recv(buf, src=src)
            full[c][b:b + rows] = buf.numpy()
    return full


def _worker(rank, world, port, cfg, mode, q):
    """Each rank holds its slab of every Θ(c) (its rows [r0, r1) of the sorted left positions, cut by the
    library's flop-balanced rule; oracle values stand in for its kernel output on this GPU-less host) and
    executes the library's own gather schedule (tn_gather_schedule_host — the list tn_theta_exec_sharded
    walks); every receiving rank must end with the full oracle sectors."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2301_12814_b200 as tn
        import synth
        case = synth.make_config(cfg, shuffled=True)
        N, d = case.N, case.d
        counts = [np.bincount(x, minlength=N + 1) for x in (case.q_l, case.q_c, case.q_r)]
        bounds = tn.shard_rows_host(d, N, *counts, world)
        allb = [None] * world
        dist.all_gather_object(allb, bounds.tolist())
        assert all(b == allb[0] for b in allb), "ranks disagree on the shard bounds"
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        secs, perms, offs, _ = oracle.theta_sectors(N, d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                                    case.gamma_k1, case.lam_l, case.lam_r, case.theta, case.phi)
        sched = tn.gather_schedule_host(d, N, offs[0], offs[2], bounds, mode)
        alls = [None] * world
        dist.all_gather_object(alls, sched)
        assert all(x == alls[0] for x in alls), "ranks disagree on the schedule"

        def slab_of(c):  # this rank's rows of Θ(c), from the oracle's sector row range (not from the schedule)
            (a0, a1), _ = oracle.sector_ranges(offs[0], offs[2], N, d, c)
            l0, l1 = min(max(a0, r0), r1), min(max(a1, r0), r1)
            return secs[c][l0 - a0:l1 - a0]

        full = _execute_schedule(sched, rank, slab_of, [s_.shape for s_ in secs])
        owners = tn.sector_owners_host([s_.size for s_ in secs], world)
        for c in range(N + 1):
            dst = 0 if mode == tn.TN_GATHER_ROOT else int(owners[c])
            if secs[c].shape[1] == 0 or secs[c].shape[0] == 0:
                continue
            if rank == dst:
                assert c in full and np.array_equal(full[c], secs[c]), f"sector {c} not reassembled on rank {rank}"
            else:
                assert c not in full
        q.put((rank, "ok", bounds.tolist()))
    except Exception:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


def _run(world, target, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] == "ok", f"rank {r[0]}:\n{r[1]}"
    return res


@pytest.mark.parametrize("world,cfg", [(2, 0), (2, 1), (4, 1)])
@pytest.mark.parametrize("mode", [1, 2])  # TN_GATHER_ROOT, TN_GATHER_SECTOR_OWNER
def test_gloo_gather_executes_library_schedule(world, cfg, mode):
    res = _run(world, _worker, (cfg, mode))
    b = res[0][2]
    assert b[0] == 0 and b[-1] == synth_chi(cfg) and b[1] > 0


def synth_chi(cfg):
    import synth
    return synth.CONFIGS[cfg]["chi"]


@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_gather_schedule_host_tiles_every_sector(cfg, world):
    """Host-only properties of the schedule: for each mode, every non-empty sector's rows are covered exactly
    once, in source-rank order, each source's rows are its shard's rows of the sector, and the destination is
    rank 0 (ROOT) or the LPT owner (SECTOR_OWNER); TN_GATHER_NONE has no entries."""
    import oracle
    import paper_2301_12814_b200 as tn
    import synth
    N, d, ql, qc, qr = synth.make_charges(cfg)
    perm_l, off_l = oracle.sort_bonds(ql, N)
    perm_r, off_r = oracle.sort_bonds(qr, N)
    counts = [np.bincount(x, minlength=N + 1) for x in (ql, qc, qr)]
    bounds = tn.shard_rows_host(d, N, *counts, world)
    assert tn.gather_schedule_host(d, N, off_l, off_r, bounds, tn.TN_GATHER_NONE) == []
    shapes = []
    for c in range(N + 1):
        (a0, a1), (b0, b1) = oracle.sector_ranges(off_l, off_r, N, d, c)
        shapes.append((a0, a1, b1 - b0))
    owners = tn.sector_owners_host([(a1 - a0) * cc for a0, a1, cc in shapes], world)
    for mode in (tn.TN_GATHER_ROOT, tn.TN_GATHER_SECTOR_OWNER):
        sched = tn.gather_schedule_host(d, N, off_l, off_r, bounds, mode)
        for c, (a0, a1, cc) in enumerate(shapes):
            ent = [t for t in sched if t["sector"] == c]
            if cc == 0 or a1 == a0:
                assert ent == []
                continue
            pos = 0
            for t in ent:
                assert t["row_begin"] == pos and t["rows"] > 0 and t["cols"] == cc
                src = t["src"]
                lo, hi = max(a0, bounds[src]), min(a1, bounds[src + 1])
                assert (t["row_begin"], t["rows"]) == (lo - a0, hi - lo)
                assert t["dst"] == (0 if mode == tn.TN_GATHER_ROOT else owners[c])
                pos += t["rows"]
            assert pos == a1 - a0
            assert [t["src"] for t in ent] == sorted(t["src"] for t in ent)


def test_gather_schedule_host_errors():
    import paper_2301_12814_b200 as tn
    off = np.array([0, 2, 4, 6, 8], dtype=np.int32)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.gather_schedule_host(4, 3, off, off, [0, 8], 7)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.gather_schedule_host(4, 3, off[::-1].copy(), off, [0, 8], 1)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.gather_schedule_host(4, 3, off, off, [0, 5, 3], 1)
    with pytest.raises(ValueError):
        tn.gather_schedule_host(4, 3, off[:4], off, [0, 8], 1)


def test_sector_owner_rule_is_lpt():
    import sys
    sys.path.insert(0, ROOT)
    import paper_2301_12814_b200 as tn
    sizes = [50, 10, 40, 30, 20, 0]
    # sorted 50,40,30,20,10,0 → r0, r1, r1 (40<50), r0 (50<70), r0 (tie 70=70 → lower), r1
    assert tn.sector_owners_host(sizes, 2).tolist() == [0, 0, 1, 1, 0, 1]
    assert tn.sector_owners_host(sizes, 1).tolist() == [0] * 6
