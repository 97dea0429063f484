"""B200-native charge-sectored two-site Θ(c) builder (arXiv 2301.12814, Supplementary Eq. S5).

Python face of the C ABI in include/tn_theta.h, with the same names. PyTorch is used for device memory
and streams only; every computing step runs in libtn_theta.so's sm_100a kernels:
  K1 bond sort (plan) → K2 U builder → K3 staging → K4 grouped complex DMMA contraction → K5 U-mix.

    plan = Plan(d, N, q_l, q_c, q_r)                 # tn_theta_plan
    U = build_bs_unitary(plan, theta, phi)           # tn_build_bs_unitary
    theta = theta_exec(plan, gk, lk, gk1, ll, lr, U) # tn_theta_exec → list of N+1 complex128 tensors
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import (lib, check, TnError, STATUS, TN_BOND_LEFT, TN_BOND_CENTER, TN_BOND_RIGHT, TN_GATHER_NONE,
                   TN_GATHER_ROOT, TN_GATHER_SECTOR_OWNER, TN_MAX_N, TN_MAX_MIX, TN_CONTRACT_F64_DMMA, TN_CONTRACT_INT8_OZAKI, LIB_PATH,
                   TN_BCAST_NONE, TN_BCAST_SLABS, TN_BCAST_FULL, Transfer)

__all__ = ["TN_CONTRACT_F64_DMMA", "TN_CONTRACT_INT8_OZAKI", "Plan", "Plan2", "Comm", "svd_truncate", "build_bs_unitary", "theta_exec", "theta_exec_sharded", "alloc_theta",
           "shard_rows_host", "release_cached_memory", "TnError", "lib", "LIB_PATH", "TN_GATHER_NONE", "TN_GATHER_ROOT",
           "TN_GATHER_SECTOR_OWNER", "sector_owners_host", "TN_BCAST_NONE", "TN_BCAST_SLABS", "TN_BCAST_FULL",
           "gather_schedule_host", "pack_row_slab", "theta_exec_slab",
           "theta_exec_to_owners", "ipc_handle"]


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(int(stream.cuda_stream))


def _ptr(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        if not t.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(t.ctypes.data)
    raise TypeError(type(t))


def _charges(q):
    if isinstance(q, torch.Tensor):
        if q.dtype != torch.int32:
            q = q.to(torch.int32)
        return q.contiguous()
    return np.ascontiguousarray(np.asarray(q, dtype=np.int32))


def _ready(qs):
    # the plan reads device charges on its own stream (include/tn_theta.h): the producing work — typically on
    # the current stream (a dtype cast above, an SVD step's q_new) — must have finished
    if any(isinstance(q, torch.Tensor) and q.is_cuda for q in qs):
        torch.cuda.current_stream().synchronize()


class Plan:
    """tn_theta_plan: bond re-indexing (K1) and work decomposition for one gate's bond charges."""

    def __init__(self, d: int, N: int, q_l, q_c, q_r, world_size: int = 1, rank: int = 0):
        self._keep = [_charges(q) for q in (q_l, q_c, q_r)]
        _ready(self._keep)
        ql, qc, qr = self._keep
        self.d, self.N = int(d), int(N)
        self.chi = (int(ql.shape[0]), int(qc.shape[0]), int(qr.shape[0]))
        self.world_size, self.rank = int(world_size), int(rank)
        h = C.c_void_p()
        check(lib.tn_theta_plan(self.d, self.N, *self.chi, _ptr(ql), _ptr(qc), _ptr(qr), self.world_size,
                                self.rank, C.byref(h)), "tn_theta_plan")
        self._h = h
        self.nsec = self.N + 1
        del self._keep

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ValueError("plan destroyed")
        return self._h

    def destroy(self) -> None:
        if getattr(self, "_h", None) is not None:
            lib.tn_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def sector_shape(self, c: int):
        R, Cc = C.c_int64(), C.c_int64()
        check(lib.tn_plan_sector_shape(self.handle, int(c), C.byref(R), C.byref(Cc)), "tn_plan_sector_shape")
        return R.value, Cc.value

    def local_sector_shape(self, c: int):
        R, Cc, r0 = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.tn_plan_local_sector_shape(self.handle, int(c), C.byref(R), C.byref(Cc), C.byref(r0)),
              "tn_plan_local_sector_shape")
        return R.value, Cc.value, r0.value

    def perm(self, bond: int) -> np.ndarray:
        out = np.empty(self.chi[bond], dtype=np.int32)
        check(lib.tn_plan_perm(self.handle, int(bond), _ptr(out)), "tn_plan_perm")
        return out

    def offsets(self, bond: int) -> np.ndarray:
        out = np.empty(self.nsec + 1, dtype=np.int32)
        check(lib.tn_plan_offsets(self.handle, int(bond), _ptr(out)), "tn_plan_offsets")
        return out

    def shard_rows(self, r: int):
        a, b = C.c_int64(), C.c_int64()
        check(lib.tn_plan_shard_rows(self.handle, int(r), C.byref(a), C.byref(b)), "tn_plan_shard_rows")
        return a.value, b.value

    def sector_owner(self, c: int) -> int:
        o = C.c_int()
        check(lib.tn_plan_sector_owner(self.handle, int(c), C.byref(o)), "tn_plan_sector_owner")
        return o.value

    def flops(self):
        v = [C.c_int64() for _ in range(5)]
        check(lib.tn_plan_flops(self.handle, *(C.byref(x) for x in v)), "tn_plan_flops")
        return dict(zip(("f_contract", "f_mix", "f_exec", "f_contract_local", "f_mix_local"), (x.value for x in v)))

    def slab_rows(self, c: int, rank: int):
        """tn_plan_slab_rows: (first row, rows) of rank `rank`'s slab inside the full Θ(c)."""
        b, n = C.c_int64(), C.c_int64()
        check(lib.tn_plan_slab_rows(self.handle, int(c), int(rank), C.byref(b), C.byref(n)), "tn_plan_slab_rows")
        return b.value, n.value

    def gather_schedule(self, gather_mode: int):
        """tn_plan_gather_schedule: the transfer list tn_theta_exec_sharded executes, as a list of dicts
        (sector, src, dst, row_begin, rows, cols)."""
        n = C.c_int64()
        check(lib.tn_plan_gather_schedule(self.handle, int(gather_mode), 0, None, C.byref(n)), "tn_plan_gather_schedule")
        arr = (Transfer * max(1, n.value))()
        check(lib.tn_plan_gather_schedule(self.handle, int(gather_mode), n.value, arr, C.byref(n)),
              "tn_plan_gather_schedule")
        return [{f: getattr(arr[i], f) for f, _ in Transfer._fields_} for i in range(n.value)]

    def exec_launches(self) -> int:
        """tn_plan_exec_launches: kernel launches of one tn_theta_exec with the current engine."""
        n = C.c_int64()
        check(lib.tn_plan_exec_launches(self.handle, C.byref(n)), "tn_plan_exec_launches")
        return n.value

    def reserve(self, count: int) -> None:
        """tn_plan_reserve: pool blocks for `count` live plans of this shape (no cudaMalloc on the enqueue path
        of pipelined gates)."""
        check(lib.tn_plan_reserve(self.handle, int(count)), "tn_plan_reserve")

    def u_size(self) -> int:
        n = C.c_int64()
        check(lib.tn_plan_u_size(self.handle, C.byref(n)), "tn_plan_u_size")
        return n.value

    def set_contraction(self, mode, slices: int = 7):
        """tn_plan_set_contraction: "dmma" (FP64 tensor cores) or "int8" (tcgen05 INT8 emulation)."""
        m = {"dmma": TN_CONTRACT_F64_DMMA, "int8": TN_CONTRACT_INT8_OZAKI, "literal": 2}.get(mode, mode)
        check(lib.tn_plan_set_contraction(self.handle, int(m), int(slices)), "tn_plan_set_contraction")
        return self

    def contraction(self):
        m, s = C.c_int(), C.c_int()
        check(lib.tn_plan_get_contraction(self.handle, C.byref(m), C.byref(s)), "tn_plan_get_contraction")
        return {TN_CONTRACT_F64_DMMA: "dmma", TN_CONTRACT_INT8_OZAKI: "int8", 2: "literal"}[m.value], s.value

    def kernel_times(self):
        """Device ms of the most recent K1 (plan), K2, K3, K4, K5 launched with this plan (−1: not run)."""
        ms = np.empty(5, dtype=np.float32)
        check(lib.tn_plan_kernel_times(self.handle, _ptr(ms)), "tn_plan_kernel_times")
        return dict(zip(("k1_sort", "k2_unitary", "k3_stage", "k4_contract", "k5_mix"), ms.tolist()))

    def workspace_bytes(self) -> int:
        n = C.c_int64()
        check(lib.tn_plan_workspace_bytes(self.handle, C.byref(n)), "tn_plan_workspace_bytes")
        return n.value


class Plan2(Plan):
    """tn_theta2_plan: the MPO (doubled-charge) plan — every bond carries a charge pair (q1, q2); sectors are
    Θ(c1, c2), indexed s = c1·(N+1) + c2 (use `sector(c1, c2)`). theta_exec returns (N+1)² tensors."""

    def __init__(self, d: int, N: int, q1_l, q2_l, q1_c, q2_c, q1_r, q2_r, world_size: int = 1, rank: int = 0):
        self._keep = [_charges(q) for q in (q1_l, q2_l, q1_c, q2_c, q1_r, q2_r)]
        _ready(self._keep)
        k = self._keep
        self.d, self.N = int(d), int(N)
        self.chi = (int(k[0].shape[0]), int(k[2].shape[0]), int(k[4].shape[0]))
        self.world_size, self.rank = int(world_size), int(rank)
        h = C.c_void_p()
        check(lib.tn_theta2_plan(self.d, self.N, *self.chi, *(_ptr(x) for x in k), self.world_size, self.rank,
                                 C.byref(h)), "tn_theta2_plan")
        self._h = h
        self.nsec = (self.N + 1) ** 2
        del self._keep

    def sector(self, c1: int, c2: int) -> int:
        return int(c1) * (self.N + 1) + int(c2)


def build_bs_unitary(plan: Plan, theta: float, phi: float, out: torch.Tensor | None = None, stream=None):
    """tn_build_bs_unitary → packed complex128 U on the current device (layout in include/tn_theta.h)."""
    if out is None:
        out = torch.empty(plan.u_size(), dtype=torch.complex128, device="cuda")
    if out.dtype != torch.complex128 or out.numel() < plan.u_size() or not out.is_cuda:
        raise ValueError("U must be a CUDA complex128 tensor of tn_plan_u_size entries")
    check(lib.tn_build_bs_unitary(plan.handle, float(theta), float(phi), _stream_ptr(stream), _ptr(out)),
          "tn_build_bs_unitary")
    return out


def alloc_theta(plan: Plan, device="cuda", full: bool = False):
    """Device buffers for every sector: this rank's slabs (or the full Θ(c) if `full`)."""
    outs = []
    for c in range(plan.nsec):
        R, Cc = plan.sector_shape(c) if full else plan.local_sector_shape(c)[:2]
        outs.append(torch.empty((R, Cc), dtype=torch.complex128, device=device))
    return outs


def _theta_ptrs(outs):
    arr = (C.c_void_p * len(outs))()
    for i, t in enumerate(outs):
        if t is not None and t.numel() > 0:
            if t.dtype != torch.complex128 or not t.is_cuda:
                raise ValueError("Θ buffers must be CUDA complex128 tensors")
            arr[i] = _ptr(t).value
        else:
            arr[i] = None
    return arr


def _check_inputs(plan, gk, lk, gk1, ll, lr, U):
    chi_l, chi_c, chi_r = plan.chi
    for t, shp, dt in ((gk, (chi_l, chi_c) if gk is not None else None, torch.complex128),
                       (gk1, (chi_c, chi_r), torch.complex128),
                       (lk, (chi_c,), torch.float64), (ll, (chi_l,), torch.float64),
                       (lr, (chi_r,), torch.float64)):
        if shp is None:  # validated by the caller (a packed Γk slab)
            continue
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dt or tuple(t.shape) != shp:
            raise ValueError(f"expected CUDA {dt} tensor of shape {shp}")
    if not isinstance(U, torch.Tensor) or not U.is_cuda or U.dtype != torch.complex128 or U.numel() < plan.u_size():
        raise ValueError("U must be a CUDA complex128 tensor of tn_plan_u_size entries")


def theta_exec(plan: Plan, gk, lk, gk1, ll, lr, U, out=None, stream=None):
    """tn_theta_exec: every sector Θ(c), c = 0..N (this rank's slabs). Returns the list `out`."""
    _check_inputs(plan, gk, lk, gk1, ll, lr, U)
    if out is None:
        out = alloc_theta(plan)
    ptrs = _theta_ptrs(out)
    check(lib.tn_theta_exec(plan.handle, _stream_ptr(stream), _ptr(gk), _ptr(lk), _ptr(gk1), _ptr(ll), _ptr(lr),
                            _ptr(U), ptrs), "tn_theta_exec")
    return out


def pack_row_slab(plan: Plan, gk, rank: int, out=None, stream=None):
    """tn_pack_row_slab: rank `rank`'s rows of Γk packed in sorted order, a CUDA tensor [(r1−r0), χ_c]."""
    r0, r1 = plan.shard_rows(rank)
    if out is None:
        out = torch.empty((r1 - r0, plan.chi[1]), dtype=torch.complex128, device=gk.device)
    if out.numel() < (r1 - r0) * plan.chi[1] or out.dtype != torch.complex128 or not out.is_cuda:
        raise ValueError("slab buffer too small or not CUDA complex128")
    _check_inputs_gk(plan, gk)
    check(lib.tn_pack_row_slab(plan.handle, _stream_ptr(stream), _ptr(gk), int(rank), _ptr(out)), "tn_pack_row_slab")
    return out


def theta_exec_slab(plan: Plan, gk_slab, lk, gk1, ll, lr, U, out=None, stream=None):
    """tn_theta_exec_slab: tn_theta_exec for the plan's rank with Γk given as its packed row slab."""
    r0, r1 = plan.shard_rows(plan.rank)
    if not (isinstance(gk_slab, torch.Tensor) and gk_slab.is_cuda and gk_slab.dtype == torch.complex128
            and gk_slab.is_contiguous() and gk_slab.numel() >= (r1 - r0) * plan.chi[1]):
        raise ValueError("gk_slab must be a contiguous CUDA complex128 tensor of ≥ (r1−r0)·χ_c entries")
    _check_inputs(plan, None, lk, gk1, ll, lr, U)
    if out is None:
        out = alloc_theta(plan)
    check(lib.tn_theta_exec_slab(plan.handle, _stream_ptr(stream), _ptr(gk_slab), _ptr(lk), _ptr(gk1), _ptr(ll),
                                 _ptr(lr), _ptr(U), _theta_ptrs(out)), "tn_theta_exec_slab")
    return out


def _check_inputs_gk(plan, gk):
    if not isinstance(gk, torch.Tensor) or not gk.is_cuda or gk.dtype != torch.complex128 or \
            tuple(gk.shape) != (plan.chi[0], plan.chi[1]) or not gk.is_contiguous():
        raise ValueError(f"expected contiguous CUDA complex128 Γk of shape {(plan.chi[0], plan.chi[1])}")


def svd_truncate(plan: Plan, theta, ll, lr, chi_max: int, cutoff: float = 1e-14, stream=None, form: str = "vidal"):
    """tn_svd_truncate: per-sector SVD + global top-χ + new canonical factors (single-charge or MPO pair
    plans). `theta` (the list from theta_exec) is only read. Returns dict(chi, q_new, lam_new, gamma_k_new [χ_l × chi], gamma_k1_new
    [chi × χ_r], discarded) as contiguous CUDA tensors (views of chi_max-capacity buffers).
    form="b": tn_svd_truncate_bform — right-canonical factors B^{[k]}_new, B^{[k+1]}_new (`lr` unused)."""
    chi_l, _, chi_r = plan.chi
    dev = ll.device
    q_new = torch.zeros(chi_max, dtype=torch.int32, device=dev)
    lam_new = torch.zeros(chi_max, dtype=torch.float64, device=dev)
    gk = torch.empty((chi_l, chi_max), dtype=torch.complex128, device=dev)
    gk1 = torch.empty((chi_max, chi_r), dtype=torch.complex128, device=dev)
    chi_out, disc = C.c_int64(), C.c_double()
    if form == "b":
        check(lib.tn_svd_truncate_bform(plan.handle, _stream_ptr(stream), _theta_ptrs(theta), _ptr(ll), int(chi_max),
                                        float(cutoff), _ptr(q_new), _ptr(lam_new), _ptr(gk), _ptr(gk1),
                                        C.byref(chi_out), C.byref(disc)), "tn_svd_truncate_bform")
    else:
        check(lib.tn_svd_truncate(plan.handle, _stream_ptr(stream), _theta_ptrs(theta), _ptr(ll), _ptr(lr),
                                  int(chi_max), float(cutoff), _ptr(q_new), _ptr(lam_new), _ptr(gk), _ptr(gk1),
                                  C.byref(chi_out), C.byref(disc)), "tn_svd_truncate")
    k = chi_out.value
    res = dict(chi=k, q_new=q_new[:k], lam_new=lam_new[:k], gamma_k_new=gk.view(-1)[:chi_l * k].view(chi_l, k),
               gamma_k1_new=gk1[:k], discarded=disc.value)
    if isinstance(plan, Plan2):  # q_new holds the pair key c1·(N+1) + c2
        res["q1_new"], res["q2_new"] = q_new[:k] // (plan.N + 1), q_new[:k] % (plan.N + 1)
    return res


class Comm:
    """tn_comm over NCCL; the 128-byte unique id is distributed with a torch.distributed group."""

    def __init__(self, rank: int, world_size: int, group=None):
        import torch.distributed as dist
        uid = (C.c_char * 128)()
        if rank == 0:
            check(lib.tn_comm_unique_id(uid), "tn_comm_unique_id")
        obj = [bytes(uid)]
        if world_size > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib.tn_comm_init(uid, int(rank), int(world_size), C.byref(h)), "tn_comm_init")
        self._h, self.rank, self.world_size = h, rank, world_size

    @property
    def handle(self):
        return self._h

    def async_error(self) -> None:
        """tn_comm_async_error: raises TnError (TN_ERR_NCCL) if the communicator holds an asynchronous error."""
        check(lib.tn_comm_async_error(self._h), "tn_comm_async_error")

    def destroy(self):
        if self._h is not None:
            lib.tn_comm_destroy(self._h)
            self._h = None


def theta_exec_sharded(plan: Plan, comm: Comm, gk, lk, gk1, ll, lr, U, out=None, bcast_operands=TN_BCAST_NONE,
                       gather_mode=TN_GATHER_NONE, stream=None):
    """tn_theta_exec_sharded: this rank's rows (+ optional operand distribution from rank 0 and the NCCL gather
    to rank 0 / the sector owners). bcast_operands: TN_BCAST_NONE / TN_BCAST_SLABS (Γk row slabs; on ranks > 0
    `gk` receives the packed slab and may be any CUDA complex128 tensor with ≥ (r1−r0)·χ_c elements) /
    TN_BCAST_FULL; True means TN_BCAST_SLABS."""
    bc = int(bcast_operands) if not isinstance(bcast_operands, bool) else (TN_BCAST_SLABS if bcast_operands else TN_BCAST_NONE)
    if bc == TN_BCAST_SLABS and plan.rank > 0:
        r0, r1 = plan.shard_rows(plan.rank)
        if not (isinstance(gk, torch.Tensor) and gk.is_cuda and gk.dtype == torch.complex128 and gk.is_contiguous()
                and gk.numel() >= (r1 - r0) * plan.chi[1]):
            raise ValueError("TN_BCAST_SLABS: gk must be a contiguous CUDA complex128 tensor of ≥ (r1−r0)·χ_c entries")
        _check_inputs(plan, None, lk, gk1, ll, lr, U)
    else:
        _check_inputs(plan, gk, lk, gk1, ll, lr, U)
    if out is None:
        out = alloc_theta(plan, full=(gather_mode == TN_GATHER_ROOT and plan.rank == 0))
        if gather_mode == TN_GATHER_SECTOR_OWNER:
            for c in range(plan.nsec):
                if plan.sector_owner(c) == plan.rank:
                    out[c] = torch.empty(plan.sector_shape(c), dtype=torch.complex128, device=out[c].device)
    ptrs = _theta_ptrs(out)
    check(lib.tn_theta_exec_sharded(plan.handle, _stream_ptr(stream), comm.handle, _ptr(gk), _ptr(lk), _ptr(gk1),
                                    _ptr(ll), _ptr(lr), _ptr(U), ptrs, bc, int(gather_mode)),
          "tn_theta_exec_sharded")
    return out


def release_cached_memory():
    """tn_release_cached_memory → (bytes freed, bytes still held by live plans)."""
    f, c = C.c_int64(), C.c_int64()
    check(lib.tn_release_cached_memory(C.byref(f), C.byref(c)), "tn_release_cached_memory")
    return f.value, c.value


def shard_rows_host(d: int, N: int, n_l, n_c, n_r, world_size: int) -> np.ndarray:
    """tn_shard_rows_host: flop-balanced row-shard bounds from per-charge bond counts (no GPU)."""
    a = [np.ascontiguousarray(np.asarray(x, dtype=np.int64)) for x in (n_l, n_c, n_r)]
    for x in a:
        if x.shape != (N + 1,):
            raise ValueError("counts must have N+1 entries")
    out = np.empty(world_size + 1, dtype=np.int64)
    i64p = C.POINTER(C.c_int64)
    check(lib.tn_shard_rows_host(int(d), int(N), *(x.ctypes.data_as(i64p) for x in a), int(world_size),
                                 out.ctypes.data_as(i64p)), "tn_shard_rows_host")
    return out


def sector_owners_host(sizes, world_size: int) -> np.ndarray:
    """tn_sector_owners_host: the plan's TN_GATHER_SECTOR_OWNER assignment for element counts `sizes`."""
    sz = np.ascontiguousarray(np.asarray(sizes, dtype=np.int64))
    out = np.empty(sz.shape[0], dtype=np.int32)
    check(lib.tn_sector_owners_host(int(sz.shape[0]), sz.ctypes.data_as(C.POINTER(C.c_int64)), int(world_size),
                                    out.ctypes.data_as(C.POINTER(C.c_int32))), "tn_sector_owners_host")
    return out


def gather_schedule_host(d: int, N: int, off_l, off_r, bounds, gather_mode: int):
    """tn_gather_schedule_host: the gather transfer list from host offsets and shard bounds (no plan, no GPU)."""
    ol = np.ascontiguousarray(np.asarray(off_l, dtype=np.int32))
    orr = np.ascontiguousarray(np.asarray(off_r, dtype=np.int32))
    b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    if ol.shape != (N + 2,) or orr.shape != (N + 2,):
        raise ValueError("offsets must have N+2 entries")
    world = b.shape[0] - 1
    i32p, i64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    args = (int(d), int(N), ol.ctypes.data_as(i32p), orr.ctypes.data_as(i32p), int(world), b.ctypes.data_as(i64p),
            int(gather_mode))
    n = C.c_int64()
    check(lib.tn_gather_schedule_host(*args, 0, None, C.byref(n)), "tn_gather_schedule_host")
    arr = (Transfer * max(1, n.value))()
    check(lib.tn_gather_schedule_host(*args, n.value, arr, C.byref(n)), "tn_gather_schedule_host")
    return [{f: getattr(arr[i], f) for f, _ in Transfer._fields_} for i in range(n.value)]


def ipc_handle(t: torch.Tensor):
    """tn_ipc_get_handle: (64-byte handle, byte offset) exporting a CUDA tensor's memory to another process."""
    h = (C.c_char * 64)()
    off = C.c_int64()
    check(lib.tn_ipc_get_handle(_ptr(t), h, C.byref(off)), "tn_ipc_get_handle")
    return bytes(h), off.value


def theta_exec_to_owners(plan: Plan, gk, lk, gk1, ll, lr, U, group=None, stream=None):
    """The SECTOR_OWNER gather fused into the computation (tn_theta_exec_remote): every rank's K5 writes its
    slab of Θ(c) straight into the owner's full Θ(c) (CUDA IPC / NVLink peer memory); handles are exchanged
    with torch.distributed (any backend) and a barrier after the streams drain orders the owners' reads.
    Returns {c: full Θ(c)} for the sectors this rank owns."""
    import torch.distributed as dist
    _check_inputs(plan, gk, lk, gk1, ll, lr, U)
    world, rank = plan.world_size, plan.rank
    dev = gk.device
    owned = {}
    for c in range(plan.nsec):
        R, Cc = plan.sector_shape(c)
        if plan.sector_owner(c) == rank and R * Cc > 0:
            owned[c] = torch.empty((R, Cc), dtype=torch.complex128, device=dev)
    # the caching allocator may hand out blocks that this rank's pending kernels still use: peers write into
    # them through NVLink outside this stream's order, so drain the stream before publishing the handles
    (stream or torch.cuda.current_stream()).synchronize()
    mine = {c: ipc_handle(t) for c, t in owned.items()}
    allh = [None] * world
    if world > 1:
        dist.all_gather_object(allh, mine, group=group)
    else:
        allh = [mine]
    opened = {}
    dst = (C.c_void_p * plan.nsec)()
    try:
        for c in range(plan.nsec):
            R, Cc, row0 = plan.local_sector_shape(c)
            if R * Cc == 0:
                dst[c] = None
                continue
            o = plan.sector_owner(c)
            if o == rank:
                base = owned[c].data_ptr()
            else:
                hnd, off = allh[o][c]
                if hnd not in opened:
                    p = C.c_void_p()
                    check(lib.tn_ipc_open(hnd, C.byref(p)), "tn_ipc_open")
                    opened[hnd] = p.value
                base = opened[hnd] + off
            dst[c] = base + row0 * Cc * 16
        check(lib.tn_theta_exec_remote(plan.handle, _stream_ptr(stream), _ptr(gk), _ptr(lk), _ptr(gk1), _ptr(ll),
                                       _ptr(lr), _ptr(U), dst), "tn_theta_exec_remote")
        (stream or torch.cuda.current_stream()).synchronize()
        if world > 1:
            dist.barrier(group=group)
    finally:
        for p in opened.values():
            lib.tn_ipc_close(C.c_void_p(p))
    return owned
