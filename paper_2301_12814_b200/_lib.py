"""ctypes binding of libtn_theta.so (include/tn_theta.h). Argument marshalling only: every step of
the Θ path runs in the library's sm_100a kernels; there is no Python or CPU fallback. If the shared
library is missing this module raises ImportError (build it with `python -m paper_2301_12814_b200.build`
or `__graft_entry__.build()`)."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtn_theta.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2301_12814_b200.build` "
                      "(the Θ path has no CPU fallback)")
lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

STATUS = {0: "TN_OK", 1: "TN_ERR_DOMAIN", 2: "TN_ERR_DIMENSION", 3: "TN_ERR_CONSISTENCY", 4: "TN_ERR_CUDA",
          5: "TN_ERR_OOM", 6: "TN_ERR_NCCL", 7: "TN_ERR_UNSUPPORTED"}
TN_BOND_LEFT, TN_BOND_CENTER, TN_BOND_RIGHT = 0, 1, 2
TN_GATHER_NONE, TN_GATHER_ROOT, TN_GATHER_SECTOR_OWNER = 0, 1, 2
TN_BCAST_NONE, TN_BCAST_SLABS, TN_BCAST_FULL = 0, 1, 2


class Transfer(C.Structure):
    """tn_transfer: rank `src`'s slab of `sector` (rows × cols) lands at row `row_begin` of the full Θ on `dst`."""
    _fields_ = [("sector", C.c_int64), ("src", C.c_int64), ("dst", C.c_int64), ("row_begin", C.c_int64),
                ("rows", C.c_int64), ("cols", C.c_int64)]

TN_CONTRACT_F64_DMMA, TN_CONTRACT_INT8_OZAKI = 0, 1
TN_MAX_N, TN_MAX_MIX = 100, 64

_p = C.c_void_p
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)

# name: (argtypes) — every function returns tn_status (int) unless listed in _RESTYPE
SIGNATURES = {
    "tn_theta_plan": [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, _p, _p, _p, C.c_int, C.c_int,
                      C.POINTER(_p)],
    "tn_theta2_plan": [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, _p, _p, _p, _p, _p, _p, C.c_int, C.c_int,
                       C.POINTER(_p)],
    "tn_plan_destroy": [_p],
    "tn_plan_sector_shape": [_p, C.c_int, _i64p, _i64p],
    "tn_plan_local_sector_shape": [_p, C.c_int, _i64p, _i64p, _i64p],
    "tn_plan_perm": [_p, C.c_int, _p],
    "tn_plan_offsets": [_p, C.c_int, _p],
    "tn_plan_shard_rows": [_p, C.c_int, _i64p, _i64p],
    "tn_plan_flops": [_p, _i64p, _i64p, _i64p, _i64p, _i64p],
    "tn_plan_u_size": [_p, _i64p],
    "tn_plan_exec_launches": [_p, _i64p],
    "tn_plan_reserve": [_p, C.c_int32],
    "tn_plan_slab_rows": [_p, C.c_int, C.c_int, _i64p, _i64p],
    "tn_plan_gather_schedule": [_p, C.c_int, C.c_int64, _p, _i64p],
    "tn_gather_schedule_host": [C.c_int, C.c_int, _i32p, _i32p, C.c_int, _i64p, C.c_int, C.c_int64, _p, _i64p],
    "tn_comm_async_error": [_p],
    "tn_pack_row_slab": [_p, _p, _p, C.c_int, _p],
    "tn_theta_exec_slab": [_p, _p, _p, _p, _p, _p, _p, _p, C.POINTER(_p)],
    "tn_plan_workspace_bytes": [_p, _i64p],
    "tn_plan_kernel_times": [_p, _p],
    "tn_plan_set_contraction": [_p, C.c_int, C.c_int],
    "tn_plan_get_contraction": [_p, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "tn_release_cached_memory": [_i64p, _i64p],
    "tn_build_bs_unitary": [_p, C.c_double, C.c_double, _p, _p],
    "tn_theta_exec": [_p, _p, _p, _p, _p, _p, _p, _p, C.POINTER(_p)],
    "tn_svd_truncate": [_p, _p, C.POINTER(_p), _p, _p, C.c_int64, C.c_double, _p, _p, _p, _p, _i64p,
                        C.POINTER(C.c_double)],
    "tn_svd_truncate_bform": [_p, _p, C.POINTER(_p), _p, C.c_int64, C.c_double, _p, _p, _p, _p, _i64p,
                              C.POINTER(C.c_double)],
    "tn_theta_exec_remote": [_p, _p, _p, _p, _p, _p, _p, _p, C.POINTER(_p)],
    "tn_ipc_get_handle": [_p, _p, _i64p],
    "tn_ipc_open": [_p, C.POINTER(_p)],
    "tn_ipc_close": [_p],
    "tn_comm_unique_id": [_p],
    "tn_comm_init": [_p, C.c_int, C.c_int, C.POINTER(_p)],
    "tn_comm_destroy": [_p],
    "tn_theta_exec_sharded": [_p, _p, _p, _p, _p, _p, _p, _p, _p, C.POINTER(_p), C.c_int, C.c_int],
    "tn_shard_rows_host": [C.c_int, C.c_int, _i64p, _i64p, _i64p, C.c_int, _i64p],
    "tn_sector_owners_host": [C.c_int, _i64p, C.c_int, _i32p],
    "tn_plan_sector_owner": [_p, C.c_int, C.POINTER(C.c_int)],
    "tn_status_string": [C.c_int],
    "tn_last_error": [],
    "tn_version": [],
}
_RESTYPE = {"tn_status_string": C.c_char_p, "tn_last_error": C.c_char_p, "tn_version": C.c_int}

for _name, _args in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _RESTYPE.get(_name, C.c_int)


class TnError(RuntimeError):
    """A non-TN_OK status from the library; `.status` holds its name."""

    def __init__(self, status: int, where: str):
        self.status = STATUS.get(status, str(status))
        detail = lib.tn_last_error().decode(errors="replace")
        super().__init__(f"{where}: {self.status}: {detail}")


def check(st: int, where: str) -> None:
    if st != 0:
        raise TnError(st, where)
