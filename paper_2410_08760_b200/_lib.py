"""ctypes binding of libfednl_b200.so (include/fednl_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (or
`python -m paper_2410_08760_b200.build`).  There is no fallback: if the
library or a CUDA device is missing, every device-backed call raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfednl_b200.so")

FB_OK = 0
FB_ERR_CUDA = 1
FB_ERR_INVALID = 2
FB_ERR_NOT_PD = 3
FB_ERR_NONFINITE = 4
FB_ERR_DIVERGED = 5
FB_ERR_LINE_SEARCH = 6
FB_ERR_UNSUPPORTED = 7
FB_ERR_EIGEN = 9

TOPK_PATH_AUTO, TOPK_PATH_STREAM, TOPK_PATH_SPLIT = 0, 1, 2
BSTORE_AUTO, BSTORE_F64 = 0, 1

ALG_CODE = {"fednl": 0, "fednl-ls": 1, "fednl-pp": 2}
INIT_CODE = {"lambda-identity": 0, "zero": 1, "exact": 2}


class FbConfig(C.Structure):
    _fields_ = [
        ("d", C.c_int32),
        ("n_clients", C.c_int32),
        ("n_samples", C.c_int32),
        ("algorithm", C.c_int32),
        ("kind", C.c_int32),
        ("k", C.c_int32),
        ("topk_weighted", C.c_int32),
        ("tau", C.c_int32),
        ("hessian_init", C.c_int32),
        ("option", C.c_int32),
        ("alpha", C.c_double),
        ("lam", C.c_double),
        ("ls_c", C.c_double),
        ("ls_gamma", C.c_double),
        ("run_seed", C.c_uint64),
        ("ls_steps_table", C.c_double * 61),
        ("mu", C.c_double),
        ("topk_path", C.c_int32),
        ("b_store", C.c_int32),
    ]


class FbStatus(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("round", C.c_int32),
        ("pivot_index", C.c_int32),
        ("client", C.c_int32),
        ("pivot_value", C.c_double),
        ("f_start", C.c_double),
        ("f_best", C.c_double),
    ]


class FbProfile(C.Structure):
    _fields_ = [
        ("rounds", C.c_int32),
        ("launches_per_round", C.c_int32),
        ("ms_oracle", C.c_double),
        ("ms_hessian", C.c_double),
        ("ms_reduce", C.c_double),
        ("ms_compress", C.c_double),
        ("ms_solve", C.c_double),
        ("ms_fold", C.c_double),
        ("ms_round", C.c_double),
    ]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_U32 = C.POINTER(C.c_uint32)
_U64 = C.POINTER(C.c_uint64)
_I64 = C.POINTER(C.c_int64)

# every symbol include/fednl_b200.h declares, with its prototype
PROTOTYPES = {
    "fb_abi_sizes": (C.c_int, [_I32]),
    "fb_create": (C.c_int, [C.POINTER(FbConfig), C.POINTER(C.c_void_p)]),
    "fb_destroy": (None, [_P]),
    "fb_last_error": (C.c_char_p, [_P]),
    "fb_get_status": (C.c_int, [_P, C.POINTER(FbStatus)]),
    "fb_device_info": (C.c_int, [C.c_char_p, C.c_int32, _I32, _I32, _I32]),
    "fb_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "fb_set_shard": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_uint8)]),
    "fb_upload_shards": (C.c_int, [_P, C.POINTER(_D)]),
    "fb_upload_shards_ex": (C.c_int, [_P, C.POINTER(_D), _I32, _D]),
    "fb_bstore_kind": (C.c_int, [_P]),
    "fb_init_state": (C.c_int, [_P, _D]),
    "fb_run_rounds": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_double, C.c_int32, _D, _D, _I32,
                                _I32, _D, _I32]),
    "fb_final_eval": (C.c_int, [_P, _D, _D]),
    "fb_get_profile": (C.c_int, [_P, C.POINTER(FbProfile)]),
    "fb_get_x": (C.c_int, [_P, _D]),
    "fb_set_x": (C.c_int, [_P, _D]),
    "fb_get_client_hest": (C.c_int, [_P, C.c_int32, C.c_int32, _D]),
    "fb_set_client_hest": (C.c_int, [_P, C.c_int32, C.c_int32, _D]),
    "fb_get_master_hest": (C.c_int, [_P, _D]),
    "fb_set_master_hest": (C.c_int, [_P, _D]),
    "fb_get_pp_state": (C.c_int, [_P, _D, _D, _D, _D]),
    "fb_get_round_diff": (C.c_int, [_P, C.c_int32, _D]),
    "fb_get_round_delta": (C.c_int, [_P, C.c_int32, _U32, _D, _I32]),
    "fb_get_round_grads": (C.c_int, [_P, _D, _D]),
    "fb_get_round_scalars": (C.c_int, [_P, _D, _D]),
    "fb_compress": (C.c_int, [_P, _D, _U64, _U32, _D, _I32, _I32]),
    "fb_oracle_eval": (C.c_int, [_P, _D, _D, _D, _D]),
    "fb_shifted_solve": (C.c_int, [_P, _D, C.c_double, _D, _D]),
    "fb_eigen_clamp": (C.c_int, [_P, _D, C.c_double, _D, _D, _D]),
    "fb_solve_phase_cycles": (C.c_int, [_P, _D, C.c_double, _D, C.c_int32, C.POINTER(C.c_longlong),
                                        C.POINTER(C.c_float)]),
    "fb_debug_counters": (C.c_int, [C.c_int32, C.POINTER(C.c_longlong)]),
    "fb_debug_timeline": (C.c_int, [C.POINTER(C.c_ulonglong)]),
    "fb_prg_u64": (C.c_int, [C.c_uint64, C.c_int32, _U64]),
    "fb_prg_randrange": (C.c_int, [C.c_uint64, _U64, C.c_int32, C.c_int32, _U64, _U64]),
    "fb_prg_partial_shuffle": (C.c_int, [C.c_uint64, C.c_int64, C.c_int32, _I64]),
    "fb_round_seeds": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, _U64]),
    "fb_fp64_peak": (C.c_int, [_D, _D]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load() -> C.CDLL:
    """Load the library (once) and attach prototypes; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def last_error(ctx=None) -> str:
    msg = load().fb_last_error(ctx)
    return msg.decode() if msg else ""


def check(rc: int, ctx=None, what: str = "") -> None:
    if rc != FB_OK:
        raise RuntimeError(f"{what or 'libfednl_b200'} failed (code {rc}): {last_error(ctx)}")


def device_info() -> dict:
    lib = load()
    name = C.create_string_buffer(128)
    sms, ma, mi = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib.fb_device_info(name, 128, C.byref(sms), C.byref(ma), C.byref(mi)), None, "fb_device_info")
    return {"name": name.value.decode(), "sm_count": sms.value, "cc": (ma.value, mi.value)}
