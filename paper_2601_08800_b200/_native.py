"""ctypes binding of the C-ABI library (``include/mixserve_b200.h``).

The shared object is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2601_08800_b200/csrc``) into
``paper_2601_08800_b200/lib/libmixserve_b200.so``.  There is no fallback:
if the library is missing every entry point raises ``NativeLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import CapacityError, MoeplanError, StrategyError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmixserve_b200.so"

MX_OK = 0
MX_ERR_INVALID = -1
MX_ERR_CAPACITY = -2
MX_ERR_CUDA = -3
MX_ERR_UNSUPPORTED = -4
MX_ERR_TIMEOUT = -5

MX_F64, MX_F32, MX_BF16 = 0, 1, 2
MX_EXPERT_AFFINE, MX_EXPERT_SWIGLU, MX_EXPERT_SWIGLU_FP8 = 0, 1, 2
MX_WIRE_SLOT, MX_WIRE_TOKEN = 0, 1
MX_ROUTER_SOFTMAX, MX_ROUTER_GROUP_LIMITED = 0, 1
(MX_BUF_RECV, MX_BUF_PARTIAL, MX_BUF_Y, MX_BUF_IDS, MX_BUF_WEIGHTS,
 MX_BUF_SLOT_POS, MX_BUF_SLOT_TM, MX_BUF_CNT_ALL, MX_BUF_EXP_OFF,
 MX_BUF_EXP_CNT, MX_BUF_SEND, MX_BUF_ACT, MX_BUF_UPOS, MX_BUF_XBUF,
 MX_BUF_STAMPS) = range(15)


class NativeLibraryError(MoeplanError, RuntimeError):
    """The CUDA extension is missing or failed; there is no CPU fallback."""


class PlanDesc(C.Structure):
    _fields_ = [("n_group", C.c_int), ("tp", C.c_int), ("tokens", C.c_int),
                ("hidden", C.c_int), ("num_experts", C.c_int),
                ("top_k", C.c_int), ("inter", C.c_int),
                ("act_dtype", C.c_int), ("expert_kind", C.c_int),
                ("renormalize", C.c_int), ("wire", C.c_int),
                ("shared_inter", C.c_int), ("capacity", C.c_longlong),
                ("router", C.c_int), ("router_groups", C.c_int),
                ("router_topk_groups", C.c_int), ("routed_scaling", C.c_float),
                ("router_bias", C.c_void_p)]


class ExpertParams(C.Structure):
    _fields_ = [("scales", C.c_void_p), ("biases", C.c_void_p),
                ("w13", C.c_void_p), ("w2", C.c_void_p),
                ("w13_scale", C.c_void_p), ("w2_scale", C.c_void_p),
                ("w13_shared", C.c_void_p), ("w2_shared", C.c_void_p),
                ("w13_shared_scale", C.c_void_p), ("w2_shared_scale", C.c_void_p)]


VP, I, LL, SZ = C.c_void_p, C.c_int, C.c_longlong, C.c_size_t
PSZ = C.POINTER(C.c_size_t)
PVP = C.POINTER(C.c_void_p)

# name -> argtypes (every entry point returns int)
SIGNATURES = {
    "mx_abi_version": [],
    "mx_device_sm_count": [I, C.POINTER(C.c_int)],
    "mx_comm_create": [I, I, I, I, SZ, PVP],
    "mx_comm_ipc_handle": [VP, VP],
    "mx_comm_open_peers": [VP, VP],
    "mx_comm_heap": [VP, I, PVP, PSZ],
    "mx_comm_destroy": [VP],
    "mx_comm_barrier": [VP, VP],
    "mx_comm_barrier_split": [VP, I, I, VP],
    "mx_plan_heap_bytes": [C.POINTER(PlanDesc), PSZ],
    "mx_plan_create": [VP, C.POINTER(PlanDesc), PVP],
    "mx_plan_destroy": [VP],
    "mx_plan_buffer": [VP, I, I, PVP, PSZ],
    "mx_route": [VP, I, VP, VP, VP, VP],
    "mx_layout": [VP, I, I, VP],
    "mx_dispatch": [VP, I, VP, VP],
    "mx_expert": [VP, I, C.POINTER(ExpertParams), VP],
    "mx_expert_stage": [VP, I, C.POINTER(ExpertParams), I, VP],
    "mx_combine": [VP, I, VP, VP],
    "mx_stamp": [VP, I, I, VP],
    "mx_forward": [VP, I, VP, VP, VP, VP, C.POINTER(ExpertParams), VP, VP],
    "mx_plan_check": [VP, I, VP],
    "mx_nvlink_probe": [VP, SZ, VP],
    "mx_baseline_dispatch_pack": [VP, I, VP, VP, VP, VP],
    "mx_baseline_dispatch_unpack": [VP, I, VP, VP],
    "mx_baseline_combine_pack": [VP, I, VP, VP, VP],
    "mx_baseline_combine_unpack": [VP, I, VP, VP, VP],
    "mx_swiglu_pack_w13": [VP, VP, VP, I, I, I, VP],
    "mx_dense_moe": [I, I, I, I, I, I, I, VP, VP, VP, VP, VP, VP, VP, VP,
                     VP, VP],
    "mx_grouped_gemm": [VP, VP, VP, I, VP, VP, I, LL, I, I, I, VP],
    "mx_quant_rows_e4m3": [VP, LL, VP, LL, LL, I, VP],
    "mx_grouped_gemm_fp8": [VP, LL, VP, VP, VP, VP, VP, I, LL, I, I, I, VP],
}

_lib = None


def load():
    """Load (once) and return the library; raise if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("MIXSERVE_B200_LIB", LIB_PATH))
    if not path.exists():
        raise NativeLibraryError(
            f"CUDA extension not built: {path} is missing. Run "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback).")
    lib = C.CDLL(str(path))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = C.c_int
    lib.mx_last_error.argtypes = []
    lib.mx_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Map an MX_ERR_* code to the reference's exception hierarchy
    (errors.py:16-41): invalid -> StrategyError, capacity -> CapacityError."""
    if rc == MX_OK:
        return
    msg = load().mx_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == MX_ERR_INVALID:
        raise StrategyError(msg)
    if rc == MX_ERR_CAPACITY:
        raise CapacityError(msg)
    raise NativeLibraryError(f"[{rc}] {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
