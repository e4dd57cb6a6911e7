"""ctypes loader for libautooverlap.so (the C ABI of include/autooverlap.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of the
library.  Importing fails loudly when the shared library is missing (there is no CPU
fallback); `python -m paper_2601_20595_b200.build` builds it in-tree.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libautooverlap.so")

AO_MAX_WORLD = 8
AO_HANDLE_BYTES = 256

STATUS = {0: "AO_OK", 1: "AO_ERR_INVALID_ARG", 2: "AO_ERR_UNSUPPORTED", 3: "AO_ERR_CUDA", 4: "AO_ERR_OOM",
          5: "AO_ERR_PEER", 6: "AO_ERR_TIMEOUT", 7: "AO_ERR_STATE"}
OPS = {"ag_gemm": 0, "gemm_rs": 1, "gemm_ar": 2, "a2a_gemm": 3, "sp_attn": 4, "hp_attn": 5}
BACKENDS = {"ce": 0, "tma": 1, "ldst": 2}
DIRS = {"push": 0, "pull": 1}
CHUNK_ORDERS = {"shard_major": 0, "chunk_major": 1}
INTRAS = {"row": 0, "col": 1, "grouped": 2}
WIRES = {"fp32": 0, "bf16": 1}
RS_REDUCE = {"slots": 0, "atomic": 1}


class AOError(RuntimeError):
    def __init__(self, status, detail):
        self.status = STATUS.get(status, str(status))
        super().__init__(f"{self.status}: {detail}")


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("op", ctypes.c_int32),
        ("world_size", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("M", ctypes.c_int64),
        ("N", ctypes.c_int64),
        ("K", ctypes.c_int64),
        ("chunk_rows", ctypes.c_int32),
        ("backend", ctypes.c_int32),
        ("dir", ctypes.c_int32),
        ("chunk_order", ctypes.c_int32),
        ("intra", ctypes.c_int32),
        ("group_m", ctypes.c_int32),
        ("tile_m", ctypes.c_int32),
        ("tile_n", ctypes.c_int32),
        ("n_cta", ctypes.c_int32),
        ("comm_ctas", ctypes.c_int32),
        ("n_slices", ctypes.c_int32),
        ("rs_wire", ctypes.c_int32),
        ("timeout_ns", ctypes.c_uint64),
        ("rs_reduce", ctypes.c_int32),
        ("topk", ctypes.c_int32),
        ("causal", ctypes.c_int32),
        ("stream_k", ctypes.c_int32),
    ]


class HandleBlob(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * AO_HANDLE_BYTES)]


_lib = None

# (name, restype-is-status, argtypes)
_SIGS = {
    "ao_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "ao_last_error": (ctypes.c_char_p, []),
    "ao_version": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "ao_plan_desc_init": (ctypes.c_int, [ctypes.POINTER(PlanDesc)]),
    "ao_plan_validate": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t,
                                        ctypes.POINTER(ctypes.c_int)]),
    "ao_plan_create_host": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "ao_plan_export_json": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t,
                                           ctypes.POINTER(ctypes.c_size_t)]),
    "ao_plan_hash": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]),
    "ao_plan_info": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int32)] * 6),
    "ao_plan_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.POINTER(ctypes.c_size_t)]),
    "ao_plan_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "ao_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_size_t,
                                     ctypes.POINTER(ctypes.c_void_p)]),
    "ao_ctx_export_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HandleBlob)]),
    "ao_ctx_import_handles": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HandleBlob)]),
    "ao_ctx_check_async": (ctypes.c_int, [ctypes.c_void_p]),
    "ao_ctx_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "ao_plan_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PlanDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "ao_ag_gemm": (ctypes.c_int, [ctypes.c_void_p] * 6),
    "ao_gemm_rs": (ctypes.c_int, [ctypes.c_void_p] * 5),
    "ao_ag_gemm_group": (ctypes.c_int, [ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 5 + [ctypes.c_void_p]),
    "ao_gemm_rs_group": (ctypes.c_int, [ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 4 + [ctypes.c_void_p]),
    "ao_gemm_ar": (ctypes.c_int, [ctypes.c_void_p] * 5),
    "ao_gemm_ar_group": (ctypes.c_int, [ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 4 + [ctypes.c_void_p]),
    "ao_group_schedule_export": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                                ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t,
                                                ctypes.POINTER(ctypes.c_size_t)]),
    "ao_a2a_gemm": (ctypes.c_int, [ctypes.c_void_p] * 8),
    "ao_a2a_gemm_group": (ctypes.c_int, [ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 7 + [ctypes.c_void_p]),
    "ao_sp_attn": (ctypes.c_int, [ctypes.c_void_p] * 6),
    "ao_sp_attn_group": (ctypes.c_int, [ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 5 + [ctypes.c_void_p]),
    "ao_hp_attn": (ctypes.c_int, [ctypes.c_void_p] * 6),
    "ao_hp_attn_group": (ctypes.c_int, [ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 5 + [ctypes.c_void_p]),
    "ao_gemm": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]),
    "ao_gemm_batched": (ctypes.c_int, [ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 3 +
                        [ctypes.c_int64] * 3 + [ctypes.c_int32] * 4 + [ctypes.c_void_p]),
    "ao_debug_set": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64]),
    "ao_transfer_bench": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_float)]),
    "ao_device_query": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]),
    "ao_ctx_trace_enable": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    "ao_ctx_trace_dump": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]),
}

EXPORTED = sorted(_SIGS)


def lib():
    """The loaded library (raises ImportError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2601_20595_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status):
    if status != 0:
        detail = lib().ao_last_error().decode(errors="replace")
        raise AOError(status, detail)


def make_desc(d: dict) -> PlanDesc:
    """Dict with the oracle's desc keys (oracle/schedule.py default_desc) -> PlanDesc."""
    x = PlanDesc()
    check(lib().ao_plan_desc_init(ctypes.byref(x)))
    x.op = OPS[d.get("op", "ag_gemm")]
    x.world_size = int(d.get("world_size", 1))
    x.rank = int(d.get("rank", 0))
    x.M, x.N, x.K = int(d["M"]), int(d["N"]), int(d["K"])
    x.chunk_rows = int(d.get("chunk_rows", 128))
    x.backend = BACKENDS[d.get("backend", "ce")]
    x.dir = DIRS[d.get("dir", "push")]
    x.chunk_order = CHUNK_ORDERS[d.get("chunk_order", "shard_major")]
    x.intra = INTRAS[d.get("intra", "row")]
    x.group_m = int(d.get("group_m", 1))
    x.tile_m = int(d.get("tile_m", 0))
    x.tile_n = int(d.get("tile_n", 0))
    x.n_cta = int(d.get("n_cta", 0))
    x.comm_ctas = int(d.get("comm_ctas", 0))
    x.n_slices = int(d.get("n_slices", 1))
    x.rs_wire = WIRES[d.get("rs_wire", "fp32")]
    x.timeout_ns = int(d.get("timeout_ns", 0))
    x.rs_reduce = RS_REDUCE[d.get("rs_reduce", "slots")]
    x.topk = int(d.get("topk", 0))
    x.causal = int(d.get("causal", 0))
    x.stream_k = int(d.get("stream_k", 0))
    return x
