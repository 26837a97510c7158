"""ctypes binding of include/shardweave_b200.h (the C ABI).

The library is built in-tree (`make`, or `__graft_entry__.build()`); there is no fallback:
a missing or unloadable library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# SW_LIB_PATH: load an experiment build instead (`make variant`); still no fallback
LIB_PATH = os.environ.get("SW_LIB_PATH") or os.path.join(_HERE, "libshardweave_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "shardweave_b200.h")

STATUS_NAMES = {
    0: "OK", 1: "SHAPE", 2: "PARTITION", 3: "CONFIG", 4: "NONFINITE", 5: "CHECKPOINT",
    6: "AUTODIFF", 7: "CUDA", 8: "NCCL", 9: "INTERNAL",
}


class SwError(RuntimeError):
    """Raised for a non-OK sw_status; `.status` holds the code name."""

    def __init__(self, status: int, message: str):
        super().__init__(f"[{STATUS_NAMES.get(status, status)}] {message}")
        self.status = STATUS_NAMES.get(status, str(status))
        self.message = message


class ShapeError(SwError):
    pass


class PartitionError(SwError):
    pass


class ConfigError(SwError):
    pass


class NonFiniteError(SwError):
    pass


class CheckpointError(SwError):
    """Corrupt or truncated snapshot (errors.hpp:23-35); the message carries the byte offset."""


_ERR_CLASSES = {1: ShapeError, 2: PartitionError, 3: ConfigError, 4: NonFiniteError, 5: CheckpointError}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build()) first")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().sw_last_error().decode()
        raise _ERR_CLASSES.get(status, SwError)(status, msg)


def declared_symbols() -> list[str]:
    """Every function name declared in include/shardweave_b200.h."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"SW_API\s+[^;(]*?\b(sw_\w+)\s*\(", text)))


def take_string(ptr: C.c_void_p) -> str:
    if not ptr:
        return ""
    s = C.cast(ptr, C.c_char_p).value.decode()
    lib().sw_free(ptr)
    return s


vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f32 = C.c_float
f64 = C.c_double


def _declare(L: C.CDLL) -> None:
    L.sw_last_error.restype = C.c_char_p
    L.sw_version.restype = C.c_char_p
    L.sw_free.argtypes = [vp]
    L.sw_free.restype = None
    L.sw_k_gemm_bf16.argtypes = [C.c_int, C.c_int, C.c_int, vp, i64, C.c_int, vp, i64, C.c_int,
                                 C.c_int, vp, i64, vp, i64, vp, vp, i64, f32, C.c_int, vp]
    L.sw_k_gemm_bf16.restype = C.c_int
    L.sw_k_attention_fwd.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]
    L.sw_k_decode_attention.argtypes = [vp, vp, vp] + [C.c_int] * 6 + [vp, vp, vp]
    L.sw_k_decode_attention.restype = C.c_int
    L.sw_k_attention_bwd.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]
    L.sw_k_attention_bwd_scratch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
    L.sw_k_attention_bwd_scratch.restype = C.c_longlong
    L.sw_k_layernorm_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, C.c_int, f32, vp]
    L.sw_k_layernorm_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, C.c_int, C.c_int, vp]
    L.sw_k_gemm_bf16_swiglu.argtypes = [C.c_int, C.c_int, C.c_int, vp, i64, vp, i64, vp, i64, vp, i64, vp]
    L.sw_k_gemm_bf16_swiglu_bwd.argtypes = [C.c_int, C.c_int, C.c_int, vp, i64, C.c_int, vp, i64, C.c_int, vp,
                                            i64, vp, i64, vp]
    L.sw_k_rmsnorm_fwd.argtypes = [vp, vp, vp, vp, i64, C.c_int, f32, vp]
    L.sw_k_rmsnorm_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, C.c_int, C.c_int, vp]
    L.sw_k_xent.argtypes = [vp, i64, i64, C.c_int, vp, vp, vp, vp, C.c_int, vp]
    L.sw_k_adamw.argtypes = [vp, vp, vp, vp, vp, i64, f32, f32, f32, f32, f32, f32, f32, vp]
    L.sw_k_gemm_bf16_adamw.argtypes = [C.c_int, C.c_int, C.c_int, vp, i64, C.c_int, vp, i64, C.c_int,
                                       vp, vp, vp, vp, i64, vp, f32, f32, f32, f32, f32, f32, f32, vp]
    for fn in ("sw_k_attention_fwd", "sw_k_attention_bwd", "sw_k_layernorm_fwd",
               "sw_k_layernorm_bwd", "sw_k_xent", "sw_k_adamw", "sw_k_gemm_bf16_adamw",
               "sw_k_rmsnorm_fwd", "sw_k_rmsnorm_bwd", "sw_k_gemm_bf16_swiglu", "sw_k_gemm_bf16_swiglu_bwd"):
        getattr(L, fn).restype = C.c_int
