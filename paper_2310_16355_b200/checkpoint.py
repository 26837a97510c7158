"""Host-side SWCK snapshot codec (the reference's checkpoint format, checkpoint.hpp:18-28),
through the C ABI's sw_checkpoint_* functions. Device state moves through
engine.Model.save_checkpoint / load_checkpoint; this module reads and writes files without a
GPU (inspection, conversion, tests)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib


def _declare():
    L = _lib.lib()
    if getattr(L, "_ckpt_declared", False):
        return L
    vp, u64p = C.c_void_p, C.POINTER(C.c_uint64)
    L.sw_checkpoint_read.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.sw_checkpoint_info.argtypes = [vp, u64p, u64p, C.POINTER(C.c_uint32), u64p]
    L.sw_checkpoint_rng.argtypes = [vp, C.c_uint32, C.POINTER(C.c_char_p), u64p, u64p, u64p]
    L.sw_checkpoint_record.argtypes = [vp, C.c_uint64, C.POINTER(C.c_char_p), C.POINTER(C.c_uint32),
                                       C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_float)),
                                       C.POINTER(C.c_int64)]
    L.sw_checkpoint_write.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(C.c_char_p), u64p,
                                      u64p, u64p, C.c_uint64, C.POINTER(C.c_char_p), C.POINTER(C.c_uint32),
                                      C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_float))]
    L.sw_checkpoint_free.argtypes = [vp]
    L.sw_checkpoint_free.restype = None
    for fn in ("sw_checkpoint_read", "sw_checkpoint_info", "sw_checkpoint_rng", "sw_checkpoint_record",
               "sw_checkpoint_write"):
        getattr(L, fn).restype = C.c_int
    L._ckpt_declared = True
    return L


@dataclass
class Snapshot:
    """LoadedCheckpoint (checkpoint.hpp:222-226) before re-sharding: gathered full tensors."""
    step: int = 0
    seed: int = 0
    rngs: list = field(default_factory=list)      # [(name, seed, stream_id, counter)]
    records: list = field(default_factory=list)   # [(name, np.ndarray float32)] in file order

    def tensors(self, kind: str = "params") -> dict:
        return {n[len(kind) + 1:]: a for n, a in self.records if n.startswith(kind + "/")}


def read(path: str) -> Snapshot:
    L = _declare()
    h = C.c_void_p()
    _lib.check(L.sw_checkpoint_read(path.encode(), C.byref(h)))
    try:
        step, seed, nr = C.c_uint64(), C.c_uint64(), C.c_uint64()
        ng = C.c_uint32()
        _lib.check(L.sw_checkpoint_info(h, C.byref(step), C.byref(seed), C.byref(ng), C.byref(nr)))
        snap = Snapshot(step.value, seed.value)
        for i in range(ng.value):
            name = C.c_char_p()
            s, sid, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
            _lib.check(L.sw_checkpoint_rng(h, i, C.byref(name), C.byref(s), C.byref(sid), C.byref(c)))
            snap.rngs.append((name.value.decode(), s.value, sid.value, c.value))
        for i in range(nr.value):
            name = C.c_char_p()
            rank = C.c_uint32()
            dims = C.POINTER(C.c_int64)()
            data = C.POINTER(C.c_float)()
            n = C.c_int64()
            _lib.check(L.sw_checkpoint_record(h, i, C.byref(name), C.byref(rank), C.byref(dims), C.byref(data),
                                              C.byref(n)))
            shape = tuple(dims[k] for k in range(rank.value))
            arr = np.ctypeslib.as_array(data, shape=(n.value,)).copy().reshape(shape) if n.value else \
                np.zeros(shape, np.float32)
            snap.records.append((name.value.decode(), arr))
        return snap
    finally:
        L.sw_checkpoint_free(h)


def write(path: str, snap: Snapshot) -> None:
    L = _declare()
    ng, nr = len(snap.rngs), len(snap.records)
    g_names = (C.c_char_p * max(ng, 1))(*[g[0].encode() for g in snap.rngs])
    g_seed = (C.c_uint64 * max(ng, 1))(*[g[1] for g in snap.rngs])
    g_id = (C.c_uint64 * max(ng, 1))(*[g[2] for g in snap.rngs])
    g_ctr = (C.c_uint64 * max(ng, 1))(*[g[3] for g in snap.rngs])
    arrays = [np.array(a, dtype=np.float32, order="C") for _, a in snap.records]  # keeps 0-d
    dims = [np.array(a.shape, dtype=np.int64) for a in arrays]
    r_names = (C.c_char_p * max(nr, 1))(*[n.encode() for n, _ in snap.records])
    r_rank = (C.c_uint32 * max(nr, 1))(*[a.ndim for a in arrays])
    r_dims = (C.POINTER(C.c_int64) * max(nr, 1))(*[d.ctypes.data_as(C.POINTER(C.c_int64)) for d in dims])
    r_data = (C.POINTER(C.c_float) * max(nr, 1))(*[a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrays])
    _lib.check(L.sw_checkpoint_write(path.encode(), snap.step, snap.seed, ng, g_names, g_seed, g_id, g_ctr, nr,
                                     r_names, r_rank, r_dims, r_data))
