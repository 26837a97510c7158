"""Python face of the B200 executor (C ABI: sw_mesh_* / sw_model_*).

Mirrors the reference's runtime surface for the hot path:
  build_mesh (mesh.hpp:47-52)                      -> Mesh
  shard_params / replica_param_views (train_state.hpp:50-110) + the traced transformer_loss
  program (model.hpp:144-152)                      -> Model
  spmd_forward_backward (spmd.hpp:782-814)         -> Model.forward_backward
  scale_grads / dp_sync_grads / adamw_step (train_state.hpp:146-220)
                                                   -> Model.scale_grads / dp_sync / adamw_step
  gather_params (train_state.hpp:78-93)            -> Model.get_param / get_grad / get_adam
There is no CPU path: every call runs on the GPU through libshardweave_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib, rules


def _declare():
    L = _lib.lib()
    if getattr(L, "_engine_declared", False):
        return L
    vp = C.c_void_p
    L.sw_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
    L.sw_mesh_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8),
                                 C.c_int, C.POINTER(vp)]
    L.sw_mesh_comm_report.argtypes = [vp, C.POINTER(vp)]
    L.sw_mesh_reset_comm_report.argtypes = [vp]
    L.sw_mesh_free.argtypes = [vp]
    L.sw_mesh_free.restype = None
    L.sw_model_create.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.POINTER(vp)]
    L.sw_model_create_inference.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.POINTER(vp)]
    L.sw_model_free.argtypes = [vp]
    L.sw_model_free.restype = None
    L.sw_model_init_params.argtypes = [vp, C.c_uint64, C.c_char_p]
    L.sw_model_set_param.argtypes = [vp, C.c_char_p, vp, C.c_int64]
    L.sw_model_get_tensor.argtypes = [vp, C.c_char_p, C.c_int, vp, C.c_int64]
    L.sw_model_stage_batch.argtypes = [vp, vp, vp, vp]
    L.sw_model_forward_backward.argtypes = [vp, C.c_int]
    L.sw_model_scale_grads.argtypes = [vp, C.c_double]
    L.sw_model_dp_sync.argtypes = [vp]
    L.sw_model_adamw_step.argtypes = [vp, C.POINTER(AdamWConfigC), C.c_int]
    L.sw_model_train_step.argtypes = [vp, C.POINTER(AdamWConfigC)]
    L.sw_model_last_loss.argtypes = [vp, C.POINTER(C.c_double)]
    L.sw_model_forward_logits.argtypes = [vp, vp]
    L.sw_model_stream.argtypes = [vp, C.POINTER(vp)]
    L.sw_model_launch_count.argtypes = [vp, C.POINTER(C.c_int64)]
    L.sw_model_device_bytes.argtypes = [vp, C.POINTER(C.c_int64)]
    L.sw_model_set_profiling.argtypes = [vp, C.c_int]
    L.sw_model_read_profile.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_int64)]
    u64p = C.POINTER(C.c_uint64)
    L.sw_model_save_checkpoint.argtypes = [vp, C.c_char_p, C.c_uint32, C.POINTER(C.c_char_p), u64p, u64p, u64p]
    L.sw_model_load_checkpoint.argtypes = [vp, C.c_char_p, C.POINTER(C.c_uint32)]
    L.sw_model_checkpoint_rng.argtypes = [vp, C.c_uint32, C.c_char_p, C.c_uint64, u64p, u64p, u64p]
    L.sw_model_state_info.argtypes = [vp, u64p, u64p]
    L.sw_model_generate.argtypes = [vp, vp, C.c_int, C.c_int, vp]
    L.sw_t5_create.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.sw_t5_free.argtypes = [vp]
    L.sw_t5_free.restype = None
    L.sw_t5_init_params.argtypes = [vp, C.c_uint64, C.c_char_p]
    L.sw_t5_set_tensor.argtypes = [vp, C.c_char_p, C.c_int, vp, C.c_int64]
    L.sw_t5_get_tensor.argtypes = [vp, C.c_char_p, C.c_int, vp, C.c_int64]
    L.sw_t5_stage_batch.argtypes = [vp, vp, vp, vp, vp]
    L.sw_t5_forward_backward.argtypes = [vp]
    L.sw_t5_forward_logits.argtypes = [vp, vp]
    L.sw_t5_adamw_step.argtypes = [vp, C.POINTER(AdamWConfigC)]
    L.sw_t5_train_step.argtypes = [vp, C.POINTER(AdamWConfigC)]
    L.sw_t5_last_loss.argtypes = [vp, C.POINTER(C.c_double)]
    L.sw_t5_stream.argtypes = [vp, C.POINTER(vp)]
    L.sw_t5_set_profiling.argtypes = [vp, C.c_int]
    L.sw_t5_read_profile.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.sw_t5_launch_count.argtypes = [vp, C.POINTER(C.c_int64)]
    L.sw_t5_device_bytes.argtypes = [vp, C.POINTER(C.c_int64)]
    for fn in ("sw_t5_create", "sw_t5_init_params", "sw_t5_set_tensor", "sw_t5_get_tensor", "sw_t5_stage_batch",
               "sw_t5_forward_backward", "sw_t5_forward_logits", "sw_t5_adamw_step", "sw_t5_train_step",
               "sw_t5_last_loss", "sw_t5_stream", "sw_t5_set_profiling", "sw_t5_read_profile",
               "sw_t5_launch_count", "sw_t5_device_bytes"):
        getattr(L, fn).restype = C.c_int
    for fn in ("sw_nccl_unique_id", "sw_mesh_create", "sw_mesh_comm_report",
               "sw_mesh_reset_comm_report", "sw_model_create", "sw_model_create_inference", "sw_model_init_params",
               "sw_model_set_param", "sw_model_get_tensor", "sw_model_stage_batch",
               "sw_model_forward_backward", "sw_model_scale_grads", "sw_model_dp_sync",
               "sw_model_adamw_step", "sw_model_train_step", "sw_model_last_loss",
               "sw_model_forward_logits", "sw_model_stream", "sw_model_launch_count",
               "sw_model_device_bytes", "sw_model_set_profiling", "sw_model_read_profile",
               "sw_model_save_checkpoint", "sw_model_load_checkpoint", "sw_model_checkpoint_rng",
               "sw_model_state_info", "sw_model_generate"):
        getattr(L, fn).restype = C.c_int
    L._engine_declared = True
    return L


class AdamWConfigC(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double)]


@dataclass
class AdamWConfig:
    """AdamWConfig (train_state.hpp:172-178)."""
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0

    def c(self) -> AdamWConfigC:
        return AdamWConfigC(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay)


def nccl_unique_id() -> bytes:
    L = _declare()
    buf = (C.c_uint8 * 128)()
    _lib.check(L.sw_nccl_unique_id(buf))
    return bytes(buf)


class Mesh:
    """dp x mp device mesh. world == 1: the whole mesh is emulated in this process on one GPU;
    world == dp*mp: one device per process, NCCL communicators per mp / dp group."""

    def __init__(self, dp: int, mp: int, n_hosts: int = 1, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, cuda_device: int = 0):
        L = _declare()
        self.dp, self.mp, self.n_hosts, self.rank, self.world = dp, mp, n_hosts, rank, world
        h = C.c_void_p()
        idp = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        _lib.check(L.sw_mesh_create(dp, mp, n_hosts, rank, world, idp, cuda_device, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def comm_report(self) -> str:
        s = C.c_void_p()
        _lib.check(_declare().sw_mesh_comm_report(self._h, C.byref(s)))
        return _lib.take_string(s)

    def reset_comm_report(self):
        _lib.check(_declare().sw_mesh_reset_comm_report(self._h))

    def close(self):
        if getattr(self, "_h", None):
            _declare().sw_mesh_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter teardown: this module's globals are already cleared
            pass


def build_mesh(dp_size: int, mp_size: int, n_hosts: int = 1) -> Mesh:
    return Mesh(dp_size, mp_size, n_hosts)


class Model:
    """The traced transformer_loss program lowered onto a mesh with a sharding plan, plus its
    sharded train state (params, grads, AdamW moments) in HBM.

    inference=True builds the Predictor-only variant (sw_model_create_inference): bf16 weight
    shards + K/V cache, no gradients or optimizer state; the training methods raise ConfigError."""

    def __init__(self, spec: rules.ModelSpec, plan: rules.Plan, mesh: Mesh, batch: int, seq_len: int,
                 inference: bool = False):
        L = _declare()
        self.spec, self.plan, self.mesh = spec, plan, mesh
        self.batch, self.seq_len = batch, seq_len
        self.inference = inference
        self.shapes = dict(rules.transformer_param_shapes(spec))
        h = C.c_void_p()
        create = L.sw_model_create_inference if inference else L.sw_model_create
        _lib.check(create(spec.handle, plan.handle, mesh.handle, batch, seq_len, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _declare().sw_model_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter teardown: this module's globals are already cleared
            pass

    # ---- params ----
    def init_params(self, seed: int = 42, stream: str = "model-init"):
        _lib.check(_declare().sw_model_init_params(self._h, seed, stream.encode()))

    def set_param(self, name: str, value: np.ndarray):
        a = np.ascontiguousarray(value, dtype=np.float32)
        _lib.check(_declare().sw_model_set_param(self._h, name.encode(), a.ctypes.data, a.size))

    def _get(self, name: str, which: int) -> np.ndarray:
        shape = self.shapes[name]
        out = np.empty(shape, np.float32)
        _lib.check(_declare().sw_model_get_tensor(self._h, name.encode(), which, out.ctypes.data, out.size))
        return out

    def get_param(self, name):
        return self._get(name, 0)

    def get_grad(self, name):
        return self._get(name, 1)

    def get_adam(self, name):
        return self._get(name, 2), self._get(name, 3)

    # ---- step ----
    def stage_batch(self, tokens, targets, weights=None):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        y = np.ascontiguousarray(targets, dtype=np.int32)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
        self._staged = (t, y, w)  # keep host buffers alive until the copies are done
        _lib.check(_declare().sw_model_stage_batch(self._h, t.ctypes.data, y.ctypes.data,
                                                   None if w is None else w.ctypes.data))

    def forward_backward(self, accumulate: bool = False):
        _lib.check(_declare().sw_model_forward_backward(self._h, int(accumulate)))

    def scale_grads(self, factor: float):
        _lib.check(_declare().sw_model_scale_grads(self._h, factor))

    def dp_sync(self):
        _lib.check(_declare().sw_model_dp_sync(self._h))

    def adamw_step(self, cfg: AdamWConfig, check_finite: bool = True):
        c = cfg.c()
        _lib.check(_declare().sw_model_adamw_step(self._h, C.byref(c), int(check_finite)))

    def train_step(self, cfg: AdamWConfig):
        c = cfg.c()
        _lib.check(_declare().sw_model_train_step(self._h, C.byref(c)))

    def loss(self) -> float:
        x = C.c_double()
        _lib.check(_declare().sw_model_last_loss(self._h, C.byref(x)))
        return x.value

    def forward_logits(self) -> np.ndarray:
        rows = self.batch * (self.mesh.dp if self.mesh.world == 1 else 1)
        out = np.empty((rows, self.seq_len, self.spec.vocab_size), np.float32)
        _lib.check(_declare().sw_model_forward_logits(self._h, out.ctypes.data))
        return out

    def stream(self) -> int:
        s = C.c_void_p()
        _lib.check(_declare().sw_model_stream(self._h, C.byref(s)))
        return s.value or 0

    def launch_count(self) -> int:
        x = C.c_int64()
        _lib.check(_declare().sw_model_launch_count(self._h, C.byref(x)))
        return x.value

    PROFILE_CATEGORIES = ("gemm", "attn_fwd", "attn_bwd", "layernorm", "xent", "adamw", "comm", "other")

    def set_profiling(self, on: bool):
        _lib.check(_declare().sw_model_set_profiling(self._h, int(on)))

    def read_profile(self) -> dict:
        ms = (C.c_double * 8)()
        work = (C.c_double * 8)()
        cnt = (C.c_int64 * 8)()
        _lib.check(_declare().sw_model_read_profile(self._h, ms, work, cnt))
        return {c: {"ms": ms[i], "work": work[i], "launches": cnt[i]}
                for i, c in enumerate(self.PROFILE_CATEGORIES)}

    def device_bytes(self) -> int:
        x = C.c_int64()
        _lib.check(_declare().sw_model_device_bytes(self._h, C.byref(x)))
        return x.value

    # -- SWCK snapshots (checkpoint.hpp:193-298) ------------------------------------------------
    def save_checkpoint(self, path: str, rngs=()):
        """save_checkpoint(path, state, mesh, rngs): rngs is a sequence of
        (name, seed, stream_id, counter). Under NCCL every rank calls it; rank 0 writes."""
        rngs = list(rngs)
        n = len(rngs)
        names = (C.c_char_p * max(n, 1))(*[r[0].encode() for r in rngs])
        seeds = (C.c_uint64 * max(n, 1))(*[r[1] for r in rngs])
        ids = (C.c_uint64 * max(n, 1))(*[r[2] for r in rngs])
        ctrs = (C.c_uint64 * max(n, 1))(*[r[3] for r in rngs])
        _lib.check(_declare().sw_model_save_checkpoint(self._h, path.encode(), n, names, seeds, ids, ctrs))

    def load_checkpoint(self, path: str):
        """load_checkpoint re-cut onto this model's plan and mesh; returns the stored RNG streams
        as [(name, seed, stream_id, counter)]."""
        L = _declare()
        n = C.c_uint32()
        _lib.check(L.sw_model_load_checkpoint(self._h, path.encode(), C.byref(n)))
        out = []
        for i in range(n.value):
            buf = C.create_string_buffer(4096)
            s, sid, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
            _lib.check(L.sw_model_checkpoint_rng(self._h, i, buf, 4096, C.byref(s), C.byref(sid), C.byref(c)))
            out.append((buf.value.decode(), s.value, sid.value, c.value))
        return out

    def state_info(self):
        """(optimizer step, state seed) of the TrainState (train_state.hpp:24-27)."""
        step, seed = C.c_uint64(), C.c_uint64()
        _lib.check(_declare().sw_model_state_info(self._h, C.byref(step), C.byref(seed)))
        return step.value, seed.value

    # -- greedy generation (Predictor loop, cli.cpp:425-447) ------------------------------------
    def generate(self, prompts, n_new: int) -> np.ndarray:
        """prompts [batch, P] token ids -> [batch, n_new] greedy continuations (KV-cached while the
        context fits seq_len, sliding window after, like the reference)."""
        p = np.ascontiguousarray(prompts, dtype=np.int32)
        if p.ndim != 2:
            raise ValueError("prompts must be [batch, P]")
        out = np.empty((p.shape[0], n_new), np.int32)
        _lib.check(_declare().sw_model_generate(self._h, p.ctypes.data, p.shape[1], n_new, out.ctypes.data))
        return out


class T5Model:
    """Extension (BASELINE cfg4): the T5 encoder-decoder step on the mesh with
    the plan the reference rules give its tree (oracle/t5_ref.py is the math). dp = 1."""

    PROFILE_CATEGORIES = Model.PROFILE_CATEGORIES

    def __init__(self, spec: rules.ModelSpec, plan: rules.Plan, mesh: Mesh, batch: int, enc_len: int, dec_len: int):
        L = _declare()
        self.spec, self.plan, self.mesh = spec, plan, mesh
        self.batch, self.enc_len, self.dec_len = batch, enc_len, dec_len
        self.shapes = dict(rules.transformer_param_shapes(spec))
        h = C.c_void_p()
        _lib.check(L.sw_t5_create(spec.handle, plan.handle, mesh.handle, batch, enc_len, dec_len, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _declare().sw_t5_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter teardown: this module's globals are already cleared
            pass

    def init_params(self, seed: int = 42, stream: str = "model-init"):
        _lib.check(_declare().sw_t5_init_params(self._h, seed, stream.encode()))

    def set_param(self, name: str, value: np.ndarray, which: int = 0):
        a = np.ascontiguousarray(value, dtype=np.float32)
        _lib.check(_declare().sw_t5_set_tensor(self._h, name.encode(), which, a.ctypes.data, a.size))

    def _get(self, name: str, which: int) -> np.ndarray:
        out = np.empty(self.shapes[name], np.float32)
        _lib.check(_declare().sw_t5_get_tensor(self._h, name.encode(), which, out.ctypes.data, out.size))
        return out

    def get_param(self, name):
        return self._get(name, 0)

    def get_grad(self, name):
        return self._get(name, 1)

    def get_adam(self, name):
        return self._get(name, 2), self._get(name, 3)

    def stage_batch(self, enc_tokens, dec_tokens, targets, weights=None):
        e = np.ascontiguousarray(enc_tokens, dtype=np.int32)
        t = np.ascontiguousarray(dec_tokens, dtype=np.int32)
        y = np.ascontiguousarray(targets, dtype=np.int32)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
        self._staged = (e, t, y, w)
        _lib.check(_declare().sw_t5_stage_batch(self._h, e.ctypes.data, t.ctypes.data, y.ctypes.data,
                                                None if w is None else w.ctypes.data))

    def forward_backward(self):
        _lib.check(_declare().sw_t5_forward_backward(self._h))

    def forward_logits(self) -> np.ndarray:
        out = np.empty((self.batch, self.dec_len, self.spec.vocab_size), np.float32)
        _lib.check(_declare().sw_t5_forward_logits(self._h, out.ctypes.data))
        return out

    def adamw_step(self, cfg: AdamWConfig):
        c = cfg.c()
        _lib.check(_declare().sw_t5_adamw_step(self._h, C.byref(c)))

    def train_step(self, cfg: AdamWConfig):
        c = cfg.c()
        _lib.check(_declare().sw_t5_train_step(self._h, C.byref(c)))

    def loss(self) -> float:
        x = C.c_double()
        _lib.check(_declare().sw_t5_last_loss(self._h, C.byref(x)))
        return x.value

    def stream(self) -> int:
        s = C.c_void_p()
        _lib.check(_declare().sw_t5_stream(self._h, C.byref(s)))
        return s.value or 0

    def launch_count(self) -> int:
        x = C.c_int64()
        _lib.check(_declare().sw_t5_launch_count(self._h, C.byref(x)))
        return x.value

    def set_profiling(self, on: bool):
        _lib.check(_declare().sw_t5_set_profiling(self._h, int(on)))

    def read_profile(self) -> dict:
        ms, work, cnt = (C.c_double * 8)(), (C.c_double * 8)(), (C.c_int64 * 8)()
        _lib.check(_declare().sw_t5_read_profile(self._h, ms, work, cnt))
        return {c: {"ms": ms[i], "work": work[i], "launches": cnt[i]} for i, c in enumerate(self.PROFILE_CATEGORIES)}

    def device_bytes(self) -> int:
        x = C.c_int64()
        _lib.check(_declare().sw_t5_device_bytes(self._h, C.byref(x)))
        return x.value
