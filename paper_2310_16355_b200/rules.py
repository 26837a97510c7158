"""Python face of the host rule engine (C ABI: sw_model_spec_* / sw_infer_roles / sw_plan_*).

Names, argument meaning and error behaviour mirror the reference's C++ API:
parse_model_spec (model_spec.hpp:30-34), transformer_param_shapes (model.hpp:17-43),
infer_roles (roles.hpp:58-64), derive_plan (plan.hpp:35-47), validate_plan / serialize_plan /
parse_plan (plan.hpp:52-59), local_shape / shard ranges (sharded_tensor.hpp:14-74) and
expected_state_elements (train_state.hpp:236-245). Errors raise ConfigError / PartitionError
with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _lib
from ._lib import ConfigError, PartitionError  # noqa: F401  (re-exported)

ShapeMap = list  # [(name, [dims...]), ...] in tree order


def _declare():
    L = _lib.lib()
    if getattr(L, "_rules_declared", False):
        return L
    cp = C.c_char_p
    cpp = C.POINTER(C.c_char_p)
    vp = C.c_void_p
    out_str = C.POINTER(C.c_void_p)
    L.sw_model_spec_parse.argtypes = [cp, C.POINTER(vp)]
    L.sw_model_spec_dims.argtypes = [vp, C.POINTER(C.c_int64)]
    L.sw_model_spec_overrides.argtypes = [vp, out_str]
    L.sw_model_spec_variant.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.sw_model_spec_variant.restype = C.c_int
    L.sw_model_spec_t5.argtypes = [vp, C.POINTER(C.c_int64)]
    L.sw_model_spec_t5.restype = C.c_int
    L.sw_t5_rel_buckets.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, vp]
    L.sw_t5_rel_buckets.restype = C.c_int
    L.sw_model_spec_free.argtypes = [vp]
    L.sw_model_spec_free.restype = None
    L.sw_transformer_param_shapes.argtypes = [vp, out_str]
    shp = [cpp, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_size_t]
    L.sw_infer_roles.argtypes = shp + [cpp, cpp, C.c_size_t, out_str, out_str]
    L.sw_plan_derive.argtypes = shp + [cpp, cpp, C.c_size_t, C.c_int, C.POINTER(vp)]
    L.sw_plan_parse.argtypes = [cp, C.c_int, C.POINTER(vp)]
    L.sw_plan_serialize.argtypes = [vp, out_str]
    L.sw_plan_validate.argtypes = [vp] + shp + [out_str]
    L.sw_plan_warnings.argtypes = [vp, out_str]
    L.sw_plan_size.argtypes = [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_int)]
    L.sw_plan_entry.argtypes = [vp, C.c_size_t, C.POINTER(C.c_char_p), C.POINTER(C.c_int),
                                C.POINTER(C.c_int64)]
    L.sw_plan_free.argtypes = [vp]
    L.sw_plan_free.restype = None
    L.sw_shard_range.argtypes = [C.POINTER(C.c_int64), C.c_int32, C.c_int, C.c_int64, C.c_int,
                                 C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64)]
    L.sw_expected_state_elements.argtypes = [vp] + shp + [C.c_int, C.POINTER(C.c_int64)]
    for fn in ("sw_model_spec_parse", "sw_model_spec_dims", "sw_model_spec_overrides",
               "sw_transformer_param_shapes", "sw_infer_roles", "sw_plan_derive", "sw_plan_parse",
               "sw_plan_serialize", "sw_plan_validate", "sw_plan_warnings", "sw_plan_size",
               "sw_plan_entry", "sw_shard_range", "sw_expected_state_elements"):
        getattr(L, fn).restype = C.c_int
    L._rules_declared = True
    return L


def _take(ptr: C.c_void_p) -> str:
    return _lib.take_string(ptr)


def _encode_shapes(shapes):
    n = len(shapes)
    names = (C.c_char_p * max(n, 1))(*[s[0].encode() for s in shapes])
    ranks = (C.c_int32 * max(n, 1))(*[len(s[1]) for s in shapes])
    flat = [int(d) for s in shapes for d in s[1]]
    dims = (C.c_int64 * max(len(flat), 1))(*flat)
    return names, ranks, dims, n


def _encode_overrides(overrides):
    n = len(overrides)
    pats = (C.c_char_p * max(n, 1))(*[o[0].encode() for o in overrides])
    roles = (C.c_char_p * max(n, 1))(*[o[1].encode() for o in overrides])
    return pats, roles, n


@dataclass
class ModelSpec:
    vocab_size: int
    n_layers: int
    d_model: int
    n_heads: int
    d_ff: int
    max_seq_len: int
    tie_embeddings: bool = False
    overrides: list = field(default_factory=list)  # [(pattern, role_name)]
    mlp: str = "gelu"          # extension key: gelu | swiglu
    norm: str = "layernorm"    # extension key: layernorm | rmsnorm
    # extension: arch = t5 encoder-decoder
    arch: str = "decoder"
    n_dec_layers: int = 0
    d_kv: int = 0
    rel_buckets: int = 32
    rel_max_distance: int = 128
    _handle: object = field(default=None, repr=False, compare=False)

    def __del__(self):
        if self._handle:
            _lib.lib().sw_model_spec_free(self._handle)
            self._handle = None

    @property
    def handle(self):
        return self._handle

    def text(self) -> str:
        lines = [f"vocab_size = {self.vocab_size}", f"n_layers = {self.n_layers}",
                 f"d_model = {self.d_model}", f"n_heads = {self.n_heads}", f"d_ff = {self.d_ff}",
                 f"max_seq_len = {self.max_seq_len}",
                 f"tie_embeddings = {'true' if self.tie_embeddings else 'false'}"]
        if self.mlp != "gelu":
            lines.append(f"mlp = {self.mlp}")
        if self.arch == "t5":
            lines += ["arch = t5", f"n_dec_layers = {self.n_dec_layers}", f"d_kv = {self.d_kv}",
                      f"rel_buckets = {self.rel_buckets}", f"rel_max_distance = {self.rel_max_distance}"]
        elif self.norm != "layernorm":
            lines.append(f"norm = {self.norm}")
        lines += [f"role {p} = {r}" for p, r in self.overrides]
        return "\n".join(lines) + "\n"


def parse_model_spec(text: str) -> ModelSpec:
    L = _declare()
    h = C.c_void_p()
    _lib.check(L.sw_model_spec_parse(text.encode(), C.byref(h)))
    dims = (C.c_int64 * 7)()
    _lib.check(L.sw_model_spec_dims(h, dims))
    s = C.c_void_p()
    _lib.check(L.sw_model_spec_overrides(h, C.byref(s)))
    ovr = [tuple(ln.split("\t")) for ln in _take(s).splitlines() if ln]
    sg, rn = C.c_int(), C.c_int()
    _lib.check(L.sw_model_spec_variant(h, C.byref(sg), C.byref(rn)))
    t5 = (C.c_int64 * 5)()
    _lib.check(L.sw_model_spec_t5(h, t5))
    return ModelSpec(int(dims[0]), int(dims[1]), int(dims[2]), int(dims[3]), int(dims[4]),
                     int(dims[5]), bool(dims[6]), ovr, "swiglu" if sg.value else "gelu",
                     "rmsnorm" if rn.value else "layernorm", "t5" if t5[0] else "decoder", int(t5[1]), int(t5[2]),
                     int(t5[3]), int(t5[4]), h)


def t5_rel_buckets(tq: int, tk: int, bidirectional: bool, num_buckets: int, max_distance: int):
    """Bucket ids [tq, tk] of the T5 relative-position bias (host rule engine, rules.h)."""
    import numpy as np

    out = np.zeros((tq, tk), np.int32)
    _lib.check(_declare().sw_t5_rel_buckets(tq, tk, int(bidirectional), num_buckets, max_distance,
                                            out.ctypes.data))
    return out


def read_model_spec(path: str) -> ModelSpec:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(3, f"model spec: cannot open '{path}'") from None
    return parse_model_spec(text)


def transformer_param_shapes(spec: ModelSpec) -> ShapeMap:
    L = _declare()
    s = C.c_void_p()
    _lib.check(L.sw_transformer_param_shapes(spec.handle, C.byref(s)))
    out = []
    for ln in _take(s).splitlines():
        name, dims = ln.split("\t")
        out.append((name, [int(x) for x in dims.split(",") if x]))
    return out


def infer_roles(shapes: ShapeMap, overrides=()):
    """Returns ([(name, role_name, sequence_index)], warnings)."""
    L = _declare()
    names, ranks, dims, n = _encode_shapes(shapes)
    pats, roles, no = _encode_overrides(list(overrides))
    r, w = C.c_void_p(), C.c_void_p()
    _lib.check(L.sw_infer_roles(names, ranks, dims, n, pats, roles, no, C.byref(r), C.byref(w)))
    out = []
    for ln in _take(r).splitlines():
        name, role, seq = ln.split("\t")
        out.append((name, role, int(seq)))
    warn = _take(w)
    return out, (warn.split("\n") if warn else [])


class Plan:
    """ShardingPlan (plan.hpp:20-31): ordered (name, partition) entries + warnings."""

    def __init__(self, handle):
        self._h = handle
        L = _declare()
        n, ns = C.c_size_t(), C.c_int()
        _lib.check(L.sw_plan_size(self._h, C.byref(n), C.byref(ns)))
        self.n_shards = ns.value
        self.entries = []
        for i in range(n.value):
            name, kind, dim = C.c_char_p(), C.c_int(), C.c_int64()
            _lib.check(L.sw_plan_entry(self._h, i, C.byref(name), C.byref(kind), C.byref(dim)))
            self.entries.append((name.value.decode(), f"split:{dim.value}" if kind.value else "replicated"))
        w = C.c_void_p()
        _lib.check(L.sw_plan_warnings(self._h, C.byref(w)))
        text = _take(w)
        self.warnings = text.split("\n") if text else []

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib().sw_plan_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def at(self, name: str) -> str:
        for n, p in self.entries:
            if n == name:
                return p
        raise ConfigError(3, f"ShardingPlan: no entry for parameter '{name}'")

    def serialize(self) -> str:
        L = _declare()
        s = C.c_void_p()
        _lib.check(L.sw_plan_serialize(self._h, C.byref(s)))
        return _take(s)


def derive_plan(shapes: ShapeMap, n_shards: int, overrides=()) -> Plan:
    L = _declare()
    names, ranks, dims, n = _encode_shapes(shapes)
    pats, roles, no = _encode_overrides(list(overrides))
    h = C.c_void_p()
    _lib.check(L.sw_plan_derive(names, ranks, dims, n, pats, roles, no, n_shards, C.byref(h)))
    return Plan(h)


def parse_plan(text: str, n_shards: int) -> Plan:
    L = _declare()
    h = C.c_void_p()
    _lib.check(L.sw_plan_parse(text.encode(), n_shards, C.byref(h)))
    return Plan(h)


def serialize_plan(plan: Plan) -> str:
    return plan.serialize()


def validate_plan(plan: Plan, shapes: ShapeMap) -> list:
    L = _declare()
    names, ranks, dims, n = _encode_shapes(shapes)
    s = C.c_void_p()
    _lib.check(L.sw_plan_validate(plan.handle, names, ranks, dims, n, C.byref(s)))
    text = _take(s)
    return text.split("\n") if text else []


def shard_range(global_dims, partition: str, n_shards: int, rank: int):
    """(local_dims, begin, end) along the split dim for `rank` (sharded_tensor.hpp:20-74)."""
    L = _declare()
    g = (C.c_int64 * max(len(global_dims), 1))(*global_dims)
    loc = (C.c_int64 * max(len(global_dims), 1))()
    kind, dim = (0, -1) if partition == "replicated" else (1, int(partition.split(":")[1]))
    b, e = C.c_int64(), C.c_int64()
    _lib.check(L.sw_shard_range(g, len(global_dims), kind, dim, n_shards, rank, loc, C.byref(b),
                                C.byref(e)))
    return [loc[i] for i in range(len(global_dims))], b.value, e.value


def expected_state_elements(plan: Plan, shapes: ShapeMap, mp_size: int) -> int:
    L = _declare()
    names, ranks, dims, n = _encode_shapes(shapes)
    out = C.c_int64()
    _lib.check(L.sw_expected_state_elements(plan.handle, names, ranks, dims, n, mp_size, C.byref(out)))
    return out.value
