"""ORACLE (test infrastructure): numpy restatement of RngStream (rng.hpp:15-91) and of
init_transformer_params (model.hpp:49-70).

The stream is counter-based: draw(c) = mix(mix(seed ^ mix(stream_id)) + c) with splitmix64's
finaliser as `mix` (rng.hpp:76-85), so any range of draws is computed without replaying the
stream. next_normal consumes two draws (Box-Muller, rng.hpp:36-43); next_below is u64 % n.
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15


def mix_int(z: int) -> int:
    z = (z + GOLDEN_GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(GOLDEN_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for c in s.encode():
        h ^= c
        h = (h * 0x100000001B3) & M64
    return h


class RngStream:
    def __init__(self, seed: int, name_or_id, counter: int = 0):
        self.seed = seed & M64
        self.stream_id = fnv1a(name_or_id) if isinstance(name_or_id, str) else name_or_id & M64
        self.counter = counter

    def _key(self) -> int:
        return mix_int(self.seed ^ mix_int(self.stream_id))

    def draws(self, n: int) -> np.ndarray:
        """The next n u64 draws (advances the counter)."""
        c = np.arange(self.counter, self.counter + n, dtype=np.uint64)
        with np.errstate(over="ignore"):
            out = mix_np(np.uint64(self._key()) + c)
        self.counter += n
        return out

    def uniforms(self, n: int) -> np.ndarray:
        return (self.draws(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def normals(self, n: int) -> np.ndarray:
        u = self.uniforms(2 * n)
        u1, u2 = u[0::2].copy(), u[1::2]
        u1[u1 <= 0.0] = 2.0 ** -53
        r = np.sqrt(-2.0 * np.log(u1))
        return r * np.cos(2.0 * 3.14159265358979323846 * u2)

    def below(self, n: int, bound: int) -> np.ndarray:
        return (self.draws(n) % np.uint64(bound)).astype(np.int64)

    def permutation(self, n: int) -> np.ndarray:
        """Fisher-Yates (rng.hpp:57-65)."""
        perm = list(range(n))
        for i in range(n, 1, -1):
            j = int(self.draws(1)[0] % np.uint64(i))
            perm[i - 1], perm[j] = perm[j], perm[i - 1]
        return np.array(perm)

    def child(self, index_or_name) -> "RngStream":
        seed = mix_int(self.seed ^ self.stream_id)
        if isinstance(index_or_name, str):
            return RngStream(seed, index_or_name)
        return RngStream(seed, mix_int((index_or_name + GOLDEN_GAMMA) & M64), 0)


def normals_exact(rng: RngStream, n: int) -> np.ndarray:
    """Same as rng.normals but with libm log/cos per element (bit-for-bit with std::log/cos)."""
    u = rng.uniforms(2 * n)
    out = np.empty(n)
    for i in range(n):
        u1 = u[2 * i] if u[2 * i] > 0.0 else 2.0 ** -53
        out[i] = math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * 3.14159265358979323846 * u[2 * i + 1])
    return out


def t5_param_shapes(spec: dict):
    """Extension: the T5 encoder-decoder tree, named with the reference's
    attn / cross_attn / mlp scopes (roles.cpp:36-43) so its rule engine plans it. Per block:
    ln1, attn q/k/v [H*d_kv, d], o [d, H*d_kv], (block 0 only) attn/rel_bias [buckets, H],
    decoder ln_x + cross_attn, ln2, mlp fc1 [d_ff, d] / fc2 [d, d_ff]; no biases; RMSNorm scales."""
    d, V, H = spec["d_model"], spec["vocab_size"], spec["n_heads"]
    inner = H * spec["d_kv"]
    out = [("embed/tok/kernel", (V, d))]

    def attn(b, scope):
        return [(b + f"{scope}/{p}/kernel", (inner, d)) for p in "qkv"] + [(b + f"{scope}/o/kernel", (d, inner))]

    for st, layers, dec in (("enc", spec["n_layers"], False), ("dec", spec["n_dec_layers"], True)):
        for l in range(layers):
            b = f"{st}/block_{l}/"
            out += [(b + "ln1/scale", (d,))] + attn(b, "attn")
            if l == 0:
                out.append((b + "attn/rel_bias/kernel", (spec.get("rel_buckets", 32), H)))
            if dec:
                out += [(b + "ln_x/scale", (d,))] + attn(b, "cross_attn")
            out += [(b + "ln2/scale", (d,)), (b + "mlp/fc1/kernel", (spec["d_ff"], d)),
                    (b + "mlp/fc2/kernel", (d, spec["d_ff"]))]
        out.append((f"{st}/final_ln/scale", (d,)))
    out.append(("lm_head/kernel", (V, d)))
    return out


def transformer_param_shapes(spec: dict):
    """model.hpp:17-43 (tree order); mlp = swiglu / norm = rmsnorm extension leaves."""
    if spec.get("arch", "decoder") == "t5":
        return t5_param_shapes(spec)
    d, V = spec["d_model"], spec["vocab_size"]
    rms = spec.get("norm", "layernorm") == "rmsnorm"
    swiglu = spec.get("mlp", "gelu") == "swiglu"

    def norm(p):
        return [(p + "/scale", (d,))] + ([] if rms else [(p + "/bias", (d,))])

    out = [("embed/tok/kernel", (V, d)), ("embed/pos/kernel", (spec["max_seq_len"], d))]
    for l in range(spec["n_layers"]):
        b = f"block_{l}/"
        out += norm(b + "ln1")
        for p in "qkvo":
            out += [(b + f"attn/{p}/kernel", (d, d)), (b + f"attn/{p}/bias", (d,))]
        out += norm(b + "ln2")
        if swiglu:
            out += [(b + "mlp/fc1/gate/kernel", (spec["d_ff"], d)), (b + "mlp/fc1/kernel", (spec["d_ff"], d)),
                    (b + "mlp/fc2/kernel", (d, spec["d_ff"]))]
        else:
            out += [(b + "mlp/fc1/kernel", (spec["d_ff"], d)), (b + "mlp/fc1/bias", (spec["d_ff"],)),
                    (b + "mlp/fc2/kernel", (d, spec["d_ff"])), (b + "mlp/fc2/bias", (d,))]
    out += norm("final_ln")
    if not spec.get("tie_embeddings", False):
        out.append(("lm_head/kernel", (V, d)))
    return out


def init_transformer_params(spec: dict, seed: int = 42, name: str = "model-init",
                            dtype=np.float64, exact: bool = False) -> dict:
    """model.hpp:49-70: kernels N(0, 1/fan_in), embeddings N(0, 0.02^2), biases 0, scales 1,
    all drawn from one stream in tree order."""
    rng = RngStream(seed, name)
    params = {}
    for pname, shape in transformer_param_shapes(spec):
        leaf = pname.rsplit("/", 1)[1]
        n = int(np.prod(shape))
        if leaf == "bias":
            params[pname] = np.zeros(shape, dtype)
        elif leaf == "scale":
            params[pname] = np.ones(shape, dtype)
        else:
            scale = 0.02 if pname.startswith("embed/") else 1.0 / math.sqrt(float(shape[1]))
            z = normals_exact(rng, n) if exact else rng.normals(n)
            params[pname] = (z * scale).astype(dtype).reshape(shape)
    return params


def audit_batch(seed: int, step: int, batch: int, seq: int, vocab: int):
    """cli.cpp:211-228: tokens then targets from RngStream(seed,"audit-batch").child(step)."""
    rng = RngStream(seed, "audit-batch").child(step)
    tokens = rng.below(batch * seq, vocab).reshape(batch, seq)
    targets = rng.below(batch * seq, vocab).reshape(batch, seq)
    return tokens, targets, np.ones((batch, seq))
