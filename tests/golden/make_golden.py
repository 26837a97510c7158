"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
It builds oracle/_ref/sw_ref_driver (oracle/Makefile: the reference's own sources + our Eigen
shim + a CLI-free driver) and records:

  rules.json   rule-engine cases: role inference, derive_plan (+warnings / errors),
               validate_plan, parse_plan, model-spec parsing, expected_state_elements —
               the reference test cases of tests/test_plan.cpp, tests/test_model.cpp, every
               config spec in oracle/specs at n_shards 1/2/4/8, naming traps from SURVEY.md §8
               and a seeded random fuzz of parameter trees.
  mini_*.npz   full numeric trajectories (init params, logits, loss, grads, params after
               AdamW) of a small decoder, f64/f32, single-device and sharded.
  tiny_*.npz   checksums of the cfg1 (BASELINE configs[0]) trajectory.
"""
from __future__ import annotations

import json
import os
import random
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
ORACLE = os.path.join(ROOT, "oracle")
DRIVER = os.path.join(ORACLE, "_ref", "sw_ref_driver")
SPECS = os.path.join(ORACLE, "specs")


def build():
    subprocess.run(["make", "-C", ORACLE], check=True, stdout=subprocess.DEVNULL)


def run(args, tmp):
    r = subprocess.run([DRIVER] + args, capture_output=True, text=True, cwd=tmp)
    return r.stdout


def write(tmp, name, text):
    p = os.path.join(tmp, name)
    with open(p, "w") as f:
        f.write(text)
    return p


def shapes_tsv(shapes):
    return "".join(f"{n}\t{','.join(str(d) for d in s)}\n" for n, s in shapes)


CANONICAL = [
    ("block_0/attn/q/kernel", [64, 64]), ("block_0/attn/k/kernel", [64, 64]),
    ("block_0/attn/v/kernel", [64, 64]), ("block_0/attn/o/kernel", [64, 64]),
    ("block_0/attn/q/bias", [64]), ("block_0/ln1/scale", [64]), ("block_0/ln1/bias", [64]),
    ("block_0/mlp/fc1/kernel", [256, 64]), ("block_0/mlp/fc1/bias", [256]),
    ("block_0/mlp/fc2/kernel", [64, 256]), ("block_0/mlp/fc2/bias", [64]),
    ("embed/tok/kernel", [50, 64]),
]

FIXED_CASES = [
    # tests/test_plan.cpp
    ("canonical", CANONICAL, [], [1, 2, 4]),
    ("alternate_conventions", [
        ("layer_0/self_attn/q_proj/kernel", [32, 32]), ("layer_0/self_attn/out_proj/kernel", [32, 32]),
        ("layer_0/attention/qkv/kernel", [96, 32]), ("layer_0/ffn/dense1/kernel", [128, 32]),
        ("layer_0/ffn/dense2/kernel", [32, 128]), ("token_embedding/kernel", [100, 32]),
        ("final_norm/scale", [32])], [], [1, 2]),
    ("fc_restart_per_block", [
        ("block_0/mlp/fc1/kernel", [128, 32]), ("block_0/mlp/fc2/kernel", [32, 128]),
        ("block_1/mlp/fc1/kernel", [128, 32]), ("block_1/mlp/fc2/kernel", [32, 128])], [], [2]),
    ("unmatched_other", [("mystery/kernel", [16, 16])], [], [1, 2]),
    ("override_longest", [("block_0/mlp/fc1/kernel", [128, 32])],
     [("fc1", "other"), ("mlp/fc1", "attention_qkv")], [2]),
    ("override_conflict", [("block_0/mlp/fc1/kernel", [128, 32])],
     [("fc1", "other"), ("mlp", "attention_qkv")], [2]),
    ("indivisible", [("block_0/mlp/fc1/kernel", [10, 64]), ("block_0/mlp/fc2/kernel", [64, 12])], [], [4]),
    ("cannot_split", [("block_0/mlp/fc1/kernel", [4, 4]), ("block_0/mlp/fc2/kernel", [4, 4]),
                      ("block_0/ln1/scale", [4])], [], [4, 8, 0, -2]),
    ("serialize", [("block_0/attn/q/kernel", [64, 64]), ("block_0/attn/o/kernel", [64, 64]),
                   ("block_0/ln1/scale", [64])], [], [2]),
    # SURVEY.md §8 notes: naming traps and the SwiGLU naming of D3
    ("swiglu_gate_naming", [
        ("block_0/mlp/fc1/gate/kernel", [1024, 256]), ("block_0/mlp/fc1/kernel", [1024, 256]),
        ("block_0/mlp/fc2/kernel", [256, 1024])], [], [2, 4]),
    ("hf_swiglu_order", [
        ("layers_0/mlp/gate_proj/kernel", [1024, 256]), ("layers_0/mlp/up_proj/kernel", [1024, 256]),
        ("layers_0/mlp/down_proj/kernel", [256, 1024])], [], [2]),
    ("t5_hf_names", [
        ("encoder/block_0/layer_0/SelfAttention/q/kernel", [64, 64]),
        ("encoder/block_0/layer_0/SelfAttention/o/kernel", [64, 64]),
        ("encoder/block_0/layer_1/DenseReluDense/wi/kernel", [256, 64]),
        ("encoder/block_0/layer_1/DenseReluDense/wo/kernel", [64, 256]),
        ("decoder/block_0/layer_1/EncDecAttention/k/kernel", [64, 64]),
        ("decoder/block_0/cross_attn/k/kernel", [64, 64]),
        ("encoder/block_0/attn/relative_attention_bias/kernel", [32, 8])], [], [2]),
    ("opt_hf_names", [
        ("decoder/layers_0/self_attn/q_proj/kernel", [64, 64]),
        ("decoder/layers_0/self_attn/out_proj/kernel", [64, 64]),
        ("decoder/layers_0/fc1/kernel", [256, 64]), ("decoder/layers_0/fc2/kernel", [64, 256]),
        ("decoder/layers_0/self_attn_layer_norm/weight", [64]),
        ("decoder/embed_tokens/kernel", [1000, 64])], [], [2, 8]),
    ("fused_qkv", [("block_0/attn/qkv/kernel", [192, 64]), ("block_0/attn/o/kernel", [64, 64])], [], [2, 3]),
    ("lm_head_override", [("embed/tok/kernel", [32000, 64]), ("lm_head/kernel", [32000, 64])],
     [("lm_head/kernel", "fully_connected")], [8]),
    ("override_case_insensitive", [("Block_0/MLP/FC1/Kernel", [64, 32]), ("x/Attn/Q/w", [32, 32])],
     [("MLP/fc1", "attention_out")], [2]),
    ("empty_leaf_and_scalars", [("a//kernel", [8, 8]), ("scalar", []), ("b/ffn", [8, 8, 2]),
                                ("norm_x/v", [8]), ("c/beta", [8]), ("d/b", [8]), ("e/g", [8])], [], [1, 2]),
]

SEGMENTS = ["block_0", "block_1", "layer_2", "h", "attn", "Attention", "self_attn", "mha",
            "cross_attention", "self_attention", "q", "k", "v", "query", "key", "value", "qkv",
            "wq", "wk", "wv", "q_proj", "k_proj", "v_proj", "o", "out", "out_proj", "output",
            "o_proj", "wo", "mlp", "ffn", "fc1", "fc2", "fc", "dense", "dense_1", "DenseX",
            "embed", "embedding", "tok_embeddings", "ln1", "ln_f", "norm", "LayerNorm", "rms_norm",
            "kernel", "weight", "bias", "scale", "gamma", "beta", "g", "b", "w", "x", "proj",
            "up", "gate", "down", "lm_head", "router", "experts"]
ROLES = ["attention_qkv", "attention_out", "fully_connected", "embedding", "norm", "bias",
         "other"]


def fuzz_cases(n=160, seed=20231016):
    rng = random.Random(seed)
    cases = []
    for i in range(n):
        shapes, seen = [], set()
        for _ in range(rng.randint(1, 14)):
            depth = rng.randint(1, 5)
            name = "/".join(rng.choice(SEGMENTS) for _ in range(depth))
            if name in seen:
                continue
            seen.add(name)
            rank = rng.choice([1, 1, 2, 2, 2, 3])
            shapes.append((name, [rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 24, 64]) for _ in range(rank)]))
        ovr = []
        if rng.random() < 0.3:
            for _ in range(rng.randint(1, 2)):
                ovr.append((rng.choice(SEGMENTS), rng.choice(ROLES)))
        cases.append((f"fuzz_{i}", shapes, ovr, [rng.choice([1, 2, 3, 4, 8])]))
    return cases


VALIDATE_EDITS = [
    ("fc2_same_dim", {"block_0/mlp/fc2/kernel": "split:0"}, 2),
    ("dim_out_of_range", {"block_0/attn/q/bias": "split:2"}, 2),
    ("not_divisible", {}, 3),
    ("attention_wrong_dims", {"block_0/attn/q/kernel": "split:1", "block_0/attn/o/kernel": "split:0"}, 2),
    ("attention_replicated", {"block_0/attn/v/kernel": "replicated"}, 2),
    ("unknown_param", {"__extra__": "split:0"}, 2),
]

PARSE_TEXTS = [
    ("malformed_line", "a/kernel\tsplit:0\nb/kernel no tab here\n", 2),
    ("unknown_layout", "a/kernel\tdiagonal\n", 2),
    ("bad_dim", "a/kernel\tsplit:x\n", 2),
    ("negative_dim", "a/kernel\tsplit:-1\n", 2),
    ("zero_shards", "a/kernel\treplicated\n", 0),
    ("blank_lines", "\na/kernel\tsplit:1\n\nb\treplicated\n", 2),
    ("leading_tab", "\tsplit:0\n", 2),
]

SPEC_TEXTS = [
    ("ok_comments", "# c\nvocab_size = 10\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 16\n"
                    "max_seq_len = 4   # trailing\n\ntie_embeddings = yes\n"),
    ("missing_key", "vocab_size = 10\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 16\n"),
    ("duplicate_key", "vocab_size = 10\nvocab_size = 11\nn_layers = 1\nd_model = 8\nn_heads = 2\n"
                      "d_ff = 16\nmax_seq_len = 4\n"),
    ("bad_int", "vocab_size = ten\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 16\nmax_seq_len = 4\n"),
    ("unknown_key", "vocab_size = 10\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 16\n"
                    "max_seq_len = 4\nheads = 3\n"),
    ("heads_divide", "vocab_size = 10\nn_layers = 1\nd_model = 9\nn_heads = 2\nd_ff = 16\nmax_seq_len = 4\n"),
    ("no_equals", "vocab_size 10\n"),
    ("bad_role", "vocab_size = 10\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 16\nmax_seq_len = 4\n"
                 "role lm_head = linear\n"),
    ("empty_pattern", "role  = other\n"),
    ("bad_bool", "vocab_size = 10\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 16\nmax_seq_len = 4\n"
                 "tie_embeddings = maybe\n"),
    ("nonpositive", "vocab_size = 0\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 16\nmax_seq_len = 4\n"),
    ("tied_with_override", "vocab_size = 10\nn_layers = 2\nd_model = 8\nn_heads = 2\nd_ff = 16\n"
                           "max_seq_len = 4\ntie_embeddings = true\nrole fc2 = other\n"),
]


def gen_rules(tmp):
    out = {"plan_cases": [], "validate_cases": [], "parse_cases": [], "spec_cases": [],
           "spec_plans": []}
    for name, shapes, ovr, ns in FIXED_CASES + fuzz_cases():
        sp = write(tmp, "shapes.tsv", shapes_tsv(shapes))
        args_o = []
        if ovr:
            args_o = [write(tmp, "ovr.tsv", "".join(f"{p}\t{r}\n" for p, r in ovr))]
        for n in ns:
            text = run(["plan-shapes", sp, str(n)] + args_o, tmp)
            out["plan_cases"].append({"name": name, "shapes": shapes, "overrides": ovr,
                                      "n_shards": n, "expected": text})
    base = run(["plan-shapes", write(tmp, "shapes.tsv", shapes_tsv(CANONICAL)), "2"], tmp)
    plan_lines = [ln for ln in base.splitlines() if "\t" in ln and ln.split("\t")[1].startswith(("split", "repl"))]
    for name, edits, n in VALIDATE_EDITS:
        lines = []
        for ln in plan_lines:
            k, v = ln.split("\t")
            lines.append(f"{k}\t{edits.get(k, v)}")
        for k, v in edits.items():
            if k not in dict(ln.split("\t") for ln in plan_lines):
                lines.append(f"{k}\t{v}")
        plan_text = "\n".join(lines) + "\n"
        sp = write(tmp, "shapes.tsv", shapes_tsv(CANONICAL))
        pp = write(tmp, "plan.txt", plan_text)
        out["validate_cases"].append({"name": name, "shapes": CANONICAL, "plan": plan_text,
                                      "n_shards": n, "expected": run(["validate", sp, pp, str(n)], tmp)})
    for name, text, n in PARSE_TEXTS:
        sp = write(tmp, "shapes.tsv", "")
        pp = write(tmp, "plan.txt", text)
        out["parse_cases"].append({"name": name, "plan": text, "n_shards": n,
                                   "expected": run(["validate", sp, pp, str(n)], tmp)})
    for name, text in SPEC_TEXTS:
        p = write(tmp, "model.spec", text)
        out["spec_cases"].append({"name": name, "text": text, "expected": run(["shapes", p], tmp),
                                  "plan2": run(["plan", p, "2"], tmp)})
    for fn in sorted(os.listdir(SPECS)):
        text = open(os.path.join(SPECS, fn)).read()
        for n in [1, 2, 4, 8]:
            out["spec_plans"].append({"spec": fn, "text": text, "n_shards": n,
                                      "expected": run(["plan", os.path.join(SPECS, fn), str(n)], tmp),
                                      "shapes": run(["shapes", os.path.join(SPECS, fn)], tmp)})
    with open(os.path.join(HERE, "rules.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("rules.json:", {k: len(v) for k, v in out.items()})


def load_dump(d):
    data = np.fromfile(os.path.join(d, "data.bin"), dtype=np.float64)
    out = {}
    for ln in open(os.path.join(d, "index.tsv")):
        name, shape, off, cnt = ln.rstrip("\n").split("\t")
        shp = [int(x) for x in shape.strip("[]").split(",") if x]
        out[name] = data[int(off):int(off) + int(cnt)].reshape(shp)
    out["__comm_csv__"] = np.array(open(os.path.join(d, "comm_report.csv")).read())
    return out


def gen_numeric(tmp, tag, spec, dtype, dp, mp, gb, seq, steps, lr, wd, full):
    d = tempfile.mkdtemp(dir=tmp)
    subprocess.run([DRIVER, "golden", os.path.join(SPECS, spec), dtype, "42", str(dp), str(mp),
                    str(gb), str(seq), str(steps), str(lr), str(wd), d], check=True)
    dump = load_dump(d)
    meta = dict(spec=spec, dtype=dtype, seed=42, dp=dp, mp=mp, global_batch=gb, seq=seq,
                steps=steps, lr=lr, weight_decay=wd, batch_convention="cli.cpp:211-228 audit-batch child(step)")
    if full:
        arrays = {k: v for k, v in dump.items()}
    else:
        arrays = {"__comm_csv__": dump["__comm_csv__"]}
        for k, v in dump.items():
            if k.startswith("__"):
                continue
            flat = v.reshape(-1)
            if flat.size == 1:
                arrays[k] = v
            else:
                arrays["sum/" + k] = np.array(flat.sum())
                arrays["sumsq/" + k] = np.array((flat * flat).sum())
                arrays["head/" + k] = flat[:16].copy()
    arrays["__meta__"] = np.array(json.dumps(meta))
    path = os.path.join(HERE, f"{tag}.npz")
    np.savez_compressed(path, **arrays)
    print(tag, os.path.getsize(path), "bytes")


TRAINER_CASES = [
    # name, spec, seed, dp, mp, per_device_batch, accumulate, epochs, n_examples, seq, lr, wd, warmup
    ("trainer_mini_dp2_mp2_acc2", "mini.spec", 42, 2, 2, 2, 2, 2, 24, 16, 0.01, 0.01, 0.25),
    ("trainer_tiny_dp1_mp2", "tiny.spec", 42, 1, 2, 2, 1, 1, 8, 128, 1e-3, 0.01, 0.1),
]


def gen_trainer(tmp):
    out = {}
    for name, spec, seed, dp, mp, pdb, acc, ep, n, seq, lr, wd, wu in TRAINER_CASES:
        d = tempfile.mkdtemp(dir=tmp)
        r = subprocess.run([DRIVER, "trainer", os.path.join(SPECS, spec), str(seed), str(dp), str(mp), str(pdb),
                            str(acc), str(ep), str(n), str(seq), str(lr), str(wd), str(wu), d],
                           capture_output=True, text=True, check=True).stdout
        steps = [ln.split("\t") for ln in r.splitlines() if ln.startswith("STEP")]
        log = r.split("LOG\n", 1)[1]
        out[name] = dict(spec=spec, seed=seed, dp=dp, mp=mp, per_device_batch_size=pdb, accumulate=acc, epochs=ep,
                         n_examples=n, seq=seq, lr=lr, weight_decay=wd, warmup_rate=wu,
                         examples="RngStream(seed, 'examples'): n x (seq+1) next_below(vocab) in order; "
                                  "tokens = ex[:-1], targets = ex[1:], weights = 1",
                         losses=[float(x[2]) for x in steps], lrs=[float(x[3]) for x in steps], log=log)
    with open(os.path.join(HERE, "trainer.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("trainer.json:", {k: len(v["losses"]) for k, v in out.items()})


def gen_ext_plans(tmp):
    """Plans the REFERENCE derives (plan-shapes) for the SwiGLU / RMSNorm extension trees
    (SURVEY D2/D3): the rule engine itself is the reference's, so the gate / up / down splits of
    the extension are pinned exactly like the reference family's."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from oracle import rng_ref  # noqa: E402
    cases = []
    for spec_name, n_list in (("mini_swiglu.spec", (1, 2, 4)), ("llama7b_swiglu.spec", (1, 2, 4, 8)),
                              ("mini_t5.spec", (1, 2, 4)), ("t5_11b.spec", (1, 2, 4, 8))):
        kv, ovr = {}, []
        for ln in open(os.path.join(SPECS, spec_name)):
            ln = ln.split("#")[0].strip()
            if not ln:
                continue
            k, v = (x.strip() for x in ln.split("=", 1))
            if k.startswith("role "):
                ovr.append((k[5:].strip(), v))
            else:
                kv[k] = v if k in ("mlp", "norm", "arch") else int(v)
        shapes = [(n, list(sh)) for n, sh in rng_ref.transformer_param_shapes(kv)]
        sp = write(tmp, "shapes.tsv", shapes_tsv(shapes))
        args_o = [write(tmp, "ovr.tsv", "".join(f"{p}\t{r}\n" for p, r in ovr))] if ovr else []
        for n in n_list:
            cases.append({"name": spec_name, "shapes": shapes, "overrides": ovr, "n_shards": n,
                          "expected": run(["plan-shapes", sp, str(n)] + args_o, tmp)})
    with open(os.path.join(HERE, "ext_plans.json"), "w") as f:
        json.dump({"plan_cases": cases}, f)
    print("ext_plans.json:", len(cases))


CKPT_CASES = {
    # name -> how the test derives the file from the golden snapshot
    "cut1000": "first 1000 bytes",
    "cut61": "first 61 bytes (header + RNG block, no records)",
    "empty": "empty file",
    "magic": "b'NOPE' + 64 zero bytes",
    "version": "byte 4 set to 0xEE",
    "dtype": "byte 88 (dtype of the first record) set to 1",
    "rank": "byte 89..92 (rank of the first record) set to 99",
    "order": "the first params/ record renamed to adam_x/ (same length)",
}


def ckpt_transform(name, raw):
    if name == "cut1000":
        return raw[:1000]
    if name == "cut61":
        return raw[:61]
    if name == "empty":
        return b""
    if name == "magic":
        return b"NOPE" + bytes(64)
    b = bytearray(raw)
    if name == "version":
        b[4] = 0xEE
    elif name == "dtype":
        b[88] = 1
    elif name == "rank":
        b[89:93] = (99).to_bytes(4, "little")
    elif name == "order":
        i = raw.index(b"params/embed/tok/kernel")
        b[i:i + 7] = b"adam_x/"
    return bytes(b)


def gen_checkpoint(tmp):
    """SWCK golden: the reference's save_checkpoint of the mini decoder after 3 sharded AdamW
    steps (f32, dp=1, mp=2, seed 42, "train" stream advanced 17 draws), plus the reference's
    load_checkpoint verdict on it and on corrupted copies (checkpoint.hpp:233-298)."""
    d = tempfile.mkdtemp(dir=tmp)
    path = os.path.join(HERE, "mini_f32_mp2_step3.swck")
    env = dict(os.environ, SW_REF_CKPT=path)
    subprocess.run([DRIVER, "golden", os.path.join(SPECS, "mini.spec"), "f32", "42", "1", "2", "2", "16", "3",
                    "0.01", "0.01", d], check=True, env=env, stdout=subprocess.DEVNULL)
    raw = open(path, "rb").read()

    def verdict(fpath, mp=2, dtype="f32"):
        r = subprocess.run([DRIVER, "ckload", os.path.join(SPECS, "mini.spec"), dtype, str(mp), fpath],
                           capture_output=True, text=True, check=True)
        return r.stdout.strip()

    cases = {}
    for name, how in CKPT_CASES.items():
        f = os.path.join(tmp, name + ".swck")
        open(f, "wb").write(ckpt_transform(name, raw))
        cases[name] = dict(transform=how, message=verdict(f))
    out = dict(file=os.path.basename(path), spec="mini.spec", seed=42, dp=1, mp=2, global_batch=2, seq=16,
               steps=3, lr=0.01, weight_decay=0.01, size=len(raw),
               rngs=[dict(name="train", note="RngStream(42, 'train') after 17 next_u64()")],
               ok={str(mp): verdict(path, mp) for mp in (1, 2, 4)},
               f64_load=verdict(path, 2, "f64"), cases=cases)
    with open(os.path.join(HERE, "checkpoint.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("checkpoint.json:", out["ok"], {k: v["message"][:40] for k, v in cases.items()})


def main():
    build()
    with tempfile.TemporaryDirectory() as tmp:
        gen_rules(tmp)
        gen_trainer(tmp)
        gen_numeric(tmp, "mini_f64_dp1_mp2", "mini.spec", "f64", 1, 2, 2, 16, 3, 1e-2, 0.01, True)
        gen_numeric(tmp, "mini_f64_dp2_mp2", "mini.spec", "f64", 2, 2, 4, 16, 2, 1e-2, 0.01, False)
        gen_numeric(tmp, "mini_f32_dp1_mp4", "mini.spec", "f32", 1, 4, 2, 16, 2, 1e-2, 0.01, False)
        gen_numeric(tmp, "tiny_f64_dp1_mp2", "tiny.spec", "f64", 1, 2, 4, 128, 1, 1e-3, 0.01, False)
        gen_checkpoint(tmp)
        gen_ext_plans(tmp)


if __name__ == "__main__":
    if sys.argv[1:] == ["checkpoint"]:
        build()
        with tempfile.TemporaryDirectory() as tmp:
            gen_checkpoint(tmp)
    elif sys.argv[1:] == ["ext_plans"]:
        build()
        with tempfile.TemporaryDirectory() as tmp:
            gen_ext_plans(tmp)
    else:
        sys.exit(main())
