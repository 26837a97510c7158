"""Inference-only models (sw_model_create_inference): the Predictor path of cli.cpp:425-447 /
pipeline.hpp:189-246 without the train state. Same program, same kernels, so logits and generated
tokens must be bit-identical to a training model holding the same parameters; the training entry
points must refuse; and the footprint must be the bf16 weights + K/V cache (what lets the
OPT-66B shape, cfg5, fit one B200)."""
import os

import numpy as np
import pytest

from oracle import model_ref, rng_ref
from paper_2310_16355_b200 import engine, rules

pytestmark = pytest.mark.gpu
SPECS = os.path.join(os.path.dirname(__file__), "..", "oracle", "specs")


def make(spec_name, mp, batch, seq, inference, seed=7):
    spec = rules.read_model_spec(os.path.join(SPECS, spec_name))
    plan = rules.derive_plan(rules.transformer_param_shapes(spec), mp, spec.overrides)
    model = engine.Model(spec, plan, engine.Mesh(1, mp), batch, seq, inference=inference)
    model.init_params(seed, "model-init")
    return model, spec


def tokens(spec, batch, seq, name="tokens"):
    return rng_ref.RngStream(5, name).below(batch * seq, spec.vocab_size).reshape(batch, seq).astype(np.int32)


@pytest.mark.parametrize("spec_name,mp", [("mini.spec", 1), ("mini.spec", 2), ("mini_swiglu.spec", 2),
                                          ("mini_vocab_parallel.spec", 2), ("tiny.spec", 1)])
def test_inference_logits_and_tokens_match_training_model(spec_name, mp):
    batch, seq = 2, 16
    train, spec = make(spec_name, mp, batch, seq, False)
    infer, _ = make(spec_name, mp, batch, seq, True)
    x = tokens(spec, batch, seq)
    y = np.roll(x, -1, 1)
    for m in (train, infer):
        m.stage_batch(x, y)
    a, b = train.forward_logits(), infer.forward_logits()
    assert np.array_equal(a, b)
    assert train.loss() == infer.loss()
    # parameters read back: fp32 small parameters exactly, GEMM weights as their bf16 shadow
    for name, shape in train.shapes.items():
        p, q = train.get_param(name), infer.get_param(name)
        if len(shape) == 2 and not name.startswith("embed/"):
            p = model_ref.bf16_round(p.astype(np.float64)).astype(np.float32)
        assert np.array_equal(p, q), name
    # greedy generation, cached steps and the sliding window
    prompts = tokens(spec, batch, 5, "prompts")
    assert np.array_equal(train.generate(prompts, 20), infer.generate(prompts, 20))


def test_inference_model_refuses_training():
    model, spec = make("mini.spec", 2, 2, 16, True)
    x = tokens(spec, 2, 16)
    model.stage_batch(x, x)
    cfg = engine.AdamWConfig()
    for call in (lambda: model.forward_backward(), lambda: model.train_step(cfg), lambda: model.adamw_step(cfg),
                 lambda: model.dp_sync(), lambda: model.scale_grads(0.5), lambda: model.get_grad("embed/tok/kernel"),
                 lambda: model.get_adam("embed/tok/kernel"), lambda: model.save_checkpoint("/tmp/never.swck")):
        with pytest.raises(engine._lib.ConfigError, match="inference-only"):
            call()
    # still serves after the refusals
    assert np.isfinite(model.forward_logits()).all()


def test_inference_set_param_and_checkpoint_load(tmp_path):
    batch, seq = 2, 16
    train, spec = make("mini.spec", 2, batch, seq, False, seed=11)
    path = str(tmp_path / "m.swck")
    train.save_checkpoint(path, [])
    infer, _ = make("mini.spec", 2, batch, seq, True, seed=99)
    infer.load_checkpoint(path)  # parameters only; the AdamW records are skipped
    x = tokens(spec, batch, seq)
    for m in (train, infer):
        m.stage_batch(x, x)
    assert np.array_equal(train.forward_logits(), infer.forward_logits())
    # set_param of a column-split GEMM weight goes through the bf16 shadow only
    name = "block_0/attn/q/kernel"
    w = rng_ref.RngStream(1, "w").normals(int(np.prod(infer.shapes[name]))).reshape(infer.shapes[name])
    w = w.astype(np.float32)
    infer.set_param(name, w)
    train.set_param(name, w)
    got = infer.get_param(name)
    assert np.abs(got - w).max() <= np.abs(w).max() * 2.0 ** -8
    assert np.array_equal(train.forward_logits(), infer.forward_logits())


def test_inference_footprint():
    batch, seq = 4, 16
    train, spec = make("mini.spec", 1, batch, seq, False)
    infer, _ = make("mini.spec", 1, batch, seq, True)
    n = sum(int(np.prod(d)) for _, d in rules.transformer_param_shapes(spec))
    # training: 4 fp32 + 1 bf16 copies of the state; inference: bf16 + the small fp32 region
    assert train.device_bytes() >= 18 * n
    assert infer.device_bytes() < train.device_bytes() / 2


def test_opt66b_width_tp8_generation_matches_tp1(tmp_path):
    """cfg5 at OPT-66B width (2 of 64 layers, tied 50272 x 9216 embedding, 72 heads of 128): the
    TP=8 plan's KV-cached greedy generation (inference-only model, the 8 ranks emulated on one
    GPU) picks the tokens of the unsharded model's teacher-forced full-window forward except at
    near-ties; the per-rank footprint is the TP=8 shard of the bf16 weights + K/V cache."""
    path = tmp_path / "opt66b_2l.spec"
    path.write_text("vocab_size = 50272\nn_layers = 2\nd_model = 9216\nn_heads = 72\nd_ff = 36864\n"
                    "max_seq_len = 256\ntie_embeddings = true\n")
    spec = rules.read_model_spec(str(path))
    shapes = rules.transformer_param_shapes(spec)
    batch, P, n_new = 2, 24, 40
    prompts = rng_ref.RngStream(4, "prompts").below(batch * P, spec.vocab_size).reshape(batch, P)
    got = {}
    for mp in (8, 1):
        plan = rules.derive_plan(shapes, mp, spec.overrides)
        model = engine.Model(spec, plan, engine.Mesh(1, mp), batch, 256, inference=True)
        model.init_params(3, "model-init")
        model.set_param("embed/tok/kernel", model.get_param("embed/tok/kernel") * 24.0)
        got[mp] = model.generate(prompts, n_new)
        if mp == 8:
            per_rank = model.device_bytes() / 8
            continue
        ctx = np.concatenate([prompts, got[8]], 1)
        win = np.zeros((batch, 256), np.int32)
        win[:, :P + n_new - 1] = ctx[:, :P + n_new - 1]
        model.stage_batch(win, win)
        logits = model.forward_logits()[:, P - 1:P + n_new - 1]
    srt = np.sort(logits, -1)
    margin = (srt[..., -1] - srt[..., -2]) / np.maximum(np.abs(srt[..., -1]), 1.0)
    decisive = margin >= 0.02
    assert np.array_equal(logits.argmax(-1)[decisive], got[8][decisive])
    assert decisive.mean() > 0.5
    n_params = sum(int(np.prod(d)) for _, d in shapes)
    assert per_rank < 2 * n_params / 8 + 4 * (50272 + 256) * 9216 + 1.5e9
