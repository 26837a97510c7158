"""SWCK snapshot codec vs the reference (checkpoint.hpp:18-298), host only.

tests/golden/mini_f32_mp2_step3.swck was written by the reference's own save_checkpoint (mini
decoder, 3 sharded AdamW steps, dp=1 mp=2, seed 42, a "train" stream advanced 17 draws;
tests/golden/make_golden.py). checkpoint.json holds the reference's load_checkpoint verdict on
that file and on corrupted copies; the codec must agree byte-for-byte and message-for-message
(tests/test_checkpoint.cpp:66-233)."""
import json
import os

import numpy as np
import pytest

from oracle import rng_ref
from paper_2310_16355_b200 import _lib, checkpoint, rules
from tests.golden.make_golden import ckpt_transform

HERE = os.path.dirname(__file__)
GOLD = os.path.join(HERE, "golden")
META = json.load(open(os.path.join(GOLD, "checkpoint.json")))
FILE = os.path.join(GOLD, META["file"])


def test_reads_reference_snapshot():
    snap = checkpoint.read(FILE)
    assert (snap.step, snap.seed) == (3, 42)
    train = rng_ref.RngStream(42, "train")
    assert snap.rngs == [("train", 42, train.stream_id, 17)]
    spec = rules.read_model_spec(os.path.join(HERE, "..", "oracle", "specs", META["spec"]))
    shapes = rules.transformer_param_shapes(spec)
    want = [(k + "/" + n, tuple(s)) for n, s in shapes for k in ("params", "adam_m", "adam_v")]
    assert [(n, a.shape) for n, a in snap.records] == want
    for n, a in snap.records:
        assert a.dtype == np.float32 and np.all(np.isfinite(a)), n
        if n.startswith("adam_v/"):
            assert np.all(a >= 0), n


def test_write_reproduces_reference_bytes(tmp_path):
    snap = checkpoint.read(FILE)
    out = str(tmp_path / "copy.swck")
    checkpoint.write(out, snap)
    assert open(out, "rb").read() == open(FILE, "rb").read()


@pytest.mark.parametrize("case", sorted(META["cases"]))
def test_corrupt_files_fail_like_the_reference(case, tmp_path):
    raw = open(FILE, "rb").read()
    bad = str(tmp_path / (case + ".swck"))
    open(bad, "wb").write(ckpt_transform(case, raw))
    want = META["cases"][case]["message"]
    if want.startswith("ok "):
        snap = checkpoint.read(bad)
        assert want == f"ok {snap.step} {snap.seed} {len(snap.records) // 3}"
        return
    with pytest.raises(_lib.CheckpointError) as e:
        checkpoint.read(bad)
    assert e.value.message == want


def test_missing_file(tmp_path):
    p = str(tmp_path / "does-not-exist.swck")
    with pytest.raises(_lib.CheckpointError) as e:
        checkpoint.read(p)
    assert e.value.message == f"checkpoint: cannot open '{p}' for reading"


def test_round_trip_synthetic(tmp_path):
    rng = np.random.default_rng(0)
    snap = checkpoint.Snapshot(step=7, seed=11, rngs=[("train", 1, 2, 3), ("eval", 4, 5, 6)])
    for name, shape in (("a/kernel", (3, 5)), ("a/bias", (5,)), ("s", ())):
        for k in ("params", "adam_m", "adam_v"):
            snap.records.append((f"{k}/{name}", rng.standard_normal(shape).astype(np.float32)))
    p = str(tmp_path / "s.swck")
    checkpoint.write(p, snap)
    back = checkpoint.read(p)
    assert (back.step, back.seed, back.rngs) == (7, 11, snap.rngs)
    for (n1, a1), (n2, a2) in zip(snap.records, back.records):
        assert n1 == n2 and a1.shape == a2.shape and np.array_equal(a1.view(np.uint32), a2.view(np.uint32))


def test_wrapping_dims_are_rejected(tmp_path):
    """dims whose product wraps 2^64 (here 2^32 x 2^32 -> 0) must not pass the truncation guard
    with a shape that does not match the data (overflow-checked numel)."""
    import struct
    snap = checkpoint.Snapshot(step=1, seed=2, rngs=[])
    for k in ("params", "adam_m", "adam_v"):
        snap.records.append((f"{k}/w", np.arange(15, dtype=np.float32).reshape(3, 5)))
    p = str(tmp_path / "w.swck")
    checkpoint.write(p, snap)
    raw = open(p, "rb").read()
    dims = struct.pack("<IQQ", 2, 3, 5)
    assert raw.count(dims) == 3
    bad = raw.replace(dims, struct.pack("<IQQ", 2, 1 << 32, 1 << 32), 1)
    q = str(tmp_path / "bad.swck")
    open(q, "wb").write(bad)
    with pytest.raises(_lib.CheckpointError) as e:
        checkpoint.read(q)
    assert e.value.message.startswith("checkpoint: truncated, needed 4 more bytes")
    # an empty tensor with a huge leading dim is still a valid (empty) record
    empty = raw.replace(dims + np.arange(15, dtype=np.float32).tobytes(),
                        struct.pack("<IQQ", 2, 1 << 40, 0))
    q2 = str(tmp_path / "empty.swck")
    open(q2, "wb").write(empty)
    back = checkpoint.read(q2)
    assert [a.shape for _, a in back.records] == [(1 << 40, 0)] * 3
