"""Trainer: the inner loop of the reference's Trainer::fit (pipeline.hpp:351-454) driving the B200
step. The user's collate_fn hook keeps its meaning (a list of examples -> named batch-major
inputs "tokens" / "targets" / "weights", ids as integers); the loss is the reference's
transformer_loss (model.hpp:144-152), lowered once onto the mesh.

Per optimizer step, as the reference: for each micro-batch collate the global batch (dp * rows),
forward+backward with gradient accumulation, then scale by 1/accumulate, average over the data
parallel axis, AdamW at the warmup/decay learning rate, and append
`step=<i> loss=<%.9g> lr=<%.9g>` to run.log. Epochs shuffle with
RngStream(seed, "data-shuffle").child(epoch).permutation(n) and drop the last partial step.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib, engine, rules
from ._lib import ConfigError


def scheduled_lr(step: int, total_steps: int, warmup_steps: int, peak: float) -> float:
    """pipeline.hpp:28-40: linear warmup to `peak`, then linear decay to zero."""
    if total_steps < 1:
        raise ConfigError(3, f"scheduled_lr: total_steps must be positive, got {total_steps}")
    if step < warmup_steps:
        return peak * float(step + 1) / float(warmup_steps)
    if step >= total_steps:
        return 0.0
    return peak * float(total_steps - step) / float(total_steps - warmup_steps)


def stream_id(name: str) -> int:
    """RngStream's named-stream id (FNV-1a 64 of the name, rng.hpp)."""
    h = 0xCBF29CE484222325
    for c in name.encode():
        h = ((h ^ c) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def permutation(seed: int, stream: str, child: int, n: int) -> np.ndarray:
    L = _lib.lib()
    L.sw_rng_permutation.argtypes = [C.c_uint64, C.c_char_p, C.c_int64, C.c_uint64, C.c_void_p]
    L.sw_rng_permutation.restype = C.c_int
    out = np.empty(n, np.uint64)
    _lib.check(L.sw_rng_permutation(seed, stream.encode(), child, n, out.ctypes.data))
    return out


@dataclass
class RunConfig:
    """RunConfig (pipeline.hpp:62-76), the fields the training step uses."""
    n_epochs: int = 1
    per_device_batch_size: int = 1
    accumulate_grad_batches: int = 1
    optimizer: engine.AdamWConfig = field(default_factory=engine.AdamWConfig)
    warmup_rate: float = 0.1


def _fmt(v: float) -> str:
    return "%.9g" % v


class Trainer:
    def __init__(self, spec: rules.ModelSpec, mesh: engine.Mesh, seq_len: int, collate_fn, config: RunConfig,
                 seed: int = 42, workdir: str = ".", init_stream: str = "model-init"):
        if collate_fn is None:
            raise ConfigError(3, "Trainer: collate_fn and loss_fn are required")
        if config.per_device_batch_size < 1:
            raise ConfigError(3, "Trainer: batch sizes must be positive")
        if config.accumulate_grad_batches < 1:
            raise ConfigError(3, "Trainer: accumulate_grad_batches must be positive, got "
                                 f"{config.accumulate_grad_batches}")
        if not 0.0 <= config.warmup_rate <= 1.0:
            raise ConfigError(3, f"Trainer: warmup_rate must be in [0, 1], got {_fmt(config.warmup_rate)}")
        self.spec, self.mesh, self.seq_len = spec, mesh, seq_len
        self.collate_fn, self.config, self.seed = collate_fn, config, seed
        shapes = rules.transformer_param_shapes(spec)
        self.plan = rules.derive_plan(shapes, mesh.mp, spec.overrides)
        self.model = engine.Model(spec, self.plan, mesh, config.per_device_batch_size, seq_len)
        self.model.init_params(seed, init_stream)
        os.makedirs(workdir, exist_ok=True)
        self.workdir = workdir
        self.log_path = os.path.join(workdir, "run.log")
        self._log = open(self.log_path, "w")
        self.step = 0

    def _stage(self, inputs: dict):
        t = np.asarray(inputs["tokens"])
        y = np.asarray(inputs["targets"])
        w = inputs.get("weights")
        rows = t.shape[0]
        for name, a in inputs.items():
            if np.asarray(a).ndim == 0:
                raise _lib.ShapeError(1, f"Trainer: collated input '{name}' is a scalar; inputs must be batch-major")
            if np.asarray(a).shape[0] != rows:
                raise _lib.ShapeError(1, "Trainer: collated inputs disagree on batch size")
        self.model.stage_batch(np.rint(t).astype(np.int32), np.rint(y).astype(np.int32),
                               None if w is None else np.asarray(w, np.float32))
        return rows

    def load(self, checkpoint_path: str):
        """Trainer::load (pipeline.hpp:338-345): restore a snapshot saved by this configuration;
        fit() then resumes at the epoch the optimizer step implies."""
        self.model.load_checkpoint(checkpoint_path)
        self.step = self.model.state_info()[0]

    def fit(self, train_examples, stop_after_epoch: int = -1):
        """Epochs up to n_epochs (absolute, so a loaded checkpoint resumes where it left off);
        stop_after_epoch pauses earlier with the LR schedule still spanning n_epochs. Every
        finished epoch writes <workdir>/last.ckpt (pipeline.hpp:536-539)."""
        cfg = self.config
        if cfg.n_epochs < 1:
            raise ConfigError(3, f"Trainer: n_epochs must be positive, got {cfg.n_epochs}")
        if not train_examples:
            raise ConfigError(3, "Trainer: no training examples")
        dp = self.mesh.dp
        global_rows = cfg.per_device_batch_size * dp
        rows_per_step = global_rows * cfg.accumulate_grad_batches
        steps_per_epoch = len(train_examples) // rows_per_step
        if steps_per_epoch == 0:
            raise ConfigError(3, f"Trainer: {len(train_examples)} examples is fewer than one optimizer step "
                                 f"of {rows_per_step}")
        total_steps = steps_per_epoch * cfg.n_epochs
        warmup_steps = int(cfg.warmup_rate * total_steps)
        losses, lrs = [], []
        first_epoch = self.step // steps_per_epoch
        last_epoch = cfg.n_epochs if stop_after_epoch < 0 else min(stop_after_epoch, cfg.n_epochs)
        self.checkpoints = []
        for epoch in range(first_epoch, last_epoch):
            perm = permutation(self.seed, "data-shuffle", epoch, len(train_examples))
            for s in range(steps_per_epoch):
                lr = scheduled_lr(self.step, total_steps, warmup_steps, cfg.optimizer.lr)
                step_cfg = engine.AdamWConfig(lr, cfg.optimizer.beta1, cfg.optimizer.beta2, cfg.optimizer.eps,
                                              cfg.optimizer.weight_decay)
                loss_sum = 0.0
                try:
                    for micro in range(cfg.accumulate_grad_batches):
                        off = s * rows_per_step + micro * global_rows
                        batch = [train_examples[int(perm[off + i])] for i in range(global_rows)]
                        rows = self._stage(self.collate_fn(batch))
                        if rows != global_rows:
                            raise _lib.ShapeError(1, f"Trainer: collate_fn returned {rows} rows for a batch of "
                                                     f"{global_rows} examples")
                        if cfg.accumulate_grad_batches == 1:
                            # one micro-batch: the fused step (optimizer inside the backward when dp == 1)
                            self.model.train_step(step_cfg)
                        else:
                            self.model.forward_backward(accumulate=micro > 0)
                        loss_sum += self.model.loss() * dp  # loss() is the mean over replicas
                    if cfg.accumulate_grad_batches > 1:
                        self.model.scale_grads(1.0 / cfg.accumulate_grad_batches)
                        self.model.dp_sync()
                        self.model.adamw_step(step_cfg)
                except _lib.NonFiniteError as e:
                    raise _lib.NonFiniteError(4, f"Trainer: aborting at step {self.step + 1}: {e.message}") from None
                loss = loss_sum / (dp * cfg.accumulate_grad_batches)
                self._log.write(f"step={self.step} loss={_fmt(loss)} lr={_fmt(lr)}\n")
                self._log.flush()
                losses.append(loss)
                lrs.append(lr)
                self.step += 1
            last = os.path.join(self.workdir, "last.ckpt")
            self.model.save_checkpoint(last, [("train", self.seed, stream_id("train"), 0)])
            self.checkpoints.append(last)
        return losses, lrs
