#!/usr/bin/env python
"""Benchmark of the B200 tensor-parallel training step (BASELINE.json configs[1]):
LLaMA-7B-shape decoder in the reference's model family (oracle/specs/llama7b.spec:
d=4096, H=32, d_ff=11008, V=32000, L=32, learned positions, LayerNorm, tanh-GeLU),
seq 2048, bf16 compute / fp32 master + AdamW, synthetic tokens, random init, TP = number of
GPUs (one process per GPU, NCCL over NVLink), one optimizer step per timed step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0). See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import re
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--spec", default=os.path.join(ROOT, "oracle", "specs", "llama7b_vocab_parallel.spec"),
                    help="model spec; the default carries `role lm_head/kernel = fully_connected` "
                         "(vocab-parallel head, SURVEY D1) - identical to llama7b.spec at TP=1")
    ap.add_argument("--batch", type=int, default=8,
                    help="sequences per replica per step (8 x 2048 tokens: 165 GB of the 180 GB at TP=1; the "
                         "per-tile optimizer traffic of the fused wgrads is amortised over twice the tokens "
                         "of batch 4: +3%% tokens/s at a lower clock, profiles/r2_bench_batch8_vs_4.txt)")
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--profile-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return FALLBACK_PEAKS, "fallback"


def shape_name(spec_path):
    """The BASELINE config a spec file stands for (oracle/specs/*.spec)."""
    base = os.path.basename(spec_path)
    for key, name in (("gptj", "GPT-J-6B-shape"), ("opt66b", "OPT-66B-shape"), ("llama7b", "LLaMA-7B-shape")):
        if base.startswith(key):
            return name
    return os.path.splitext(base)[0]


def read_spec(path):
    out = {"tie_embeddings": False}
    for ln in open(path):
        ln = ln.split("#")[0].strip()
        if "=" in ln and not ln.startswith("role"):
            k, v = (x.strip() for x in ln.split("="))
            if k in ("mlp", "norm"):
                out[k] = v
            else:
                out[k] = (v in ("true", "yes", "1")) if k == "tie_embeddings" else int(v)
    return out


def matmul_params(s, layers=None):
    L = s["n_layers"] if layers is None else layers
    d, ff, V = s["d_model"], s["d_ff"], s["vocab_size"]
    n_mlp = 3 if s.get("mlp") == "swiglu" else 2  # SwiGLU: gate, up, down (6.607 G)
    return L * (4 * d * d + n_mlp * d * ff) + V * d


def train_flops_per_token(s, T, layers=None):
    """Algorithmic fwd+bwd FLOPs/token: 6*N_matmul + 6*L*d*T (causal attention counted once),
    BASELINE.md §2 (32.60 GFLOP/token for the reference-family LLaMA-7B shape at T=2048; 41.25
    with the SwiGLU extension)."""
    L = s["n_layers"] if layers is None else layers
    return 6.0 * matmul_params(s, L) + 6.0 * L * s["d_model"] * T


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# CPU baseline: the reference itself (oracle/_ref/sw_ref_driver = unmodified reference sources)
# ------------------------------------------------------------------------------------------
def cpu_reference_run(spec_path, steps, warmup, sample_tokens=32):
    """Runs the reference's own CPU step (spmd_forward_backward + adamw_step, Trainer order)
    on a bounded sample: the full-width model truncated to ONE layer, one sequence of
    `sample_tokens` tokens, mp=1. Returns per-step seconds and the extrapolation to the full
    workload by algorithmic FLOPs."""
    drv = os.path.join(ROOT, "oracle", "_ref", "sw_ref_driver")
    if not os.path.exists(drv):
        return None, "oracle/_ref/sw_ref_driver not built"
    s = read_spec(spec_path)
    text = open(spec_path).read()
    text = re.sub(r"(?m)^n_layers\s*=.*$", "n_layers = 1", text)
    with tempfile.NamedTemporaryFile("w", suffix=".spec", delete=False) as f:
        f.write(text)
        tmp = f.name
    try:
        r = subprocess.run([drv, "bench", tmp, "1", "1", str(sample_tokens), str(steps + warmup), "0"],
                           capture_output=True, text=True, timeout=3600)
    finally:
        os.unlink(tmp)
    times = [float(ln.split("\t")[2]) for ln in r.stdout.splitlines() if ln.startswith("STEP")]
    if len(times) < steps + warmup:
        return None, "reference driver failed: " + (r.stdout + r.stderr)[-300:]
    timed = times[warmup:]
    t_step = sum(timed) / len(timed)
    f_sample = train_flops_per_token(s, sample_tokens, layers=1)
    f_full = train_flops_per_token(s, 2048)
    tok_s_sample = sample_tokens / t_step
    value = tok_s_sample * f_sample / f_full
    sample = (f"reference CPU step (spmd_forward_backward + adamw_step) of the full-width model "
              f"truncated to 1 of {s['n_layers']} layers, 1 x {sample_tokens} tokens, mp=1, "
              f"{t_step:.2f} s/step ({tok_s_sample:.2f} tok/s on the sample); value extrapolated "
              f"to the {s['n_layers']}-layer T=2048 step by algorithmic FLOPs "
              f"({f_sample / 1e9:.2f} vs {f_full / 1e9:.2f} GFLOP/token)")
    return {"value": value, "unit": "tokens/s", "cores": 1, "kind": "reference", "sample": sample,
            "seconds_per_sample_step": t_step, "steps": timed}, None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    res, err = cpu_reference_run(args.spec, args.steps, args.warmup)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return
    s = read_spec(args.spec)
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * args.batch * args.seq / res["value"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{shape_name(args.spec)} decoder (reference family) fwd+bwd+AdamW, "
                               f"seq {args.seq}, batch {args.batch}, CPU reference", "seq_len": args.seq,
                   "global_batch": args.batch, "parallelism": "cpu"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "flops_per_token": train_flops_per_token(s, args.seq),
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch

    from paper_2310_16355_b200 import _lib, engine, rules
    from paper_2310_16355_b200 import dist as D

    info = D.rank_info()
    world, rank, local = info.world, info.rank, info.local_rank
    # Tensor-parallel runs send the row-parallel all-reduce payloads in bf16 (the compute dtype;
    # half the NVLink bytes of fp32 partials). At LLaMA-7B width and mp = 8 the gradients stay
    # within 0.84% rel-L2 of mp = 1 (fp32 payloads: 0.60%), profiles/r1_ar_bf16_check.json.
    # SW_AR_BF16=0 keeps fp32 payloads.
    if world > 1:
        os.environ.setdefault("SW_AR_BF16", "1")
    torch.cuda.set_device(local)
    dist = D.init_host_group(info)
    tp, dp = world, 1

    spec = rules.read_model_spec(args.spec)
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, tp, spec.overrides)
    nccl_id = D.share_nccl_id(dist, rank)
    mesh = engine.Mesh(dp, tp, 1, rank if world > 1 else 0, world, nccl_id, local)
    B, T = args.batch, args.seq
    model = engine.Model(spec, plan, mesh, B, T)
    model.init_params(42, "model-init")
    stream = torch.cuda.ExternalStream(model.stream())
    V = spec.vocab_size
    rng = np.random.default_rng(1234)
    rows = dp * B
    batches = [(rng.integers(0, V, (rows, T), dtype=np.int32), rng.integers(0, V, (rows, T), dtype=np.int32))
               for _ in range(2)]
    ones = np.ones((rows, T), np.float32)
    cfg = engine.AdamWConfig(lr=1e-4, weight_decay=0.01)

    def barrier():
        torch.cuda.synchronize()
        stream.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        return D.max_over_ranks(dist, x)

    # ---- device-resident inputs: value ----
    model.stage_batch(*batches[0], ones)
    for _ in range(args.warmup):
        model.train_step(cfg)
    launches_per_step = model.launch_count()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        model.train_step(cfg)
    e1.record(stream)
    barrier()
    clock = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    loss = model.loss()
    tokens_per_step = rows * T
    value = tokens_per_step / (ms / 1e3)

    # ---- per-launch profile (CUDA events on the model stream) ----
    model.set_profiling(True)
    for _ in range(args.profile_steps):
        model.train_step(cfg)
    prof = model.read_profile()
    model.set_profiling(False)
    for v in prof.values():
        v["ms"] /= args.profile_steps
        v["work"] /= args.profile_steps
        v["launches"] //= args.profile_steps

    # ---- end to end through the public API with host buffers ----
    pinned = [(torch.from_numpy(t).pin_memory(), torch.from_numpy(y).pin_memory()) for t, y in batches]
    pw = torch.from_numpy(ones).pin_memory()
    L = engine._declare()
    c = cfg.c()
    loss_host = C.c_double()
    barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        tk, tg = pinned[i % 2]
        _lib.check(L.sw_model_stage_batch(model._h, tk.data_ptr(), tg.data_ptr(), pw.data_ptr()))
        _lib.check(L.sw_model_train_step(model._h, C.byref(c)))
        _lib.check(L.sw_model_last_loss(model._h, C.byref(loss_host)))
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": tokens_per_step * args.steps / e2e_s, "unit": "tokens/s",
           "h2d_bytes_per_step": int(pinned[0][0].numel() * 4 * 2 + pw.numel() * 4),
           "d2h_bytes_per_step": 8 + 4, "ms_per_step": 1e3 * e2e_s / args.steps}

    peaks, peak_src = load_peaks()
    s = read_spec(args.spec)
    fpt = train_flops_per_token(s, T)
    step_tflops_per_gpu = fpt * tokens_per_step / (ms / 1e3) / 1e12 / world
    g = prof["gemm"]
    gemm_tflops = g["work"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0
    peak_t = peaks.get("bf16_tflops_sustained", FALLBACK_PEAKS["bf16_tflops_sustained"])
    traffic = None
    tp_file = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tp_file):
        traffic = json.load(open(tp_file)).get("dram_bytes_per_launch")
    breakdown = {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                     ("tflops" if k in ("gemm", "attn_fwd", "attn_bwd") else "gbs"):
                         round(v["work"] / (v["ms"] / 1e3) / (1e12 if k in ("gemm", "attn_fwd", "attn_bwd") else 1e9), 1)
                         if v["ms"] > 0 else None}
                 for k, v in prof.items() if v["launches"] > 0}
    comm = prof["comm"]
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (uniform random token ids, random-init weights from the reference init stream)",
        "config": {"workload": f"{shape_name(args.spec)} decoder ("
                               + ("SwiGLU MLP + RMSNorm extension" if s.get("mlp") == "swiglu"
                                  else "reference model family")
                               + f", {s['n_layers']} layers, "
                               f"d={s['d_model']}, H={s['n_heads']}, d_ff={s['d_ff']}, V={s['vocab_size']}) "
                               f"train step: fwd+bwd+AdamW, seq {T}",
                   "spec": os.path.relpath(args.spec, ROOT), "global_batch": rows, "seq_len": T,
                   "parallelism": f"tp{tp}" if dp == 1 else f"dp{dp}xtp{tp}",
                   "plan": "reference rules (derive_plan) + spec overrides: lm_head/kernel "
                           + plan.at("lm_head/kernel") + (" (vocab-parallel)" if tp > 1 and plan.at("lm_head/kernel") == "split:0" else ""),
                   "l2": "inputs larger than L2 (activations/weights >> 126 MB); no flush",
                   "allreduce": ("bf16" if os.environ.get("SW_AR_BF16") == "1" else "fp32") + " payloads, "
                                 f"{os.environ.get('SW_AR_CHUNKS', '4')} row chunks on a comm stream"},
        "mfu": {"tflops_per_gpu": round(step_tflops_per_gpu, 1),
                "frac_of_measured_bf16_sustained": round(step_tflops_per_gpu / peak_t, 3),
                "frac_of_2.25PF_spec": round(step_tflops_per_gpu / 2250.0, 3),
                "flops_per_token": fpt},
        "roofline": {"kernel": "tcgen05 GEMM family (all linear fwd/dgrad/wgrad launches of the step)",
                     "bound": "tensor", "achieved": round(gemm_tflops, 1), "peak": peak_t,
                     "unit": "TFLOP/s", "frac": round(gemm_tflops / peak_t, 3), "traffic": traffic,
                     "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
                     "share_of_step": round(g["ms"] / ms, 3) if ms > 0 else None},
        "breakdown_ms_per_step": breakdown,
        "clocks": clock,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "loss": loss,
        "device_bytes": model.device_bytes(),
    }
    if world > 1 and comm["ms"] > 0:
        line["ar_bus_gbs"] = round(comm["work"] / (comm["ms"] / 1e3) / 1e9, 1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res, err = cpu_reference_run(args.spec, 2, 1)
        line["cpu_baseline"] = ({k: res[k] for k in ("value", "unit", "cores", "kind", "sample")}
                                if res else {"unavailable": err})
    if rank == 0:
        print(json.dumps(line))
    model.close()
    mesh.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
