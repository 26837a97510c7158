"""The header-only C++ face (include/shardweave_b200.hpp) as a reference-style caller would use
it: examples/cpp_train_step derives plans bit-exact with the reference (CPU) and takes
optimizer steps on the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "cpp_train_step")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "rules.json")))


def _exe():
    if not os.path.exists(EXE):
        subprocess.run(["make", "-C", ROOT, "examples/cpp_train_step"], check=True, capture_output=True)
    return EXE


@pytest.mark.parametrize("case", [c for c in GOLDEN["spec_plans"] if c["n_shards"] in (2, 8)],
                         ids=lambda c: f"{c['spec']}-n{c['n_shards']}")
def test_cpp_plan_matches_reference(case):
    spec = os.path.join(ROOT, "oracle", "specs", case["spec"])
    out = subprocess.run([_exe(), spec, str(case["n_shards"])], capture_output=True, text=True, check=True).stdout
    want = "".join(ln + "\n" for ln in case["expected"].splitlines() if not ln.startswith("STATE"))
    assert out == want


@pytest.mark.gpu
def test_cpp_train_steps_on_gpu():
    spec = os.path.join(ROOT, "oracle", "specs", "tiny.spec")
    out = subprocess.run([_exe(), spec, "2", "--run", "2", "128", "3"], capture_output=True, text=True,
                         check=True).stdout
    losses = [float(ln.split("loss=")[1]) for ln in out.splitlines() if ln.startswith("step=")]
    assert len(losses) == 3 and losses[2] < losses[0]
    assert "all_reduce,24," in out  # 2 layers x (2 fwd + 2 bwd) all-reduces per step, 3 steps
