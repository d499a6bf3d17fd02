"""CPU: bench.py's reference arm (`--impl reference`: the reference compiled
from its own sources into oracle/_ref, timed on the host cores) prints the
driver's JSON contract, at N=1 and under torchrun with two ranks (rank 0
alone prints; the other rank exits 0 without work)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAMPLE = str(1 << 20)   # 1M params per timed step: a fraction of a second


def _ref_built():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcoatsim_ref.so"))


def _check_line(line, n_gpus):
    d = json.loads(line)
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["n_gpus"] == n_gpus and d["unit"] == "params/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    return d


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built (run __graft_entry__.build())")
def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                          "--cpu-sample", SAMPLE], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = _check_line(lines[0], 1)
    assert d["steps"] == 2 and d["warmup"] == 1


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built (run __graft_entry__.build())")
def test_reference_arm_under_torchrun_prints_once():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "1", "--cpu-sample", SAMPLE],
                         cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    _check_line(lines[0], 2)
