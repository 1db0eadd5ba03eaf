"""bench.py keeps its contract (-m gpu): one JSON line with the required keys, on a small configuration."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"]


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_small_config():
    d = _run("--config", "game", "--steps", "1", "--warmup", "3", "--micro-rows", "16384", "--e2e-steps", "1",
             "--cpu-seconds", "1", "--no-next")
    for k in REQUIRED + ["e2e", "cpu_baseline"]:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.05 and r["achieved"] > 0
    assert d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert "workload" in d["config"]


def test_bench_reference_arm():
    d = _run("--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.parametrize("shard", ["vocab", "vocab-fused"])
def test_bench_vocab_shard_paths(shard):
    """The vocab-sharded step (gathered and K4-VPF) runs through bench.py at N = 1 with its own roofline line."""
    d = _run("--config", "game", "--shard", shard, "--steps", "1", "--warmup", "3", "--micro-rows", "16384",
             "--no-e2e", "--no-cpu-baseline", "--no-next")
    assert d["value"] > 0 and d["scaling"] == "strong" and d["gpu_launches"] > 0
    assert 0 < d["roofline"]["frac"] < 1.05
    assert ("BWD_VPF" in d["roofline"]["kernel"]) == (shard == "vocab-fused")
