"""The C ABI without Python: examples/c_api_step.c (masks -> advantages -> log-probs -> fused loss + dlogits on a
batch with a closed-form loss) and examples/c_api_batch_step.c (the same step batch-sharded over the library's NCCL
communicator) compile as plain C against include/otk.h and libotk.so (CPU), and run on the GPU (-m gpu) with the
closed-form loss, advantages, token count and zero-sum gradient rows."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path, name="c_api_step"):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    lib = os.path.join(ROOT, "paper_2601_07376_b200")
    if not os.path.exists(os.path.join(lib, "libotk.so")):
        pytest.skip("libotk.so not built")
    exe = str(tmp_path / name)
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", name + ".c"), "-o", exe, "-L", lib,
           "-lotk", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{lib}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_as_plain_c(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "-> ok" in r.stdout


def test_c_batch_example_compiles_as_plain_c(tmp_path):
    assert os.path.exists(_build(tmp_path, "c_api_batch_step"))


@pytest.mark.gpu
def test_c_batch_example_runs(tmp_path):
    """examples/c_api_batch_step.c: the batch-sharded step over the library's NCCL communicator, one process per
    GPU (P = 1 on a one-GPU box, P = 2 where two GPUs exist); the loss keeps its closed form on every P."""
    import torch
    exe = _build(tmp_path, "c_api_batch_step")
    for P in ([1, 2] if torch.cuda.device_count() >= 2 else [1]):
        r = subprocess.run([exe, str(P)], capture_output=True, text=True, timeout=180)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.count("-> ok") == P
