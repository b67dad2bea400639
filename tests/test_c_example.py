"""examples/fp_uniform.c: a plain C caller of the C-ABI.
CPU: it compiles and links against include/cyltomo_b200.h and the library.
GPU: it runs -- a uniform cylinder's projection equals its path lengths."""

import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA = Path("/usr/local/cuda")


def _build(tmp_path):
    lib = ROOT / "paper_2005_11976_b200" / "libcyltomo_b200.so"
    if not lib.exists():
        pytest.skip("library not built")
    exe = tmp_path / "fp_uniform"
    subprocess.run(["gcc", "-Wall", "-Werror", f"-I{ROOT / 'include'}", f"-I{CUDA / 'include'}",
                    str(ROOT / "examples" / "fp_uniform.c"), f"-L{lib.parent}", "-lcyltomo_b200",
                    f"-L{CUDA / 'lib64'}", "-lcudart", "-lm", "-o", str(exe)], check=True)
    return exe, {**os.environ, "LD_LIBRARY_PATH": f"{lib.parent}:{CUDA / 'lib64'}"}


def test_c_example_compiles_against_the_header(tmp_path):
    exe, _ = _build(tmp_path)
    assert exe.exists()


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe, env = _build(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
