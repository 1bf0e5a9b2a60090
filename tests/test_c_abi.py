"""The C-ABI boundary used from plain C (examples/c_abi_fill.c): it compiles
against include/sdrng.h + libsdrng.so with gcc here, and on a GPU it draws a
Shard(1) window and a fused dropout that match the host Philox entry point
element for element (no Python or torch on that path)."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

CUDA = "/usr/local/cuda"


def _build(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not on PATH")
    exe = tmp_path / "c_abi_fill"
    cmd = [gcc, "-O2", f"-I{ROOT}/include", f"-I{CUDA}/include", f"{ROOT}/examples/c_abi_fill.c",
           f"-L{ROOT}/paper_2509_07003_b200", "-lsdrng", f"-L{CUDA}/lib64", "-lcudart", "-lm", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_example_runs_bit_exact(tmp_path):
    exe = _build(tmp_path)
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = f"{ROOT}/paper_2509_07003_b200:{CUDA}/lib64:" + env.get("LD_LIBRARY_PATH", "")
    out = subprocess.run([str(exe)], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 mismatches" in out.stdout
