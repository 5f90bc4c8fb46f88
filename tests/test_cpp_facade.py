"""The C++ facade (include/npcg/*.hpp) compiles against the C-ABI and links
libnpcg_b200.so (CPU suite); the reference-style program runs on a B200 (GPU
suite)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "facade_test.cpp"
LIBDIR = ROOT / "paper_2110_02820_b200"


def build_facade(tmp_path_factory=None) -> Path:
    out = LIBDIR / "build_obj" / "facade_test"
    out.parent.mkdir(exist_ok=True)
    cmd = ["/usr/bin/g++", "-std=c++20", "-O1", "-Wall", "-I", str(ROOT / "include"), str(SRC), "-o", str(out),
           "-L", str(LIBDIR), "-lnpcg_b200", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_facade_compiles_and_links():
    assert build_facade().exists()


@pytest.mark.gpu
def test_facade_runs_on_b200():
    exe = build_facade()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade ok" in r.stdout
