"""The C++ facade (include/npcg/*.hpp) compiles against the C-ABI and links
libnpcg_b200.so (CPU suite); the reference-style program runs on a B200 (GPU
suite)."""
import subprocess
from pathlib import Path

import numpy as np
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


def _tridiag(n):
    """The facade test's user operator (TridiagOperator) as a dense matrix."""
    a = np.diag([2.0 + i / n for i in range(n)]) - np.eye(n, k=1) - np.eye(n, k=-1)
    return np.asfortranarray(a)


@pytest.mark.gpu
def test_facade_runs_on_b200(tmp_path, orc):
    exe = build_facade()
    dump = tmp_path / "facade.txt"
    r = subprocess.run([str(exe), str(dump)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade ok" in r.stdout
    got = {}
    for line in dump.read_text().splitlines():
        name, it, *xs = line.split()
        got[name] = (int(it), np.array([float(v) for v in xs]))
    # the user operator solved through the library vs the oracle on the same matrix
    n, mu = 200, 0.05
    op = orc.DenseOperator(_tridiag(n))
    b = np.cos(0.1 * np.arange(n))
    ref = orc.cg(op, mu, b, eta=1e-10, relative=True)
    it, x = got["user_cg_regularized"]
    assert abs(it - ref.iterations) <= 1
    assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
    approx = orc.randomized_nystrom(op, 20, orc.Rng(11))
    lam = got["user_lambda"][1]
    keep = approx.lam >= 1e-6 * approx.lam[0]
    assert np.max(np.abs(lam[keep] - approx.lam[keep]) / approx.lam[keep]) <= 1e-10
    pre = orc.build_preconditioner(approx, mu)
    ref2 = orc.nystrom_pcg(op, b, mu, pre, eta=1e-10, relative=True)
    it2, x2 = got["user_nystrom_pcg"]
    assert abs(it2 - ref2.iterations) <= 1
    assert np.linalg.norm(x2 - ref2.x) <= 1e-8 * np.linalg.norm(ref2.x)
    B = np.column_stack([np.sin(0.05 * (np.arange(n) + 1) * (j + 1)) for j in range(3)])
    ref3 = orc.block_nystrom_pcg(op, B, mu, pre, eta=1e-10, relative=True)
    it3, x3 = got["user_block_col1"]
    assert abs(it3 - ref3.iterations) <= 1
    assert np.linalg.norm(x3 - ref3.x[:, 1]) <= 1e-8 * np.linalg.norm(ref3.x[:, 1])
