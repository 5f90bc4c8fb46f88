"""Matrix ingestion: the reference's io_test.cpp KATs
(proj/tests/io_test.cpp:29-190) against the Python mirror, and the C++
facade's npcg::io compiled and run (host only: CPU suite)."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2110_02820_b200 import matrix_io as io

ROOT = Path(__file__).resolve().parents[1]


def put(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_matrix_market_symmetric_mirrored(tmp_path):  # io_test.cpp:29-40
    p = put(tmp_path, "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2.0\n2 1 1.0\n2 2 2.0\n")
    assert np.array_equal(io.load_matrix(p, "matrix-market"), [[2, 1], [1, 2]])


def test_matrix_market_general_verbatim(tmp_path):  # :42-56
    p = put(tmp_path, "gen.mtx", "%%MatrixMarket matrix coordinate real general\n% a comment line\n2 3 2\n1 2 5.0\n"
                                 "2 1 -1.0\n")
    assert np.array_equal(io.load_matrix(p, "matrix-market"), [[0, 5, 0], [-1, 0, 0]])


def test_matrix_market_failures_carry_line(tmp_path):  # :58-100
    p = put(tmp_path, "count.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1.0\n")
    with pytest.raises(RuntimeError, match="expected 3 entries, found 2") as e:
        io.load_matrix(p, "matrix-market")
    assert ":4:" in str(e.value)
    for name, text in (("empty.mtx", ""),
                       ("range.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n"),
                       ("upper.mtx", "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n")):
        with pytest.raises(RuntimeError):
            io.load_matrix(put(tmp_path, name, text), "matrix-market")
    with pytest.raises(RuntimeError):
        io.load_matrix(str(tmp_path / "nope.mtx"), "matrix-market")


def test_csv_strict(tmp_path):  # :102-128
    assert np.array_equal(io.load_matrix(put(tmp_path, "ok.csv", "1.5,2\n3,4\n"), "csv-dense"), [[1.5, 2], [3, 4]])
    with pytest.raises(RuntimeError, match=":2:"):
        io.load_matrix(put(tmp_path, "bad.csv", "1,2\n3,x\n"), "csv-dense")
    for name, text in (("ragged.csv", "1,2\n3\n"), ("empty.csv", "")):
        with pytest.raises(RuntimeError):
            io.load_matrix(put(tmp_path, name, text), "csv-dense")


def test_round_trips(tmp_path):  # :130-162
    from oracle import oracle as orc
    rng = orc.Rng(11)
    a = rng.gaussian_matrix(10, 10)
    io.save_matrix(str(tmp_path / "rt.raw"), a, "raw-f64")
    assert np.array_equal(io.load_matrix(str(tmp_path / "rt.raw"), "raw-f64"), a)  # bitwise
    b = rng.gaussian_matrix(5, 4)
    io.save_matrix(str(tmp_path / "rt.csv"), b, "csv-dense")
    assert np.array_equal(io.load_matrix(str(tmp_path / "rt.csv"), "csv-dense"), b)
    g = rng.gaussian_matrix(6, 6)
    s = g + g.T
    io.save_matrix(str(tmp_path / "rt.mtx"), s, "matrix-market")
    assert "symmetric" in (tmp_path / "rt.mtx").read_text().splitlines()[0]
    assert np.array_equal(io.load_matrix(str(tmp_path / "rt.mtx"), "matrix-market"), s)
    r = rng.gaussian_matrix(4, 3)
    io.save_matrix(str(tmp_path / "rt_gen.mtx"), r, "matrix-market")
    assert np.array_equal(io.load_matrix(str(tmp_path / "rt_gen.mtx"), "matrix-market"), r)


def test_vector_names_symmetry(tmp_path):  # :164-200
    assert np.array_equal(io.load_vector(put(tmp_path, "c.csv", "1\n2\n3\n"), "csv-dense"), [1, 2, 3])
    with pytest.raises(RuntimeError):
        io.load_vector(put(tmp_path, "w.csv", "1,2\n3,4\n"), "csv-dense")
    for n in io.FORMATS:
        assert io.format_name(io.parse_format(n)) == n
    with pytest.raises(ValueError):
        io.parse_format("hdf5")
    with pytest.raises(RuntimeError, match="solve: matrix is not symmetric"):
        io.require_symmetric([[1, 2], [2.5, 1]], "solve")
    with pytest.raises(RuntimeError, match="solve: matrix must be square"):
        io.require_symmetric(np.zeros((2, 3)), "solve")


def test_cpp_facade_io(tmp_path):
    exe = tmp_path / "io_test"
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-Wall", "-I", str(ROOT / "include"),
                        str(ROOT / "tests" / "cpp" / "io_test.cpp"), "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "io ok" in r.stdout, r.stdout + r.stderr
