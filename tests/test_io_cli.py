"""File formats and the CLI (reference io.py, cli.py).

CPU tests mirror T/test_io.py and the failure paths of T/test_cli.py that
stop before any device work; the GPU tests run the commands end to end and
compare with the reference CLI's own outputs (tests/golden/cli.npz, made by
tests/golden/make_golden.py from the same seeded inputs).
"""

import csv
import hashlib

import numpy as np
import pytest

from conftest import golden, rel_l2
from paper_1903_02153_b200 import io as fio
from paper_1903_02153_b200.cli import main
from paper_1903_02153_b200.errors import FileFormatError


def _cli_inputs():
    gen = np.random.default_rng(44)
    return gen.random((3000, 3)), gen.standard_normal((3000, 2))


def _two_points(path):
    path.write_text("x,y,z,w1\n0.0,0.0,0.0,1.0\n2.0,0.0,0.0,1.0\n")


# ---------------------------------------------------------------------------
# formats (CPU)

def test_csv_and_binary_round_trips_are_bitwise(tmp_path):
    m = np.random.default_rng(77).standard_normal((40, 5))
    fio.write_matrix_csv(tmp_path / "m.csv", [f"c{i}" for i in range(5)], m)
    names, back = fio.read_matrix_csv(tmp_path / "m.csv")
    assert names == [f"c{i}" for i in range(5)] and np.array_equal(back, m)
    fio.write_matrix_binary(tmp_path / "m.bin", m)
    assert np.array_equal(fio.read_matrix_binary(tmp_path / "m.bin"), m)
    fio.write_matrix(tmp_path / "v.bin", np.array([1.0, 2.5, -3.0]))
    assert fio.read_matrix(tmp_path / "v.bin").shape == (3, 1)


def test_files_are_byte_identical_to_the_reference_writer(tmp_path):
    g = golden("cli")
    pts, w = _cli_inputs()
    fio.write_points_file(tmp_path / "src.csv", pts, w)
    fio.write_matrix_binary(tmp_path / "w.bin", w)
    assert hashlib.sha256((tmp_path / "src.csv").read_bytes()).hexdigest() == str(g["src_csv_sha"])
    assert hashlib.sha256((tmp_path / "w.bin").read_bytes()).hexdigest() == str(g["w_bin_sha"])


def test_points_files_with_and_without_weights(tmp_path):
    gen = np.random.default_rng(5)
    p, w = gen.random((12, 3)), gen.standard_normal((12, 2))
    for name in ("a.csv", "a.bin"):
        fio.write_points_file(tmp_path / name, p, w)
        p2, w2 = fio.read_points_file(tmp_path / name)
        assert np.array_equal(p2, p) and np.array_equal(w2, w)
        fio.write_points_file(tmp_path / name, p)
        assert fio.read_points_file(tmp_path / name)[1] is None


@pytest.mark.parametrize("text,line,frag", [
    ("x,y,z\n0.1,0.2,0.3\n0.4,oops,0.6\n", 3, "oops"),
    ("x,y,z\n0.1,0.2\n", 2, "expected 3 columns"),
    ("", 1, "missing header"),
    ("x,,z\n", 1, "empty column"),
])
def test_csv_errors_name_the_line(tmp_path, text, line, frag):
    (tmp_path / "bad.csv").write_text(text)
    with pytest.raises(FileFormatError) as err:
        fio.read_matrix_csv(tmp_path / "bad.csv")
    assert err.value.line == line and frag in str(err.value)


def test_binary_errors(tmp_path):
    (tmp_path / "short.bin").write_bytes(b"BFMM")
    with pytest.raises(FileFormatError, match="truncated"):
        fio.read_matrix_binary(tmp_path / "short.bin")
    fio.write_matrix_binary(tmp_path / "ok.bin", np.ones((3, 2)))
    raw = (tmp_path / "ok.bin").read_bytes()
    (tmp_path / "magic.bin").write_bytes(b"NOTAMATX" + raw[8:])
    with pytest.raises(FileFormatError, match="bad magic"):
        fio.read_matrix_binary(tmp_path / "magic.bin")
    (tmp_path / "cut.bin").write_bytes(raw[:-8])
    with pytest.raises(FileFormatError, match="expected"):
        fio.read_matrix_binary(tmp_path / "cut.bin")
    fio.write_matrix_binary(tmp_path / "two.bin", np.ones((3, 2)))
    with pytest.raises(FileFormatError, match="at least 3 columns"):
        fio.read_points_file(tmp_path / "two.bin")
    (tmp_path / "hdr.csv").write_text("a,b,c\n1,2,3\n")
    with pytest.raises(FileFormatError, match="x,y,z"):
        fio.read_points_file(tmp_path / "hdr.csv")


# ---------------------------------------------------------------------------
# CLI failure paths that stop before device work (CPU)

def test_usage_errors_exit_two(tmp_path):
    with pytest.raises(SystemExit) as e:
        main(["evaluate", "--kernel", "laplacian"])
    assert e.value.code == 2
    _two_points(tmp_path / "p.csv")
    with pytest.raises(SystemExit) as e:
        main(["evaluate", "--kernel", "laplacian", "--sources", str(tmp_path / "p.csv"),
              "--synthetic", "10"])
    assert e.value.code == 2
    with pytest.raises(SystemExit):
        main(["evaluate", "--synthetic", "10"])


def test_runtime_errors_exit_one(tmp_path, capsys):
    assert main(["evaluate", "--kernel", "nosuch", "--synthetic", "10"]) == 1
    assert "error:" in capsys.readouterr().err
    (tmp_path / "bad.csv").write_text("x,y,z,w1\n0.1,0.2,0.3,1.0\n0.4,oops,0.6,1.0\n")
    assert main(["evaluate", "--kernel", "laplacian", "--sources", str(tmp_path / "bad.csv"),
                 "--levels", "2"]) == 1
    err = capsys.readouterr().err
    assert "line 3" in err and "oops" in err
    _two_points(tmp_path / "p.csv")
    assert main(["evaluate", "--kernel", "laplacian", "--sources", str(tmp_path / "p.csv"),
                 "--center", "0,0,0"]) == 1
    assert "--length" in capsys.readouterr().err
    assert main(["bench", "--mode", "convergence", "--kernel", "laplacian",
                 "--n", "200000"]) == 1
    assert "guard" in capsys.readouterr().err


# ---------------------------------------------------------------------------
# end to end on the GPU, against the reference CLI's outputs

gpu = pytest.mark.gpu


def _rows(path):
    with open(path, newline="") as fh:
        return list(csv.DictReader(fh))


@gpu
def test_evaluate_files_matches_reference_cli(tmp_path, capsys):
    g = golden("cli")
    pts, w = _cli_inputs()
    fio.write_points_file(tmp_path / "src.csv", pts, w)
    out = tmp_path / "phi.bin"
    assert main(["evaluate", "--kernel", "exponential", "--sources", str(tmp_path / "src.csv"),
                 "--levels", "3", "--order", "4", "--eps", "1e-6",
                 "--cache-dir", str(tmp_path / "cache"), "--out", str(out)]) == 0
    assert rel_l2(fio.read_matrix(out), g["eval_phi"]) < 1e-10
    text = capsys.readouterr().out
    # same report lines as the reference (the TS client parses "operator table")
    ref = str(g["eval_stdout"]).splitlines()
    assert text.splitlines()[0] == ref[0]
    import re
    pat = r"operator table\s+([0-9.eE+-]+) s \(([\d,]+) bytes\)"
    assert re.search(pat, text).group(2) == re.search(pat, str(g["eval_stdout"])).group(2)
    near = r"\(([\d,]+) near pairs\)"
    assert re.findall(near, text) == re.findall(near, str(g["eval_stdout"]))


@gpu
def test_synthetic_matches_reference_and_is_reproducible(tmp_path):
    g = golden("cli")
    args = ["evaluate", "--kernel", "gaussian", "--synthetic", "2000", "--seed", "9",
            "--order", "3", "--levels", "2", "--cache-dir", str(tmp_path / "cache")]
    assert main(args + ["--out", str(tmp_path / "a.bin")]) == 0
    assert main(args + ["--out", str(tmp_path / "b.bin")]) == 0
    assert (tmp_path / "a.bin").read_bytes() == (tmp_path / "b.bin").read_bytes()
    assert rel_l2(fio.read_matrix(tmp_path / "a.bin"), g["syn_phi"]) < 1e-10


@gpu
def test_two_point_inverse_distance(tmp_path, capsys):
    _two_points(tmp_path / "p.csv")
    out = tmp_path / "phi.csv"
    assert main(["evaluate", "--kernel", "laplacian", "--sources", str(tmp_path / "p.csv"),
                 "--length", "2.0", "--center", "1.0,0.0,0.0", "--levels", "2", "--order", "5",
                 "--cache-dir", str(tmp_path / "cache"), "--out", str(out)]) == 0
    phi = fio.read_matrix(out)
    assert phi.shape == (2, 1) and np.all(np.abs(phi - 0.5) < 1e-3)
    assert "near pairs" in capsys.readouterr().out


@gpu
def test_precompute_only_and_domain_errors(tmp_path, capsys):
    assert main(["evaluate", "--kernel", "gaussian", "--synthetic", "100", "--levels", "2",
                 "--order", "3", "--precompute-only", "--cache-dir", str(tmp_path / "c")]) == 0
    out = capsys.readouterr().out
    assert "operator table" in out and "first potentials" not in out
    _two_points(tmp_path / "p.csv")
    assert main(["evaluate", "--kernel", "laplacian", "--sources", str(tmp_path / "p.csv"),
                 "--length", "1.0", "--levels", "2", "--cache-dir", str(tmp_path / "c")]) == 1
    assert "error:" in capsys.readouterr().err


@gpu
def test_separate_weights_and_binary_targets(tmp_path):
    gen = np.random.default_rng(3)
    fio.write_points_file(tmp_path / "src.csv", gen.random((60, 3)))
    fio.write_matrix(tmp_path / "w.bin", gen.standard_normal((60, 2)))
    fio.write_points_file(tmp_path / "tgt.bin", gen.random((20, 3)))
    assert main(["evaluate", "--kernel", "exponential", "--sources", str(tmp_path / "src.csv"),
                 "--weights", str(tmp_path / "w.bin"), "--targets", str(tmp_path / "tgt.bin"),
                 "--levels", "2", "--order", "4", "--cache-dir", str(tmp_path / "c"),
                 "--out", str(tmp_path / "phi.bin")]) == 0
    assert fio.read_matrix(tmp_path / "phi.bin").shape == (20, 2)


@gpu
def test_bench_convergence_matches_reference_errors(tmp_path):
    g = golden("cli")
    out = tmp_path / "rows.csv"
    assert main(["bench", "--mode", "convergence", "--kernel", "laplacian", "--n", "400",
                 "--orders", "2,4", "--eps", "1e-8", "--cache-dir", str(tmp_path / "c"),
                 "--out", str(out)]) == 0
    rows = _rows(out)
    assert [r["scheme"] for r in rows] == list(g["conv_scheme"])
    assert [int(r["order"]) for r in rows] == list(g["conv_order"])
    err = np.array([float(r["error"]) for r in rows])
    # the error is ||phi - direct|| / ||direct||: phi within 1e-10 of the
    # reference moves it by far less than this
    assert np.allclose(err, g["conv_error"], rtol=1e-6, atol=0)
    for s in ("chebyshev", "uniform"):
        e = [float(r["error"]) for r in rows if r["scheme"] == s]
        assert e[1] < e[0]


@gpu
def test_bench_nscaling_and_threads(tmp_path, capsys):
    out = tmp_path / "n.csv"
    assert main(["bench", "--mode", "nscaling", "--kernel", "exponential", "--sizes",
                 "500,4000", "--order", "3", "--cache-dir", str(tmp_path / "c"),
                 "--out", str(out)]) == 0
    rows = _rows(out)
    assert len(rows) == 2 and rows[0]["slope"] == rows[1]["slope"]
    assert np.isfinite(float(rows[0]["slope"])) and float(rows[0]["direct_seconds"]) > 0
    assert "slope" in capsys.readouterr().out
    out = tmp_path / "t.csv"
    assert main(["bench", "--mode", "threads", "--kernel", "laplacian", "--n", "2000",
                 "--thread-counts", "1,2", "--order", "3", "--cache-dir", str(tmp_path / "c"),
                 "--out", str(out)]) == 0
    rows = _rows(out)
    assert [r["threads"] for r in rows] == ["1", "2"] and float(rows[0]["speedup"]) == 1.0
    assert "physical cores" in capsys.readouterr().out


@gpu
def test_bench_randsvd_matches_reference_eigs(tmp_path):
    g = golden("cli")
    eigs = tmp_path / "eigs.bin"
    out = tmp_path / "r.csv"
    assert main(["bench", "--mode", "randsvd", "--kernel", "gaussian", "--n", "300", "--rank",
                 "10", "--oversample", "5", "--power-iters", "2", "--levels", "2",
                 "--cache-dir", str(tmp_path / "c"), "--eigs-out", str(eigs),
                 "--out", str(out)]) == 0
    st = fio.read_matrix(eigs)
    assert st.shape == (301, 10)
    assert rel_l2(st[0], g["randsvd_eigs"][0]) < 1e-9
    vecs, ref = st[1:], g["randsvd_eigs"][1:]
    assert np.all(np.abs(np.abs(np.sum(vecs * ref, axis=0)) - 1.0) < 1e-8)
    row = _rows(out)[0]
    assert float(row["error"]) < 1e-3 and int(row["matvec_columns"]) == 4 * 15
