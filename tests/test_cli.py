"""The `chebpr` CLI (reference: proj/tools/chebpr_main.cpp:63-249,
proj/src/csv.cpp:37-84).  Outputs are checked byte for byte against the reference's OWN
writers (oracle/_ref: write_edge_list, write_ranks_csv, write_*_trace_csv) on the same
graphs; exit codes against chebpr_main.cpp:239-248.  The reference's own CLI suite
(proj/tests/test_cli.cpp) and acceptance criterion 7 run against this binary in
tests/test_reference_suites.py."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "paper_2112_01743_b200", "bin", "chebpr")


def cli(*args, check=None):
    if not os.path.exists(CLI):
        pytest.skip("chebpr not built (make)")
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check is not None:
        assert p.returncode == check, (args, p.returncode, p.stderr)
    return p


def read(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize("argv,code", [
    ([], 1), (["frobnicate"], 1), (["--help"], 0), (["gen", "--help"], 0),
    (["gen", "--model", "ring", "--output", "x.el"], 1),          # --n required
    (["gen", "--model", "blob", "--n", "5", "--output", "x.el"], 1),
    (["gen", "--model", "gnp", "--n", "500", "--output", "x.el"], 1),  # no --p / --avg-deg
    (["gen", "--model", "gnp", "--n", "50", "--p", "0.1", "--avg-deg", "3", "--output", "x.el"], 1),
    (["gen", "--model", "regular", "--n", "7", "--k", "3", "--output", "x.el"], 1),
    (["gen", "--model", "ring", "--n", "abc", "--output", "x.el"], 1),
    (["run", "--algo", "nope", "--input", "x", "--eps", "1"], 1),
    (["run", "--algo", "cpaa", "--input", "g.el", "--eps", "1e-3", "--rounds", "5"], 1),
    (["run", "--algo", "cpaa", "--input", "g.el"], 1),            # no stopping rule
    (["run", "--algo", "cpaa", "--input", "g.el", "--keep-multi", "--dedup", "--rounds", "2"], 1),
    (["coeffs", "--c", "1.2"], 1),
    (["coeffs", "--c", "0.85", "--max-k", "0", "--quadrature-check", "--quad-tol", "1e-300"], 2),
    (["coeffs", "--bogus"], 1),
])
def test_exit_codes(tmp_path, argv, code):
    os.chdir(tmp_path)
    (tmp_path / "g.el").write_text("0 1\n1 2\n")
    cli(*argv, check=code)


@pytest.mark.parametrize("model,args,ref_args,comment", [
    ("gnp", ["--n", "500", "--p", "0.02", "--seed", "7"], ("gnp", 500, 0.02, 7), "chebpr gen model=gnp n=500 p=0.02 seed=7"),
    ("gnp", ["--n", "2000", "--avg-deg", "6", "--seed", "3"], ("gnp", 2000, 6 / 1999, 3), None),
    ("ring", ["--n", "4"], ("ring", 4), "chebpr gen model=ring n=4"),
    ("star", ["--n", "9"], ("star", 9), "chebpr gen model=star n=9"),
    ("regular", ["--n", "12", "--k", "3"], ("regular", 12, 3), "chebpr gen model=regular n=12 k=3"),
])
def test_gen_files_equal_reference_writer(tmp_path, reference, model, args, ref_args, comment):
    """gen writes exactly the bytes of the reference's generator + write_edge_list."""
    out = tmp_path / "a.el"
    p = cli("gen", "--model", model, *args, "--output", out, check=0)
    assert p.stdout == f"wrote {out}\n"
    kind = ref_args[0]
    e = getattr(reference, f"{kind}_edges")(*ref_args[1:])
    if comment is None:  # the reference CLI formats p with %.17g
        comment = f"chebpr gen model=gnp n={ref_args[1]} p={ref_args[2]:.17g} seed={ref_args[3]}"
    want = tmp_path / "b.el"
    reference.write_edges(e, str(want), comment)
    assert read(out) == read(want)


def test_gen_config_models_match_oracle(tmp_path, oracle):
    """The B200 additions: --model rmat / chung-lu write the BASELINE config generators."""
    out = tmp_path / "r.el"
    cli("gen", "--model", "rmat", "--scale", "10", "--edge-factor", "8", "--seed", "5", "--output", out, check=0)
    e = np.loadtxt(out, dtype=np.int64, comments="#")
    assert np.array_equal(e, oracle.rmat_edges(10, 8, 0.57, 0.19, 0.19, 5))
    out = tmp_path / "c.el"
    cli("gen", "--model", "chung-lu", "--n", "3000", "--draws", "9000", "--seed", "2", "--output", out, check=0)
    e = np.loadtxt(out, dtype=np.int64, comments="#")
    assert np.array_equal(e, oracle.chung_lu_edges(3000, 2.1, 2.0, 50000.0, 9000, 2))


def test_coeffs_table_matches_reference(reference):
    p = cli("coeffs", "--c", "0.85", "--max-k", "40", check=0)
    lines = p.stdout.splitlines()
    assert lines[0] == "k,c_k,err_bound_k" and len(lines) == 42
    table, _, _ = reference.coefficients(0.85, 40)
    for k in range(41):
        assert lines[k + 1] == f"{k},{table[k]:.17g},{reference.err_bound(0.85, k):.17g}"
    q = cli("coeffs", "--c", "0.85", "--max-k", "20", "--quadrature-check", check=0)
    assert q.stdout.splitlines()[0] == "k,c_k,err_bound_k,c_k_quadrature"
    assert float(q.stderr.split(":")[1]) <= 1e-9


def _gnp_file(tmp_path, reference, n=10000, p=0.001, seed=1):
    e = reference.gnp_edges(n, p, seed)
    path = tmp_path / "g.el"
    reference.write_edges(e, str(path), "g")
    return path, reference.build_graph(e)


@pytest.mark.gpu
@pytest.mark.parametrize("algo,stop", [("cpaa", ["--eps", "1e-10"]), ("cpaa", ["--rounds", "12"]),
                                        ("power", ["--rounds", "50"]), ("power", ["--eps", "1e-6"])])
def test_run_bitexact_csv_byte_identical_to_reference(tmp_path, reference, algo, stop):
    """run --mode bitexact: the ranks CSV is byte-identical to the reference's run + its
    write_ranks_csv, and the trace CSV identical except the elapsed_ms timing column."""
    g, rg = _gnp_file(tmp_path, reference)
    ranks, trace = tmp_path / "r.csv", tmp_path / "t.csv"
    p = cli("run", "--algo", algo, "--input", g, *stop, "--mode", "bitexact", "--output", ranks,
            "--trace", trace, check=0)
    assert p.stdout.startswith(f"n={rg.n} m={rg.m} algo={algo} rounds=")
    rranks, rtrace = tmp_path / "rr.csv", tmp_path / "rt.csv"
    kw = dict(rounds=int(stop[1])) if stop[0] == "--rounds" else dict(eps=float(stop[1]))
    rg.solve_to_csv(algo, ranks_path=str(rranks), trace_path=str(rtrace), **kw)
    assert read(ranks) == read(rranks)
    col = 4 if algo == "cpaa" else 2  # elapsed_ms

    def strip(path):
        return [",".join(f for i, f in enumerate(ln.split(",")) if i != col) for ln in read(path).decode().splitlines()]
    assert strip(trace) == strip(rtrace)


@pytest.mark.gpu
def test_run_fast_mode_within_bar_and_devices(tmp_path, reference):
    """--mode fast (the product kernel): ranks within 1e-12 of the reference's; the same
    bytes for every --parallelism (acceptance criterion 7's property)."""
    g, rg = _gnp_file(tmp_path, reference, n=50000, p=0.0002, seed=4)
    outs = []
    for k in (1, 2, 8):
        out = tmp_path / f"r{k}.csv"
        cli("run", "--algo", "cpaa", "--input", g, "--eps", "1e-10", "--mode", "fast", "--parallelism", k,
            "--device", 0, "--output", out, check=0)
        outs.append(read(out))
    assert outs[0] == outs[1] == outs[2]
    mine = np.loadtxt(tmp_path / "r1.csv", delimiter=",", skiprows=1)[:, 1]
    want = rg.run_cpaa(eps=1e-10).ranks
    assert np.max(np.abs(mine - want)) <= 1e-12
    f32 = tmp_path / "f32.csv"
    cli("run", "--algo", "cpaa", "--input", g, "--eps", "1e-10", "--precision", "32", "--output", f32, check=0)
    r32 = np.loadtxt(f32, delimiter=",", skiprows=1)[:, 1]
    assert np.sum(np.abs(r32 - want)) / np.sum(want) <= 1e-6


@pytest.mark.gpu
def test_run_errors_and_compare(tmp_path):
    g = tmp_path / "g.el"
    g.write_text("0 1\n1 x\n")
    p = cli("run", "--algo", "cpaa", "--input", g, "--eps", "1e-3", check=1)
    assert ":2:" in p.stderr
    g.write_text("0 1\n3 4\n")
    cli("run", "--algo", "cpaa", "--input", g, "--eps", "1e-3", check=1)           # vertex 2 isolated
    p = cli("run", "--algo", "cpaa", "--drop-isolated", "--input", g, "--eps", "1e-3", check=0)
    assert "dropped 1 isolated" in p.stderr
    mtx = tmp_path / "g.mtx"
    mtx.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 2\n")
    assert "n=3 m=2" in cli("run", "--algo", "cpaa", "--format", "mtx", "--input", mtx, "--rounds", "12", check=0).stdout
    cli("run", "--algo", "cpaa", "--input", tmp_path / "missing.el", "--eps", "1e-3", check=1)
    cli("run", "--algo", "cpaa", "--input", mtx, "--format", "mtx", "--eps", "1e-3", "--c", "1.5", check=1)
    k2 = tmp_path / "k2.el"
    k2.write_text("0 1\n")
    p = cli("compare", "--input", k2, "--eps", "1e-3", check=0)
    rows = p.stdout.splitlines()
    assert rows[0] == "algo,parallelism,rounds,err,l1,elapsed_ms" and len(rows) == 3
