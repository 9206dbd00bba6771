"""Graph ingest parity: the device loaders (cheb_graph_load_edge_list / _matrix_market,
csrc/ingest.cu) against the reference's own loaders (graph_io.cpp:50-174, compiled
unmodified into oracle/_ref) on the same files: identical CSR, GraphStats, and on failure
the same error type and message (which names the first failing line)."""
import os
import random

import numpy as np
import pytest

STATUS_TO_API = {1: "ValidationError", 4: "ValueError", 5: "CapacityError", 8: "ParseError"}


# ---------------------------------------------------------------------------------------
# corpus
def _edge_cases():
    yield "plain", "0 1\n1 2\n2 0\n"
    yield "no_final_newline", "0 1\n1 2\n2 0"
    yield "comments_blanks", "# header\n\n0 1\n   \n\t# indented comment\n1 2\n2 0\n"
    yield "crlf", "0 1\r\n1 2\r\n2 0\r\n"
    yield "tabs_spaces", "0\t1\n 1   2 \n\t2\t0\t\n"
    yield "duplicates_loops", "0 1\n1 0\n0 1\n1 1\n1 2\n2 0\n"
    yield "leading_zeros", "000 001\n01 2\n2 0\n"
    yield "minus_zero", "-0 1\n1 2\n2 -0\n"
    yield "big_ids_isolated", "0 5\n5 1\n"
    yield "bad_token", "0 1\n1 x\n2 0\n"
    yield "negative", "0 1\n1 -2\n"
    yield "plus_sign", "0 1\n+1 2\n"
    yield "lone_minus", "0 1\n- 2\n"
    yield "one_id", "0 1\n7\n"
    yield "three_ids", "0 1\n1 2 3\n"
    yield "trailing_hash", "0 1 # edge\n"
    yield "overflow", "0 1\n99999999999999999999 1\n"
    yield "first_of_two_errors", "0 1\nbad\n1 2\nworse\n"
    yield "error_on_last_line_unterminated", "0 1\n1 2\n2 zz"
    yield "only_comments", "# nothing\n#\n"
    yield "empty", ""
    yield "just_newline", "\n"
    yield "float_id", "0 1.5\n"
    yield "hex", "0x1 2\n"


def _mm(field="pattern", sym="general", body="", size="3 3 {n}", comments=""):
    lines = body.strip("\n").split("\n") if body.strip("\n") else []
    head = f"%%MatrixMarket matrix coordinate {field} {sym}\n{comments}{size.format(n=len(lines))}\n"
    return head + ("\n".join(lines) + "\n" if lines else "")


def _mm_cases():
    yield "sym_pattern", _mm(sym="symmetric", body="2 1\n3 2\n3 1\n")
    yield "general_pattern", _mm(body="1 2\n2 1\n2 3\n3 2\n")
    yield "general_real", _mm("real", body="1 2 0.5\n2 1 -1e-3\n2 3 4\n3 2 5.\n")
    yield "real_forms", _mm("real", "symmetric", body="2 1 .5\n3 2 -0.25E+2\n3 1 7e\n".replace(" 7e", " 7"))
    yield "real_exp_rollback", _mm("real", "symmetric", body="2 1 7e\n")  # 'e' not consumed -> trailing
    yield "real_inf", _mm("real", "symmetric", body="2 1 inf\n3 2 -Infinity\n3 1 nan\n")
    yield "real_nanparen", _mm("real", "symmetric", body="2 1 nan(abc)\n3 1 1\n3 2 1\n")
    yield "real_overflow", _mm("real", "symmetric", body="2 1 1\n3 2 1e400\n3 1 1\n")
    yield "real_underflow", _mm("real", "symmetric", body="2 1 1e-400\n3 2 1\n3 1 1\n")
    yield "real_subnormal", _mm("real", "symmetric", body="2 1 4e-320\n3 2 1\n3 1 1\n")
    yield "real_big_ok", _mm("real", "symmetric", body="2 1 1.7e308\n3 2 1\n3 1 1\n")
    yield "real_zero_huge_exp", _mm("real", "symmetric", body="2 1 0e99999\n3 2 1\n3 1 1\n")
    yield "real_many_digits", _mm("real", "symmetric", body="2 1 " + "1" * 500 + "\n3 2 1\n3 1 1\n")
    yield "missing_weight", _mm("real", "symmetric", body="2 1\n")
    yield "malformed_weight", _mm("real", "symmetric", body="2 1 x\n")
    yield "weight_dot", _mm("real", "symmetric", body="2 1 .\n")
    yield "weight_plus", _mm("real", "symmetric", body="2 1 +1\n")
    yield "uncertain_then_error", _mm("real", "symmetric", body="2 1 1e400\n3 x 1\n3 1 1\n")
    yield "error_then_uncertain", _mm("real", "symmetric", body="2 x 1\n3 2 1e400\n3 1 1\n")
    yield "trailing", _mm(sym="symmetric", body="2 1 9\n")
    yield "out_of_range", _mm(sym="symmetric", body="2 1\n4 1\n")
    yield "zero_index", _mm(sym="symmetric", body="0 1\n")
    yield "malformed_entry", _mm(sym="symmetric", body="2\n")
    yield "comment_in_entries", _mm(sym="symmetric", body="2 1\n% no\n3 1\n")
    yield "blank_entry", _mm(sym="symmetric", body="2 1\n\n3 1\n")
    yield "too_few", "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 5\n2 1\n3 2\n"
    yield "extra_lines_ignored", "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 2\ngarbage\n"
    yield "size_comments", _mm(sym="symmetric", body="2 1\n3 2\n", comments="% a\n\n   % b\n")
    yield "not_symmetric", _mm(body="1 2\n2 3\n3 2\n")
    yield "not_symmetric_symmetrize", _mm(body="1 2\n2 3\n3 2\n")
    yield "general_diag", _mm(body="1 1\n1 2\n2 1\n2 3\n3 2\n")
    yield "nonsquare", "%%MatrixMarket matrix coordinate pattern general\n3 4 0\n"
    yield "bad_banner", "%%MatrixMarkt matrix coordinate pattern general\n3 3 0\n"
    yield "array_format", "%%MatrixMarket matrix array real general\n3 3\n"
    yield "complex_field", "%%MatrixMarket matrix coordinate complex general\n3 3 0\n"
    yield "skew", "%%MatrixMarket matrix coordinate pattern skew-symmetric\n3 3 0\n"
    yield "upper_case_banner", "%%MatrixMarket MATRIX Coordinate PATTERN Symmetric\n3 3 2\n2 1\n3 2\n"
    yield "missing_size", "%%MatrixMarket matrix coordinate pattern general\n% only comments\n"
    yield "malformed_size", "%%MatrixMarket matrix coordinate pattern general\n3 3\n"
    yield "empty_mm", ""
    yield "declared_isolated", "%%MatrixMarket matrix coordinate pattern symmetric\n5 5 2\n2 1\n3 2\n"
    yield "crlf_mm", _mm(sym="symmetric", body="2 1\r\n3 2\r\n3 1\r\n")
    yield "no_final_newline_mm", _mm(sym="symmetric", body="2 1\n3 2\n3 1\n").rstrip("\n")


OPTS = {
    "isolated": dict(drop_isolated=True),
    "multi": dict(dedup=False),
    "symmetrize": dict(symmetrize=True),
}


def _cases():
    for name, text in _edge_cases():
        yield f"el-{name}", "edges", text, {}
    for name, text in _mm_cases():
        opts = dict(symmetrize=True) if name.endswith("_symmetrize") else {}
        yield f"mm-{name}", "mm", text, opts
    yield "el-drop-isolated", "edges", "0 5\n5 1\n", dict(drop_isolated=True)
    yield "el-multi", "edges", "0 1\n1 0\n0 1\n1 1\n1 2\n2 0\n", dict(dedup=False)
    yield "mm-declared-drop", "mm", "%%MatrixMarket matrix coordinate pattern symmetric\n5 5 2\n2 1\n3 2\n", \
        dict(drop_isolated=True)


CASES = list(_cases())


def _ref_outcome(reference, path, fmt, opts):
    from oracle import OracleError
    try:
        g, st = reference.load(path, fmt, **opts)
    except OracleError as e:
        return ("error", STATUS_TO_API.get(e.code, str(e.code)), e.msg)
    c = g.csr()
    return ("ok", c.offsets.copy(), c.neighbors.copy(), c.degrees.copy(), st)


def _our_outcome(cheb, path, fmt, opts, text=None):
    o = cheb.LoadOptions(**opts)
    try:
        if text is not None:
            lg = cheb.parse_text(text, fmt, name=path, opts=o)
        elif fmt == "edges":
            lg = cheb.load_edge_list(path, o)
        else:
            lg = cheb.load_matrix_market(path, o)
    except (cheb.Error, ValueError) as e:
        return ("error", type(e).__name__, str(e))
    g, s = lg.graph, lg.stats
    st = dict(n=s.n, m=s.m, min_degree=s.min_degree, max_degree=s.max_degree, self_loops=s.self_loops,
              duplicates_removed=s.duplicates_removed, isolated_dropped=s.isolated_dropped,
              avg_degree=s.avg_degree)
    return ("ok", g.offsets, g.neighbors, g.degrees, st)


def _same(a, b):
    assert a[0] == b[0], (a, b)
    if a[0] == "error":
        assert a[1:] == b[1:], (a, b)
        return
    for x, y in zip(a[1:4], b[1:4]):
        assert np.array_equal(np.asarray(x, dtype=np.int64), np.asarray(y, dtype=np.int64))
    assert a[4] == b[4]


# ---------------------------------------------------------------------------------------
def test_corpus_reference_known_answers(reference, tmp_path):
    """CPU: the reference's own loader on the corpus (pins the expectations the GPU tests
    compare against) — e.g. the ':2:' line-number message of test_graph.cpp:185."""
    from oracle import OracleError
    p = tmp_path / "bad.txt"
    p.write_text("0 1\nx y\n")
    with pytest.raises(OracleError) as e:
        reference.load(str(p))
    assert ":2:" in e.value.msg and e.value.code == 8
    n_ok = n_err = 0
    for name, fmt, text, opts in CASES:
        f = tmp_path / name
        f.write_bytes(text.encode())
        out = _ref_outcome(reference, str(f), fmt, opts)
        n_ok += out[0] == "ok"
        n_err += out[0] == "error"
    assert n_ok >= 20 and n_err >= 30


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_device_loader_matches_reference(cheb, reference, tmp_path, case):
    name, fmt, text, opts = case
    f = tmp_path / name
    f.write_bytes(text.encode())
    ref = _ref_outcome(reference, str(f), fmt, opts)
    _same(_our_outcome(cheb, str(f), fmt, opts), ref)
    _same(_our_outcome(cheb, str(f), fmt, opts, text=text.encode()), ref)  # in-memory variant


def _mutate(rng, text):
    alphabet = "0123456789 \t\r\n#%-+.eExinf"
    s = list(text)
    for _ in range(rng.randint(1, 3)):
        op = rng.randrange(3)
        pos = rng.randrange(len(s) + 1)
        if op == 0:
            s.insert(pos, rng.choice(alphabet))
        elif op == 1 and s:
            del s[min(pos, len(s) - 1)]
        elif s:
            s[min(pos, len(s) - 1)] = rng.choice(alphabet)
    return "".join(s)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["edges", "mm"])
def test_device_loader_fuzz(cheb, reference, tmp_path, fmt):
    """Random single-character mutations of valid files: same verdict, message and CSR."""
    rng = random.Random(7 if fmt == "edges" else 11)
    if fmt == "edges":
        base = "".join(f"{i} {(i * 7 + 3) % 40}\n" for i in range(40))
    else:
        base = _mm("real", "general", body="".join(
            f"{i} {j} {rng.choice(['1', '0.5', '-2e3', '7.', '.25'])}\n"
            for i in range(1, 21) for j in (i % 20 + 1, (i + 18) % 20 + 1) if True), size="20 20 {n}")
        # make it symmetric: add mirrors
        lines = base.split("\n")
        head, body = lines[:2], [ln for ln in lines[2:] if ln]
        mirrored = body + [f"{ln.split()[1]} {ln.split()[0]} {ln.split()[2]}" for ln in body]
        base = f"{head[0]}\n20 20 {len(mirrored)}\n" + "\n".join(mirrored) + "\n"
    f = tmp_path / "fuzz"
    for it in range(150):
        text = _mutate(rng, base)
        f.write_bytes(text.encode())
        _same(_our_outcome(cheb, str(f), fmt, {}), _ref_outcome(reference, str(f), fmt, {}))


@pytest.mark.gpu
def test_device_loader_large_edge_list(cheb, reference, tmp_path):
    """~1.2M lines with mixed blanks, comments and CRLF: bit-exact CSR and stats."""
    rng = np.random.default_rng(5)
    E = 1_200_000
    a = rng.integers(0, 200_000, E)
    b = rng.integers(0, 200_000, E)
    seps = np.array([" ", "\t", "  ", " \t "])[rng.integers(0, 4, E)]
    ends = np.array(["\n", "\r\n", " \n"])[rng.integers(0, 3, E)]
    rows = [f"{x}{s}{y}{t}" for x, y, s, t in zip(a.tolist(), b.tolist(), seps.tolist(), ends.tolist())]
    for k in range(0, E, 5000):
        rows[k] = "# comment " + str(k) + "\n" + rows[k]
    f = tmp_path / "big.txt"
    f.write_text("".join(rows))
    _same(_our_outcome(cheb, str(f), "edges", dict(drop_isolated=True)),
          _ref_outcome(reference, str(f), "edges", dict(drop_isolated=True)))


@pytest.mark.gpu
def test_device_loader_huge_id_is_capacity_error(cheb, tmp_path):
    """An id of 2^63-1 overflows the reference's n = max id + 1 (graph.cpp:25-29; the
    reference crashes); the device path reports CapacityError (int32 column ids)."""
    f = tmp_path / "huge.txt"
    f.write_text("0 9223372036854775807\n")
    with pytest.raises(cheb.CapacityError):
        cheb.load_edge_list(str(f))


@pytest.mark.gpu
def test_loaded_graph_solves_like_built_graph(cheb, tmp_path):
    """A file loaded on the device solves bitwise like the same edges built from memory."""
    edges = np.array([[i, (i * 13 + 5) % 500] for i in range(500)] + [[i, i + 1] for i in range(499)])
    f = tmp_path / "g.txt"
    f.write_text("".join(f"{x} {y}\n" for x, y in edges))
    dg, st = cheb.load_device_graph(str(f))
    dg2, _ = cheb.build_device_graph(edges)
    cfg = cheb.SolverConfig(eps=1e-10)
    r1, r2 = cheb.run_cpaa(dg, cfg), cheb.run_cpaa(dg2, cfg)
    assert np.array_equal(r1.ranks, r2.ranks)
    assert st.n == 500 and st.self_loops == 0


@pytest.mark.gpu
def test_loader_errors(cheb, tmp_path):
    with pytest.raises(cheb.ParseError, match="cannot open"):
        cheb.load_edge_list(str(tmp_path / "missing.txt"))
    with pytest.raises(cheb.ParseError, match="cannot open"):
        cheb.load_matrix_market(str(tmp_path / "missing.mtx"))
    import ctypes as C
    from paper_2112_01743_b200 import _lib as L
    h, st = C.c_void_p(), L.cheb_graph_stats()
    o = L.cheb_load_opts()
    L.load().cheb_load_opts_default(C.byref(o))
    assert L.load().cheb_graph_parse_text(b"0 1\n", 4, 7, b"x", C.byref(o), C.byref(h), C.byref(st)) == 4  # format
