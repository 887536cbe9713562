"""GPU: read_edge_list (graph.cpp:152-200) — the GPU text parser against
the reference library's reader on the reference tests' IO cases (tests/test_graph.cpp:210-254)
and on randomized files (whitespace classes, comments, blank lines, CRLF, huge and
wrapping numbers, long lines crossing the parser's 256-byte segments, first-error reporting)."""
import gzip
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def td():
    from paper_1707_02000_b200 import trussdec
    return trussdec


def _write(path, text: str, gz=False):
    data = text.encode("latin-1")
    if gz:
        with gzip.open(path, "wb") as f:
            f.write(data)
    else:
        with open(path, "wb") as f:
            f.write(data)
    return str(path)


def _ours(td, path):
    try:
        return td.read_edge_list(path), None
    except RuntimeError as e:
        return None, str(e)


def _theirs(ref, path):
    try:
        return ref.read_edge_list(path), None
    except RuntimeError as e:
        return None, str(e)


def _same(td, ref, path):
    a, ea = _ours(td, path)
    b, eb = _theirs(ref, path)
    if eb is not None:
        assert ea is not None and ea.endswith(eb), (ea, eb)
    else:
        assert ea is None, ea
        assert a.dtype == np.uint64 and a.shape == b.shape and (a == b).all()
    return a, ea


def test_reference_io_case_comments_whitespace(td, ref, tmp_path):
    p = _write(tmp_path / "io.txt", "# comment\n% another\n 0 1 \n1\t2\n\n2 0\n")
    a, _ = _same(td, ref, p)
    assert a.tolist() == [[0, 1], [1, 2], [2, 0]]  # test_graph.cpp:218-219


def test_reference_io_case_gzip(td, ref, tmp_path):
    p = _write(tmp_path / "io.txt.gz", "0 1\n1 2\n2 0\n", gz=True)
    a, _ = _same(td, ref, p)
    assert a.tolist() == [[0, 1], [1, 2], [2, 0]]  # test_graph.cpp:221-228


def test_reference_io_case_errors(td, ref, tmp_path):
    p = _write(tmp_path / "bad.txt", "0 1\nfoo bar\n")
    _, e = _same(td, ref, p)
    assert ":2:" in e  # test_graph.cpp:230-235
    p = _write(tmp_path / "neg.txt", "0 -1\n")
    _, e = _same(td, ref, p)
    assert "negative vertex label" in e  # test_graph.cpp:237-241


def test_missing_file(td, tmp_path):
    with pytest.raises(RuntimeError, match="cannot open input file"):
        td.read_edge_list(str(tmp_path / "absent.txt"))


def test_empty_and_comment_only(td, ref, tmp_path):
    for i, text in enumerate(["", "\n\n\n", "# only\n% comments", "   \t\n"]):
        a, _ = _same(td, ref, _write(tmp_path / f"e{i}.txt", text))
        assert a.shape == (0, 2)


def test_write_read_round_trip(td, ref, oracle, tmp_path):
    """test_graph.cpp:247-254: write_edge_list ("%llu %llu\\n") then read gives the raw list."""
    raw = oracle.generate_er(40, 0.2, 11)
    text = "".join(f"{u} {v}\n" for u, v in raw.reshape(-1, 2).tolist())
    a, _ = _same(td, ref, _write(tmp_path / "rt.txt", text))
    assert (a == raw.reshape(-1, 2)).all()


@pytest.mark.parametrize("case", [
    "1 2",                     # no trailing newline
    "1 2\r\n3 4\r\n",          # CRLF
    "\v1\f2\v\n",              # every isspace class
    "18446744073709551615 0\n",             # u64 max
    "123456789012345678901234567890 7\n",  # wraps like the reference's v*10+d
    "  # indented comment\n5 6\n",
    "5 6 7\n",                 # trailing characters
    "5\n",                     # one number
    "5 x\n",
    "5 -6\n",
    "-5 6\n",
    "5 6 # comment after\n",
    "0x10 1\n",
    "1 2\n\n\n3 4\n bad\n",    # first error on line 6
    "1 2\n% x\n 3 4 \n7 8 9\n10 11\n",
])
def test_edge_cases_match_reference(td, ref, tmp_path, case):
    _same(td, ref, _write(tmp_path / "c.txt", case))


@pytest.mark.parametrize("seed", range(8))
def test_random_files_match_reference(td, ref, tmp_path, seed):
    rng = np.random.default_rng(seed)
    ws = [" ", "\t", "  ", " \t ", "\r", "\v", "\f"]
    lines = []
    for _ in range(int(rng.integers(1, 3000))):
        r = rng.random()
        if r < 0.05:
            lines.append(rng.choice(ws) * int(rng.integers(0, 3)))
        elif r < 0.1:
            lines.append(str(rng.choice(["#", "%", " #", "\t%"])) + "c" * int(rng.integers(0, 400)))
        elif r < 0.12:
            lines.append(" " * int(rng.integers(200, 900)) + "1 2")  # a line across segments
        else:
            a, b = (int(x) for x in rng.integers(0, 1 << 62, 2, dtype=np.int64))
            if rng.random() < 0.5:
                a, b = a % 1000, b % 1000
            lines.append(f"{rng.choice(ws)}{a}{rng.choice(ws)}{b}{rng.choice(['', ' ', '  ', '\t'])}")
    if seed % 4 == 3:  # plant one malformed line
        k = int(rng.integers(0, len(lines)))
        lines[k] = str(rng.choice(["7 8 9", "x 1", "1 -2", "3"]))
    text = "\n".join(lines) + ("\n" if seed % 2 else "")
    _same(td, ref, _write(tmp_path / "r.txt.gz" if seed % 3 == 0 else tmp_path / "r.txt", text, gz=seed % 3 == 0))


def test_large_file_many_segments(td, ref, tmp_path):
    rng = np.random.default_rng(7)
    e = rng.integers(0, 1 << 20, (200_000, 2))
    text = "".join(f"{u}\t{v}\n" for u, v in e.tolist())
    a, _ = _same(td, ref, _write(tmp_path / "big.txt", text))
    assert (a == e.astype(np.uint64)).all()


def test_read_canonicalize_truss_pipeline(td, ref, oracle, tmp_path):
    """The CLI's ingest path (trussdec.cpp: read_edge_list -> canonicalize -> truss) end to end
    on the GPU equals the reference pipeline."""
    raw = oracle.generate_rmat(9, 8, 3).reshape(-1, 2)
    p = _write(tmp_path / "g.txt", "".join(f"{u} {v}\n" for u, v in raw.tolist()))
    g = td.canonicalize(td.read_edge_list(p))
    r = ref.make_graph(2, 0, 0.0, 0, pairs=ref.read_edge_list(p))
    assert (g.n, g.m) == (r.n, r.m)
    assert (g.offsets == r.offsets).all() and (g.neighbors == r.neighbors).all()
    from oracle import Csr
    truss = td.truss_parallel(td.build_truss_graph(g), 1).result.truss
    assert (np.asarray(truss) == ref.truss_parallel(Csr(r.n, r.m, r.offsets, r.neighbors), 1).truss).all()
