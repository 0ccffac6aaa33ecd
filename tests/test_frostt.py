"""FROSTT text I/O: libhbk's threaded C++ parser/writer against
the reference's known-answer tests (test_coo.py:26-95) and a NumPy
restatement of parse_frostt (coo.py:117-184).  Host only: no GPU needed."""
from __future__ import annotations

import io

import numpy as np
import pytest

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200 import ParseError, load_frostt, parse_frostt, save_frostt, write_frostt


def _entries(t):
    return {tuple(int(i) for i in r): float(v) for r, v in zip(t.indices, t.values)}


# reference known answers, test_coo.py:26-95
def test_parse_basic_dims_inferred():
    t = parse_frostt("1 1 1 2.0\n2 3 1 1.5")
    assert t.dims == (2, 3, 1)
    assert _entries(t) == {(0, 0, 0): 2.0, (1, 2, 0): 1.5}


def test_parse_comments_blank_lines_order4():
    t = parse_frostt("# comment\n\n1 1 1 1 4.0\n")
    assert t.order == 4 and _entries(t) == {(0, 0, 0, 0): 4.0}


def test_parse_wrong_field_count_reports_line():
    with pytest.raises(ParseError) as exc:
        parse_frostt("1 1 1 1.0\n1 2\n")
    assert exc.value.line == 2


def test_parse_non_numeric_reports_line():
    with pytest.raises(ParseError) as exc:
        parse_frostt("1 1 1 1.0\n1 x 1 2.0\n")
    assert exc.value.line == 2


@pytest.mark.parametrize("text", ["1 1 1 1.0\n1 1 1 1 1.0\n", "0 1 1 1.0\n", "1 1 1.0\n", "1 1 1 abc\n"])
def test_parse_errors(text):
    with pytest.raises(ParseError):
        parse_frostt(text)


def test_parse_empty_input():
    with pytest.raises(ParseError) as exc:
        parse_frostt("# nothing\n\n")
    assert exc.value.line is None


def test_parse_with_dims():
    t = parse_frostt("1 1 1 1.0\n", dims=(4, 4, 4))
    assert t.dims == (4, 4, 4)
    with pytest.raises(ParseError):
        parse_frostt("3 1 1 1.0\n", dims=(2, 4, 4))
    with pytest.raises(ValueError):
        parse_frostt("1 1 1.0\n", dims=(2, 4))


def test_duplicates_kept_as_written():
    t = parse_frostt("1 1 1 1.0\n1 1 1 2.0\n")
    assert t.nnz == 2 and list(t.values) == [1.0, 2.0]


def _reference_parse(text):
    """NumPy restatement of coo.py:117-184 (the oracle for bigger inputs)."""
    idx, vals = [], []
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        idx.append([int(x) - 1 for x in tok[:-1]])
        vals.append(float(tok[-1]))
    return np.array(idx, dtype=np.int64), np.array(vals)


@pytest.mark.parametrize("threads", [0, 1, -3, -7])
def test_round_trip_bit_exact_and_chunking(tmp_path, threads):
    rng = np.random.default_rng(7)
    n = 20000
    idx = np.stack([rng.integers(0, d, n) for d in (50, 70, 90)], 1).astype(np.uint32)
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-12, 12, n)
    t = hb.CooTensor((50, 70, 90), idx, vals)
    buf = io.StringIO()
    write_frostt(t, buf)
    text = buf.getvalue()
    # the reference format: "{coords} {v:.17g}"
    first = text.splitlines()[0].split()
    assert first[:3] == [str(int(i) + 1) for i in idx[0]] and first[3] == f"{vals[0]:.17g}"
    text = "# header\n\n" + text.replace("\n", "  # c\n", 5)
    back = parse_frostt(text, threads=threads)
    ri, rv = _reference_parse(text)
    assert np.array_equal(back.indices.astype(np.int64), ri)
    assert np.array_equal(back.values.view(np.int64), vals.view(np.int64))
    assert np.array_equal(rv.view(np.int64), vals.view(np.int64))
    p = tmp_path / "t.tns"
    save_frostt(t, str(p))
    again = load_frostt(str(p), dims=(50, 70, 90))
    assert again.dims == (50, 70, 90)
    assert np.array_equal(again.indices, t.indices)
    assert np.array_equal(again.values, t.values)


def test_first_error_line_across_chunks():
    good = "".join(f"{i % 5 + 1} 1 1 {i}.5\n" for i in range(3000))
    text = good + "1 1 x 1.0\n" + good + "1 1\n"
    for threads in (1, -2, -5, -9):
        with pytest.raises(ParseError) as exc:
            parse_frostt(text, threads=threads)
        assert exc.value.line == 3001, threads
