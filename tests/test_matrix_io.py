"""ozm1 matrix files (the reference's io.hpp:26-40, the data format its CLI
feeds multiply() with): files written here are byte-identical to the
reference's, each side reads the other's bit-exactly, and malformed input
fails with the reference's messages.  Host-only (no GPU needed)."""
import numpy as np
import pytest

import paper_2506_11277_b200 as oz


def _values(rng, m, n):
    a = rng.standard_normal((m, n)) * np.exp2(rng.integers(-40, 40, size=(m, n)))
    flat = a.reshape(-1)
    flat[:8] = [0.0, -0.0, 5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, 1.0,
                -0.1, 1.0 / 3.0]
    return a


@pytest.mark.parametrize("fmt", [oz.MatrixFormat.HEX, oz.MatrixFormat.DEC])
def test_files_match_reference_bytes_and_round_trip(po, tmp_path, fmt):
    rng = np.random.default_rng(int(fmt) + 3)
    a = _values(rng, 37, 23)
    ours, theirs = tmp_path / "ours.ozm", tmp_path / "theirs.ozm"
    oz.write_matrix_file(ours, a, fmt)
    po.ref_write_matrix_file(theirs, a, int(fmt))
    assert ours.read_bytes() == theirs.read_bytes()
    back = oz.read_matrix_file(theirs, fmt)
    assert np.array_equal(back.view(np.uint64), a.view(np.uint64))
    back = po.ref_read_matrix_file(ours, int(fmt))
    assert np.array_equal(back.view(np.uint64), a.view(np.uint64))


def test_empty_and_single_row(tmp_path):
    for shape in [(0, 0), (0, 5), (1, 7), (7, 1)]:
        a = np.arange(shape[0] * shape[1], dtype=np.float64).reshape(shape) - 2.5
        p = tmp_path / f"m{shape[0]}x{shape[1]}.ozm"
        oz.write_matrix_file(p, a)
        assert np.array_equal(oz.read_matrix_file(p), a)


@pytest.mark.parametrize("text,fmt,msg", [
    ("ozm2 1 1\n3ff0000000000000\n", 0, "missing 'ozm1 <rows> <cols>' header"),
    ("ozm1 2 2\n3ff0000000000000 0000000000000000\n", 0, "truncated file"),
    ("ozm1 1 1\n3ff00000000000\n", 0, "expected a 16-hex-digit entry"),
    ("ozm1 1 1\n3ff000000000000g\n", 0, "bad hex entry"),
    ("ozm1 1 1\n1.5x\n", 1, "bad decimal entry"),
])
def test_malformed_files_raise_like_the_reference(tmp_path, text, fmt, msg):
    p = tmp_path / "bad.ozm"
    p.write_text(text)
    with pytest.raises(oz.MatrixIOError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        oz.read_matrix_file(p, oz.MatrixFormat(fmt))


def test_missing_file(tmp_path):
    with pytest.raises(oz.MatrixIOError, match="cannot open matrix file"):
        oz.read_matrix_file(tmp_path / "nope.ozm")
