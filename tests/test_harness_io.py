"""Host-side harness pieces (no GPU): the DSVD file format, MatrixSpec
validation and CLI usage errors, against pkg/src/dcsvd/harness.py:40-66,
190-231, 325-343 (same bytes, same exit codes)."""

import struct

import numpy as np
import pytest
from numpy.testing import assert_array_equal


def _h():
    from paper_2508_11467_b200 import harness

    return harness


def test_dsvd_binary_round_trip_and_layout(tmp_path):
    h = _h()
    a = np.asfortranarray(np.arange(12, dtype=np.float64).reshape(4, 3) / 7.0)
    p = tmp_path / "a.dsvd"
    h.write_matrix(p, a)
    raw = p.read_bytes()
    assert raw[:4] == b"DSVD"
    assert struct.unpack("<HQQ", raw[4:22]) == (1, 4, 3)
    assert raw[22:] == a.astype("<f8").tobytes(order="F")
    b = h.read_matrix(p)
    assert b.flags.f_contiguous
    assert_array_equal(a, b)


def test_dsvd_text_mode_round_trips_exactly(tmp_path):
    h = _h()
    a = np.random.default_rng(0).standard_normal((5, 2))
    p = tmp_path / "a.txt"
    h.write_matrix(p, a, text=True)
    assert_array_equal(h.read_matrix(p), a)
    h.write_matrix(tmp_path / "v.dsvd", np.array([1.0, 2.0]))
    assert h.read_matrix(tmp_path / "v.dsvd").shape == (2, 1)


def test_dsvd_errors(tmp_path):
    h = _h()
    p = tmp_path / "bad.dsvd"
    p.write_bytes(b"DSVD" + b"\x01\x00")
    with pytest.raises(ValueError, match="truncated"):
        h.read_matrix(p)
    p.write_bytes(b"DSVD" + struct.pack("<HQQ", 2, 1, 1) + b"\x00" * 8)
    with pytest.raises(ValueError, match="version"):
        h.read_matrix(p)
    p.write_bytes(b"DSVD" + struct.pack("<HQQ", 1, 2, 2) + b"\x00" * 8)
    with pytest.raises(ValueError, match="payload"):
        h.read_matrix(p)
    with pytest.raises(ValueError):
        h.write_matrix(tmp_path / "x.dsvd", np.zeros((2, 2, 2)))


def test_matrix_spec_validation():
    h = _h()
    for args, kw in ((("weird", 4, 4), {}), (("random", 0, 4), {}), (("geo", 4, 4), {"cond": 0.5}),
                     (("geo", 4, 4), {"seed": -1})):
        with pytest.raises(ValueError):
            h.MatrixSpec(*args, **kw)


def test_cli_usage_and_io_errors(tmp_path, capsys):
    h = _h()
    assert h.cli_main([]) == 2
    assert h.cli_main(["gen", "--kind", "nope", "--m", "2", "--n", "2", "--out", "x"]) == 2
    assert h.cli_main(["run", "--input", str(tmp_path / "missing.dsvd")]) == 1   # OSError -> 1
    assert h.cli_main(["--help"]) == 0
    err = capsys.readouterr().err
    assert "dcsvd run" in err
