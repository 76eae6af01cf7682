""".optd / .optg (io.hpp:97-192) through libmo_b200.so against the UNMODIFIED
reference: files the reference wrote (tests/golden/io, make_io_golden.py)
read back with the same shapes and values, our writer reproduces the
reference's bytes exactly, and every malformed file fails with the error the
reference raised for it (verdicts.json).  Host-side byte work: no GPU."""
import json
import os

import numpy as np
import pytest

from paper_1604_06525_b200 import EdgeTable, MoError
from paper_1604_06525_b200.optio import DenseArray, read_optd, read_optg, write_optd, write_optg

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
VERDICTS = json.load(open(os.path.join(GOLD, "verdicts.json")))


def ref_values(n, dtype):
    v = np.arange(n, dtype=np.float64) * 0.37 - 1.5  # io_ref's fill (double, then cast)
    return v.astype(np.float32) if dtype == 0 else v


@pytest.mark.parametrize("name", sorted(VERDICTS))
def test_reads_like_the_reference(name):
    verdict = VERDICTS[name]["reference_read"].split()
    path = os.path.join(GOLD, name)
    if verdict[0] == "err":
        with pytest.raises(MoError) as ei:
            read_optd(path) if name.endswith(".optd") else read_optg(path)
        assert ei.value.code == verdict[1], (name, str(ei.value))
        return
    if name.endswith(".optd"):
        a = read_optd(path)
        dt, ch, nd = int(verdict[1]), int(verdict[2]), int(verdict[3])
        assert (a.dtype, a.channels, len(a.extents)) == (dt, ch, nd)
        assert a.extents == [int(x) for x in verdict[4:4 + nd]]
        np.testing.assert_array_equal(a.values, ref_values(a.value_count(), dt))
        assert abs(float(np.sum(a.values.astype(np.float64))) - float(verdict[4 + nd])) <= 1e-9 * max(
            1.0, abs(float(verdict[4 + nd])))
    else:
        g = read_optg(path)
        assert (g.arity, g.size()) == (int(verdict[1]), int(verdict[2]))
        assert int(np.sum(g.verts.astype(np.uint64))) == int(verdict[3])


@pytest.mark.parametrize("name", [n for n in sorted(VERDICTS) if "written_by" in VERDICTS[n]
                                  and VERDICTS[n]["written_by"].startswith("reference")])
def test_writes_the_reference_bytes(name, tmp_path):
    src = os.path.join(GOLD, name)
    out = tmp_path / name
    if name.endswith(".optd"):
        write_optd(out, read_optd(src))
    else:
        write_optg(out, read_optg(src))
    assert open(out, "rb").read() == open(src, "rb").read()


def test_round_trip_bitwise(tmp_path):
    rng = np.random.default_rng(3)
    for dt in (np.float32, np.float64):
        v = rng.standard_normal((6, 5, 3)).astype(dt)
        v.ravel()[:4] = [np.nan, np.inf, -0.0, np.finfo(dt).tiny / 2]  # every bit pattern survives
        write_optd(tmp_path / "a.optd", v, channels=3)
        a = read_optd(tmp_path / "a.optd")
        assert a.extents == [6, 5] and a.channels == 3
        assert a.values.tobytes() == v.tobytes()
    g = EdgeTable(2, np.array([0, 1, 1, 2, 2**63 + 5, 7], np.uint64))
    write_optg(tmp_path / "g.optg", g)
    h = read_optg(tmp_path / "g.optg")
    assert h.arity == 2 and h.verts.tobytes() == g.verts.tobytes()


def test_write_rejects_bad_input(tmp_path):
    with pytest.raises(MoError) as ei:
        write_optd(tmp_path / "x.optd", DenseArray(1, 2, [3], np.zeros(5)))
    assert ei.value.code == "ShapeMismatch"
    with pytest.raises(MoError) as ei:
        write_optd(tmp_path / "x.optd", DenseArray(3, 1, [1], np.zeros(1)))
    assert ei.value.code == "FormatError"
    with pytest.raises(MoError) as ei:
        write_optg(tmp_path / "x.optg", EdgeTable(2, np.zeros(3, np.uint64)))
    assert ei.value.code == "ShapeMismatch"
    with pytest.raises(MoError) as ei:
        read_optd(tmp_path / "missing.optd")
    assert ei.value.code == "FormatError"
