"""the array-native XYZR parser and read_complex against golden cases made
with the real reference's parse_xyzr / read_complex (tools/make_golden_xyzr.py,
tools/make_golden_complex_docs.py).  CPU only."""
import json
import os

import numpy as np
import pytest

import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import errors

from conftest import GOLD


@pytest.fixture(scope="module")
def xyzr_cases():
    return json.load(open(os.path.join(GOLD, "xyzr_cases.json")))["cases"]


def test_parse_xyzr_arrays_matches_reference_bit_for_bit(xyzr_cases):
    checked = 0
    for name, rec in xyzr_cases.items():
        if "error" in rec:
            with pytest.raises(getattr(errors, rec["error"])) as info:
                ax.parse_xyzr_arrays(rec["text"])
            assert str(info.value) == rec["message"], name
            assert getattr(info.value, "line_number", None) == rec["line_number"], name
        else:
            centers, radii = ax.parse_xyzr_arrays(rec["text"])
            want = np.array([[float.fromhex(v) for v in row] for row in rec["values"]], dtype=np.float64).reshape(-1, 4)
            got = np.concatenate([centers, radii[:, None]], axis=1)
            assert got.shape == want.shape, name
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), name      # bit exact, incl. -0.0 / denormals
            balls = ax.parse_xyzr(rec["text"])
            assert [b.index for b in balls] == list(range(len(balls)))
        checked += 1
    assert checked >= 15


def test_format_parse_round_trip():
    c, r = ax.synth.jittered_lattice(500, 1)
    c2, r2 = ax.parse_xyzr_arrays(ax.format_xyzr_arrays(c, r))
    assert np.array_equal(c, c2) and np.array_equal(r, r2)


def test_read_complex_matches_reference_cases():
    cases = json.load(open(os.path.join(GOLD, "complex_docs.json")))["cases"]
    for name, rec in cases.items():
        if "error" in rec:
            with pytest.raises(getattr(errors, rec["error"])) as info:
                ax.read_complex(rec["text"])
            assert str(info.value) == rec["message"], name
        else:
            k = ax.read_complex(rec["text"])
            assert list(k.counts()) == rec["counts"] and repr(k.alpha) == rec["alpha"], name
            assert k.ball_count == rec["ball_count"], name
            assert ax.write_complex(k) == rec["rewritten"], name
    assert len(cases) >= 20


def test_read_complex_bulk_path_on_a_large_document():
    """100k simplices through the vectorised body parser; a defect in the middle must be reported with the
    reference's message and line number."""
    rng = np.random.default_rng(0)
    tris = np.unique(np.sort(rng.integers(0, 5000, size=(100_000, 3)), axis=1), axis=0)
    tris = tris[(np.diff(tris, axis=1) > 0).all(axis=1)]
    k = ax.AlphaComplex(np.arange(5000), np.empty((0, 2), np.int64), tris, np.empty((0, 4), np.int64), 0.25, 5000)
    text = ax.write_complex(k)
    assert ax.read_complex(text) == k
    lines = text.splitlines()
    lines[70_000] = "2 7 7 9"
    with pytest.raises(errors.MalformedLine, match=r"line 70001: vertices must be strictly increasing"):
        ax.read_complex("\n".join(lines) + "\n")
