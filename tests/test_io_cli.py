"""the array-native XYZR parser against golden vectors made with the real
reference's parse_xyzr (tools/make_golden_xyzr.py), and the CLI's argument / error surface.  CPU only."""
import json
import os

import numpy as np
import pytest

import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import cli, errors

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


def test_cli_parser_and_exit_codes(tmp_path, capsys):
    p = cli.build_parser()
    a = p.parse_args(["bench", "--random", "50", "--alpha", "0.5", "--repeat", "2", "--workers", "1,2"])
    assert a.func is cli.cmd_bench and a.random == 50 and a.repeat == 2
    # stats on a serialized complex works without a GPU (reference T/test_cli.py:25-35)
    doc = tmp_path / "k.txt"
    doc.write_text("alphax 0.1.0 n=4 alpha=0.5\n0 0\n0 1\n0 2\n0 3\n1 0 1\n1 0 2\n1 0 3\n1 1 2\n1 1 3\n1 2 3\n"
                   "2 0 1 2\n2 0 1 3\n2 0 2 3\n2 1 2 3\n3 0 1 2 3\n")
    assert cli.main(["stats", "--input", str(doc)]) == 0
    assert capsys.readouterr().out == "dim,count\n0,4\n1,6\n2,4\n3,1\ntotal,15\neuler,1\n"
    # error mapping: AlphaxError / OSError -> 1, ValueError -> 2 (reference cli.py:266-278)
    bad = tmp_path / "bad.xyzr"
    bad.write_text("0 0 0 1\n1 2\n")
    assert cli.main(["compute", "--input", str(bad), "--alpha", "0"]) == 1
    assert "line 2" in capsys.readouterr().err
    assert cli.main(["compute", "--input", str(tmp_path / "missing.xyzr"), "--alpha", "0"]) == 1
    assert cli.main(["bench", "--alpha", "0"]) == 2
    assert cli.main(["compute", "--input", str(bad), "--format", "pdb", "--alpha", "0"]) == 2


@pytest.mark.gpu
def test_cli_compute_and_bench_on_the_gpu(tmp_path, capsys):
    """compute writes the reference's canonical document (config 1 digest), bench prints the reference's CSV schema."""
    import hashlib

    c, r = ax.synth.random_globule(1000, seed=0, min_sep=1.0, radius_range=(1.2, 1.9), density=1 / 12)
    src = tmp_path / "g.xyzr"
    src.write_text(ax.format_xyzr_arrays(c, r))
    out = tmp_path / "k.txt"
    assert cli.main(["compute", "--input", str(src), "--alpha", "0.0", "--output", str(out), "--stats"]) == 0
    assert "total,8818" in capsys.readouterr().err
    assert hashlib.sha256(out.read_bytes()).hexdigest()[:16] == "00b61c8547390672"
    assert cli.main(["bench", "--random", "2000", "--alpha", "0.5", "--repeat", "2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "repeat,workers,stage,seconds" and len(lines) == 1 + 2 * 9
    rows = [l.split(",") for l in lines[1:10]]
    assert [row[2] for row in rows] == list(ax.STAGE_NAMES) + ["total"]
    assert sum(float(row[3]) for row in rows[:-1]) <= 1.05 * float(rows[-1][3])              # reference T/test_cli.py:120-143
