#!/usr/bin/env python
"""Golden cases for read_complex, made by importing the REAL reference
(read-only mount /root/reference) in the build container:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_complex_docs.py

Writes tests/golden/complex_docs.json: documents and either the parsed complex (counts + the text
write_complex gives back) or the exception type + message the reference raises.
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import alphax  # noqa: E402
from alphax.io import read_complex, write_complex  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TETRA = ("alphax 0.1.0 n=4 alpha=0.5\n0 0\n0 1\n0 2\n0 3\n1 0 1\n1 0 2\n1 0 3\n1 1 2\n1 1 3\n1 2 3\n"
         "2 0 1 2\n2 0 1 3\n2 0 2 3\n2 1 2 3\n3 0 1 2 3\n")
docs = {
    "tetra": TETRA,
    "unordered_lines_are_canonicalised": "alphax 0.1.0 n=5 alpha=-1.5\n1 2 3\n0 4\n1 0 1\n0 0\n1 0 1\n",
    "blank_lines_and_tabs": "alphax 0.1.0 n=3 alpha=1e-3\n\n0 0\n \n1\t0\t2\n  2  0 1 2\n",
    "header_only": "alphax 9.9 n=0 alpha=inf\n",
    "empty": "",
    "bad_header_word": "alphay 0.1.0 n=4 alpha=0.5\n0 0\n",
    "bad_header_fields": "alphax 0.1.0 n=4\n",
    "bad_header_n": "alphax 0.1.0 n=four alpha=0.5\n",
    "bad_header_alpha": "alphax 0.1.0 n=4 alpha=\n",
    "non_integer": "alphax 0.1.0 n=4 alpha=0.5\n0 0\n1 0 x\n",
    "float_field": "alphax 0.1.0 n=4 alpha=0.5\n1 0 1.0\n",
    "bad_dim": "alphax 0.1.0 n=4 alpha=0.5\n4 0 1 2 3 4\n",
    "negative_dim": "alphax 0.1.0 n=4 alpha=0.5\n-1 0\n",
    "arity": "alphax 0.1.0 n=4 alpha=0.5\n0 0\n2 0 1\n",
    "out_of_range": "alphax 0.1.0 n=4 alpha=0.5\n0 0\n1 0 4\n",
    "negative_vertex": "alphax 0.1.0 n=4 alpha=0.5\n1 -1 2\n",
    "not_increasing": "alphax 0.1.0 n=4 alpha=0.5\n2 0 2 1\n",
    "repeated_vertex": "alphax 0.1.0 n=4 alpha=0.5\n1 2 2\n",
    "first_error_wins": "alphax 0.1.0 n=4 alpha=0.5\n1 0 9\n1 1 0\n1 x\n",
    "huge_index": "alphax 0.1.0 n=4 alpha=0.5\n0 99999999999999999999999\n",
}
out = {"reference_version": alphax.__version__, "cases": {}}
for name, text in docs.items():
    rec = {"text": text}
    try:
        k = read_complex(text)
        rec["counts"] = list(k.counts())
        rec["alpha"] = repr(k.alpha)
        rec["ball_count"] = k.ball_count
        rec["rewritten"] = write_complex(k)
    except Exception as exc:          # noqa: BLE001
        rec["error"] = type(exc).__name__
        rec["message"] = str(exc)
    out["cases"][name] = rec
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "complex_docs.json"), "w"), indent=1)
print({k: v.get("error", v.get("counts")) for k, v in out["cases"].items()})
