#!/usr/bin/env python
"""Golden vectors for parse_xyzr, made by importing the REAL reference
(read-only mount /root/reference) in the build container:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_xyzr.py

Writes tests/golden/xyzr_cases.json: documents, the parsed values (as float hex strings, bit exact)
or the exception type + message the reference raises.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import alphax  # noqa: E402
from alphax.io import format_xyzr, parse_xyzr  # noqa: E402
from alphax.synth import random_instance  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

docs = {
    "plain": "0 0 0 1.5\n1.25 -2.5e0 3 1.9\n",
    "comments_blank": "# header\n\n 0.1 0.2 0.3 1.2  # trailing\n\t4 5 6 1.7\n   \n#only\n7 8 9 1e0",
    "roundtrip_20": format_xyzr(random_instance(20, seed=4, min_sep=1.0, radius_range=(1.2, 1.9), density=1 / 12)),
    "precision": "0.1 0.2 0.30000000000000004 1.2000000000000002\n1e-320 -0.0 123456789.123456789 5e-324\n",
    "three_fields": "0 0 0 1\n1 2 3\n",
    "five_fields": "0 0 0 1 7\n",
    "three_plus_five": "1 2 3\n4 5 6 7 8\n",
    "non_numeric": "0 0 0 1\n1 x 3 1\n",
    "nan_field": "0 0 0 1\n1 nan 3 1\n",
    "inf_radius": "0 0 0 inf\n",
    "zero_radius": "0 0 0 1\n# c\n1 2 3 0\n",
    "negative_radius": "1 2 3 -1.5\n",
    "bad_before_nonpositive": "1 2 3 0\n1 2\n",
    "nonfinite_and_nonpositive_same_line": "nan 2 3 -1\n",
    "empty": "",
    "only_comments": "# a\n# b\n",
    "fortran_exponent": "1d0 2 3 1\n",
    "underscore": "1_0 2 3 1\n",
}
out = {"reference_version": alphax.__version__, "cases": {}}
for name, text in docs.items():
    rec = {"text": text}
    try:
        balls = parse_xyzr(text)
        rec["values"] = [[float(v).hex() for v in (*b.center, b.radius)] for b in balls]
    except Exception as exc:          # noqa: BLE001
        rec["error"] = type(exc).__name__
        rec["message"] = str(exc)
        rec["line_number"] = getattr(exc, "line_number", None)
    out["cases"][name] = rec
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "xyzr_cases.json"), "w"), indent=1)
print({k: v.get("error", len(v.get("values", []))) for k, v in out["cases"].items()})
