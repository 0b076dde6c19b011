"""CPU-side checks of the C-ABI library: it loads and exports every symbol the
header declares (no compute calls without a GPU), and the package refuses to
compute without CUDA instead of falling back."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def test_library_exports_every_declared_symbol():
    from paper_1908_05944_b200 import _native
    from paper_1908_05944_b200.build import build_native

    build_native()
    lib = _native.load()
    header = open(os.path.join(ROOT, "include", "alphax_b200.h")).read()
    declared = set(re.findall(r"\b(axb_[a-z_0-9]+)\s*\(", header))
    assert declared == set(_native.SYMBOLS), declared ^ set(_native.SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.axb_version() >= 100
    assert lib.axb_status_name(0) == b"AXB_OK"
    assert lib.axb_status_name(7) == b"AXB_ERR_DEGENERATE"
    assert lib.axb_arena_hint(1_000_000, 0.0, 1.9) > 1 << 30


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1908_05944_b200 import (Ball, NativeLibraryMissing, PipelineConfig, compute_alpha_complex,
                                       compute_alpha_complex_arrays)

    with pytest.raises(NativeLibraryMissing):
        compute_alpha_complex_arrays(np.zeros((2, 3)), np.ones(2), PipelineConfig(alpha=0.0))
    with pytest.raises(NativeLibraryMissing):
        compute_alpha_complex([Ball((0, 0, 0), 1.0, 0)], PipelineConfig(alpha=0.0))


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1908_05944_b200")
    for base, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(base, f)).read()
                assert "import oracle" not in text and "alpha_oracle" not in text, f


def test_write_complex_bytes_match_reference_golden(gold_config1, gold_small):
    """The C++ formatter (no GPU needed) reproduces the reference's canonical document byte for byte."""
    import hashlib

    from paper_1908_05944_b200 import AlphaComplex, read_complex, stats_csv, write_complex

    data, meta = gold_config1
    for tag, m in meta.items():
        k = AlphaComplex(data[f"{tag}__k0"], data[f"{tag}__k1"], data[f"{tag}__k2"], data[f"{tag}__k3"], m["alpha"], 1000)
        text = write_complex(k)
        assert hashlib.sha256(text.encode()).hexdigest() == m["sha256_complex"]
        assert read_complex(text) == k
    for name, rec in gold_small.items():
        m = rec["meta"]
        k = AlphaComplex(rec["k0"], rec["k1"], rec["k2"], rec["k3"], m["alpha"], len(rec["radii"]))
        assert hashlib.sha256(write_complex(k).encode()).hexdigest() == m["sha256_complex"], name
    tetra = gold_small["tetra_a05"]
    k = AlphaComplex(tetra["k0"], tetra["k1"], tetra["k2"], tetra["k3"], 0.5, 4)
    assert stats_csv(k) == "dim,count\n0,4\n1,6\n2,4\n3,1\ntotal,15\neuler,1\n"      # reference T/test_cli.py:25-35
