"""``validate`` on the GPU path -- SURVEY.md 8(f) row 4 (reference cli.py:134-180).

The reference's ``alphax validate`` computes a complex in grid mode, compares it
with the exhaustive ``naive`` oracle (symmetric difference per dimension) and
checks two properties: closure, and monotonicity alpha -> alpha + 1.  The naive
O(n^4) oracle is out of scope for this build, so the
comparison partner is whatever the caller supplies -- typically the complex the
reference produced for the same input (``read_complex`` of its document); the
property checks run on the GPU results, the two alphas through ONE sweep
(``compute_alpha_sweep``).  Same report lines and pass criterion as the
reference's command.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .pipeline import AlphaComplex, PipelineConfig, closure_ok, compute_alpha_sweep


@dataclass(frozen=True)
class ValidationReport:
    counts: tuple
    mismatches: tuple            # per dimension: rows only in one of the two complexes (0s without a partner)
    closed: bool
    monotone: bool

    @property
    def ok(self) -> bool:
        return sum(self.mismatches) == 0 and self.closed and self.monotone

    def lines(self, label: str = "input") -> list:
        c = self.counts
        return [f"[{label}]: complex (v={c[0]}, e={c[1]}, t={c[2]}, T={c[3]})",
                "  symmetric difference: " + " ".join(f"dim{d}={m}" for d, m in enumerate(self.mismatches)),
                f"  closure: {'ok' if self.closed else 'VIOLATED'}   "
                f"monotonicity (alpha -> alpha+1): {'ok' if self.monotone else 'VIOLATED'}"]


def validate_complex(centers, radii, cfg: PipelineConfig, expected: AlphaComplex | None = None) -> ValidationReport:
    """The checks of the reference's ``cmd_validate`` for one input (cli.py:146-178)."""
    centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
    radii = np.asarray(radii, dtype=np.float64).reshape(-1)
    # the bigger complex is computed with the default tolerance, as the reference's command does (cli.py:167-174)
    if cfg.tolerance == PipelineConfig(alpha=0.0).tolerance:
        k, bigger = compute_alpha_sweep(centers, radii, [cfg.alpha, cfg.alpha + 1.0], cfg)
    else:
        (k,) = compute_alpha_sweep(centers, radii, [cfg.alpha], cfg)
        (bigger,) = compute_alpha_sweep(centers, radii, [cfg.alpha + 1.0],
                                        PipelineConfig(alpha=cfg.alpha + 1.0, biomolecule_mode=cfg.biomolecule_mode))
    mism = (0, 0, 0, 0)
    if expected is not None:
        diff = k.symmetric_difference(expected)
        mism = tuple(int(diff[d][0].shape[0] + diff[d][1].shape[0]) for d in range(4))
    return ValidationReport(counts=k.counts(), mismatches=mism, closed=closure_ok(k) and (expected is None or closure_ok(expected)),
                            monotone=k.is_subcomplex_of(bigger))
