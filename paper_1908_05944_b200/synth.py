"""Synthetic protein-like inputs for tests and benchmarks (host side, numpy).

* ``random_globule``  -- G1 of SURVEY.md 8(d): the reference's own generator
  (reference synth.py:15-71), restated here so inputs can be regenerated where
  the reference is not installed.  Bit-identical draws for the same seed.
* ``jittered_lattice`` -- G2 of SURVEY.md 8(d): vectorised jittered lattice at
  protein density (1 atom / 12 A^3), radii U[1.2, 1.9].
* ``adversarial_density`` -- config 5: G2 with 20% of the volume emptied into
  voids and 20% of the atoms packed into 3x-denser cores.
"""
from __future__ import annotations

import math

import numpy as np


def random_globule(n: int, seed: int, min_sep: float = 1.0, radius_range=(1.0, 2.0),
                   density: float = 0.05):
    """Rejection-sampled centres in a cube of volume n/density, pairwise
    separation >= min_sep, radii uniform in radius_range.
    Returns (centers (n,3) f64, radii (n,) f64)."""
    if n < 1:
        raise ValueError("n must be positive")
    if min_sep <= 0.0:
        raise ValueError("min_sep must be positive")
    r_lo, r_hi = radius_range
    if not 0.0 < r_lo <= r_hi:
        raise ValueError("radius_range must satisfy 0 < lo <= hi")
    rng = np.random.default_rng(seed)
    box = (n / density) ** (1.0 / 3.0)
    scale = 1.0 / min_sep
    sep2 = min_sep * min_sep
    buckets: dict = {}
    pts = np.empty((n, 3), dtype=np.float64)
    count = 0
    tries = 0
    while count < n:
        tries += 1
        if tries > 10_000 * n:
            raise RuntimeError(f"could not place {n} points at density {density} with min_sep {min_sep}")
        p = rng.uniform(0.0, box, size=3)
        key = tuple(int(v) for v in np.floor(p * scale))
        ok = True
        for ox in (-1, 0, 1):
            for oy in (-1, 0, 1):
                for oz in (-1, 0, 1):
                    for j in buckets.get((key[0] + ox, key[1] + oy, key[2] + oz), ()):
                        d = pts[j] - p
                        if (d * d).sum() < sep2:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if not ok:
                break
        if ok:
            pts[count] = p
            buckets.setdefault(key, []).append(count)
            count += 1
    radii = rng.uniform(r_lo, r_hi, size=n)
    return pts, radii


LATTICE_SPACING = 12.0 ** (1.0 / 3.0)


def jittered_lattice(n: int, seed: int = 0):
    """G2: n sites of an m^3 lattice (m = ceil(n^(1/3)), spacing 12^(1/3) A),
    jitter +-0.25 spacing per axis, radii U[1.2, 1.9].  Draw order:
    permutation, jitter, radii.  Returns (centers, radii)."""
    rng = np.random.default_rng(seed)
    a = LATTICE_SPACING
    m = int(np.ceil(n ** (1.0 / 3.0)))
    while m ** 3 < n:      # guard against cube-root rounding
        m += 1
    idx = np.sort(rng.permutation(m ** 3)[:n])
    ix = idx % m
    iy = (idx // m) % m
    iz = idx // (m * m)
    c = np.stack([ix, iy, iz], axis=1).astype(np.float64) * a
    c += rng.uniform(-0.25 * a, 0.25 * a, size=(n, 3))
    r = rng.uniform(1.2, 1.9, size=n)
    return c, r


def adversarial_density(n: int, seed: int = 0, void_fraction: float = 0.2,
                        core_fraction: float = 0.2, shuffle: bool = False):
    """Config 5: clustered voids and dense cores.

    Start from a G2 lattice of n sites; carve spherical voids (radius 15-40 A)
    until ``void_fraction`` of the atoms are gone; then drop spherical cores
    (radius 10-25 A) filled with a finer jittered lattice (1 atom / 4 A^3,
    jitter +-0.18 spacing, base atoms inside the core removed) until at least
    ``core_fraction`` of n are core atoms and the total reaches n; finally trim
    surplus base atoms.  Indices follow final array order (base survivors in
    lattice order, then cores), optionally shuffled.  Returns (centers, radii).
    """
    rng = np.random.default_rng(seed)
    base, _ = jittered_lattice(n, seed)
    lo = base.min(axis=0)
    hi = base.max(axis=0)
    alive = np.ones(n, dtype=bool)
    target_dead = int(void_fraction * n)
    while (~alive).sum() < target_dead:
        ctr = rng.uniform(lo, hi)
        rad = rng.uniform(15.0, 40.0)
        d2 = ((base - ctr) ** 2).sum(axis=1)
        alive &= d2 > rad * rad
    fine = 4.0 ** (1.0 / 3.0)
    cores = []
    n_core = 0
    while n_core < core_fraction * n or alive.sum() + n_core < n:
        ctr = rng.uniform(lo, hi)
        rad = rng.uniform(10.0, 25.0)
        # keep cores apart so fine lattices never interleave
        if any(math.dist(ctr, c0) < rad + r0 + 1.0 for c0, r0 in cores):
            continue
        d2 = ((base - ctr) ** 2).sum(axis=1)
        alive &= d2 > (rad + 0.6) ** 2
        k = int(np.ceil(rad / fine))
        g = np.arange(-k, k + 1, dtype=np.float64) * fine
        pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
        pts = pts + rng.uniform(-0.18 * fine, 0.18 * fine, size=pts.shape)
        pts = pts[(pts ** 2).sum(axis=1) < (rad - 0.6) ** 2] + ctr
        cores.append((ctr, rad))
        cores_pts = pts if n_core == 0 else np.concatenate([cores_pts, pts])  # noqa: F821
        n_core = cores_pts.shape[0]
    keep = np.flatnonzero(alive)
    surplus = keep.size + n_core - n
    if surplus > 0:
        drop = rng.choice(keep.size, size=surplus, replace=False)
        mask = np.ones(keep.size, dtype=bool)
        mask[drop] = False
        keep = keep[mask]
    centers = np.concatenate([base[keep], cores_pts])[:n]
    if shuffle:
        centers = centers[rng.permutation(centers.shape[0])]
    radii = rng.uniform(1.2, 1.9, size=centers.shape[0])
    return np.ascontiguousarray(centers), radii
