"""Spectral grids and colour-matching data for the B200 path.

Grids (spectrum.hpp:10-21): the reference's canonical 47-sample grid over
368-830 nm and BASELINE.json's 81-sample grid over 380-780 nm (5 nm), both
with wavelength_at(i) = lambda_min + step * i.

CMF rows are the reference's CmfTable (colorimetry.cpp:45-61: CIE 1931 2-degree
1 nm tables linearly resampled onto the grid, plus D65).  They are shipped as
package data made by tools/make_cmf_tables.py (the published CIE tables + an
in-repo resampler; oracle/make_golden.py checks them bit-exact against the
compiled reference's CmfTable); at n = 81 every 5 nm sample falls exactly on a
1 nm table entry.  XYZ uses the
radiance convention dlambda * sum cmf * s (colorimetry.cpp:75-87); sRGB the
IEC 61966-2-1 matrix (colorimetry.cpp:22-26).
"""
from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

DATA = Path(__file__).resolve().parent / "data"

# (lambda_min, lambda_max) per supported sample count.
GRIDS = {47: (368.0, 830.0), 81: (380.0, 780.0)}

XYZ_TO_LINEAR_RGB = np.array(
    [[3.2404542, -1.5371385, -0.4985314],
     [-0.9692660, 1.8760108, 0.0415560],
     [0.0556434, -0.2040259, 1.0572252]], dtype=np.float64)


def grid(n: int) -> tuple[float, float]:
    """(lambda_min, step) of the n-sample grid (spectrum.hpp:10-21)."""
    lo, hi = GRIDS[n]
    return lo, (hi - lo) / (n - 1)


def wavelengths(n: int) -> np.ndarray:
    lo, step = grid(n)
    return np.array([lo + step * i for i in range(n)], dtype=np.float64)


@lru_cache(maxsize=None)
def cmf_table(n: int) -> dict:
    """xbar, ybar, zbar, d65 on the n-grid as float64 arrays (+ 'cmf' 3 x n)."""
    path = DATA / f"cmf_n{n}.json"
    if not path.exists():
        raise FileNotFoundError(f"{path} missing (generate with `python tools/make_cmf_tables.py`)")
    d = json.loads(path.read_text())
    out = {k: np.array(d[k], dtype=np.float64) for k in ("xbar", "ybar", "zbar", "d65")}
    out["cmf"] = np.stack([out["xbar"], out["ybar"], out["zbar"]])
    out["lambda_min"], out["lambda_step"] = d["lambda_min"], d["lambda_step"]
    return out


def cmf_matrix(n: int) -> np.ndarray:
    return np.ascontiguousarray(cmf_table(n)["cmf"])


@lru_cache(maxsize=None)
def white_xyz(n: int) -> tuple[float, float, float]:
    """CmfTable::white_xyz (colorimetry.cpp:45-73): D65-weighted rows normalised so a unit
    reflectance has Y = 100, summed — in the reference's sequential fp64 order."""
    t = cmf_table(n)
    x, y, z, d = (t[r].tolist() for r in ("xbar", "ybar", "zbar", "d65"))
    norm = 0.0
    for i in range(n):
        norm += y[i] * d[i]
    scale = 100.0 / norm
    out = []
    for row in (x, y, z):
        acc = 0.0
        for i in range(n):
            acc += scale * row[i] * d[i]
        out.append(acc)
    return tuple(out)


# The analytic multi-lobe Gaussian fit of the CIE 1931 2-degree colour-matching functions
# (Wyman, Sloan & Shirley, "Simple Analytic Approximations to the CIE XYZ Color Matching
# Functions", JCGT 2(2), 2013): each function is a sum of piecewise Gaussians
# g(l; mu, s1, s2) = exp(-(l - mu)^2 / (2 s^2)) with s = s1 below mu and s2 above.  BASELINE.json
# config 1 names this fit; it lies within 1.4 % of the tabulated functions' peaks on the
# 81-sample grid (tests/test_oracle.py pins that).
_CMF_LOBES = {
    "xbar": ((1.056, 599.8, 37.9, 31.0), (0.362, 442.0, 16.0, 26.7), (-0.065, 501.1, 20.4, 26.2)),
    "ybar": ((0.821, 568.8, 46.9, 40.5), (0.286, 530.9, 16.3, 31.1)),
    "zbar": ((1.217, 437.0, 11.8, 36.0), (0.681, 459.0, 26.0, 13.8)),
}


def _lobe(lam: np.ndarray, mu: float, s1: float, s2: float) -> np.ndarray:
    s = np.where(lam < mu, s1, s2)
    t = (lam - mu) / s
    return np.exp(-0.5 * t * t)


def cmf_analytic(n: int) -> np.ndarray:
    """3 x n colour-matching rows of the analytic multi-lobe fit on the n-sample grid."""
    lam = wavelengths(n)
    rows = []
    for name in ("xbar", "ybar", "zbar"):
        rows.append(sum(a * _lobe(lam, mu, s1, s2) for a, mu, s1, s2 in _CMF_LOBES[name]))
    return np.ascontiguousarray(np.stack(rows), dtype=np.float64)
