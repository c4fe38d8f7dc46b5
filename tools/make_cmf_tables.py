"""Regenerate the package's colour-matching data (paper_2602_18741_b200/data/cmf_n{47,81}.json).

Source data: the published CIE 1931 2-degree standard observer (1 nm, 360-830 nm) and the CIE
D65 spectral power distribution (5 nm, 360-830 nm), read as plain numbers from the tables the
reference ships (reference/proj/core/src/cmf_data.cpp; sampling constants from
spectral_tables.hpp:10-22).  Nothing of the reference is compiled or executed: the numbers are
parsed and resampled here with the reference's method -- CmfTable (colorimetry.cpp:45-50)
resamples each table with resample(..., zero_outside=false) (spectrum.cpp:60-98): linear
interpolation between the bracketing samples, clamped to the end values -- onto
wavelength_at(i) = lambda_min + step * i of each grid (spectrum.hpp:10-21).

    python tools/make_cmf_tables.py [--check]     # --check: compare with the committed files

Run where /root/reference exists (this container); the JSON files are committed.
"""
from __future__ import annotations

import argparse
import bisect
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2602_18741_b200.colorimetry import DATA, grid  # noqa: E402

REF_SRC = Path("/root/reference/proj/core/src")


def _constants(text: str) -> dict:
    out = {}
    for name, val in re.findall(r"constexpr\s+(?:int|double)\s+(\w+)\s*=\s*([-0-9.eE+]+)\s*;", text):
        out[name] = float(val)
    return out


def _array(text: str, name: str) -> list:
    m = re.search(r"\b" + name + r"\s*\[[^\]]*\]\s*=\s*\{(.*?)\};", text, re.S)
    if not m:
        raise ValueError(f"table {name} not found")
    return [float(v) for v in re.findall(r"[-+]?\d*\.?\d+(?:[eE][-+]?\d+)?", m.group(1))]


def resample(src_lambda: list, src_vals: list, n: int) -> list:
    """Linear interpolation onto the n-grid, clamped to the end samples (spectrum.cpp:60-98)."""
    lo, step = grid(n)
    out = []
    for i in range(n):
        lam = lo + step * i
        if lam <= src_lambda[0]:
            out.append(src_vals[0])
        elif lam >= src_lambda[-1]:
            out.append(src_vals[-1])
        else:
            hi = bisect.bisect_right(src_lambda, lam)
            j = hi - 1
            t = (lam - src_lambda[j]) / (src_lambda[hi] - src_lambda[j])
            out.append(src_vals[j] + t * (src_vals[hi] - src_vals[j]))
    return out


def tables(n: int) -> dict:
    consts = _constants((REF_SRC / "spectral_tables.hpp").read_text())
    data = (REF_SRC / "cmf_data.cpp").read_text()
    cie_n, cie_lo, cie_step = int(consts["kCieSamples"]), consts["kCieLambdaMin"], consts["kCieLambdaStep"]
    d65_n, d65_lo, d65_step = int(consts["kD65Samples"]), consts["kD65LambdaMin"], consts["kD65LambdaStep"]
    cie_lam = [cie_lo + cie_step * i for i in range(cie_n)]
    d65_lam = [d65_lo + d65_step * i for i in range(d65_n)]
    out = {}
    for key, name in (("xbar", "kCieX"), ("ybar", "kCieY"), ("zbar", "kCieZ")):
        vals = _array(data, name)
        assert len(vals) == cie_n, (name, len(vals))
        out[key] = resample(cie_lam, vals, n)
    d65 = _array(data, "kD65")
    assert len(d65) == d65_n
    out["d65"] = resample(d65_lam, d65, n)
    return out


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--check", action="store_true", help="only compare with the committed files")
    a = ap.parse_args()
    bad = 0
    for n in (47, 81):
        t = tables(n)
        path = DATA / f"cmf_n{n}.json"
        old = json.loads(path.read_text()) if path.exists() else None
        same = old is not None and all(old[k] == t[k] for k in ("xbar", "ybar", "zbar", "d65"))
        print(f"n={n}: {'identical to' if same else 'DIFFERS from'} {path.name}")
        bad += not same
        if not a.check:
            lo, step = grid(n)
            doc = {"source": "CIE 1931 2-degree observer (1 nm) and CIE D65 (5 nm) as tabulated in the reference's "
                             "cmf_data.cpp, linearly resampled onto the grid by tools/make_cmf_tables.py "
                             "(CmfTable's method, colorimetry.cpp:45-50 / spectrum.cpp:60-98)",
                   "n": n, "lambda_min": lo, "lambda_step": step, **t}
            path.write_text(json.dumps(doc, indent=1) + "\n")
    return 1 if (a.check and bad) else 0


if __name__ == "__main__":
    sys.exit(main())
