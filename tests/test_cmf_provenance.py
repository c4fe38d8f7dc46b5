"""The package colour-matching rows (data/cmf_n{47,81}.json) are the published CIE 1931 / D65
tables resampled by tools/make_cmf_tables.py (CmfTable's method, colorimetry.cpp:45-50) -- checked
where the reference's tables are available (this container); the GPU box only has the JSON."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not Path("/root/reference/proj/core/src/cmf_data.cpp").exists(), reason="needs the reference tables")
def test_cmf_json_regenerates_bit_identically():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "make_cmf_tables.py"), "--check"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("identical to") == 2
