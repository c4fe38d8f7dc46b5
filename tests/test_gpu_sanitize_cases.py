"""The small-shape cases of every TMA / mbarrier / TMEM kernel (tools/sanitize_cases.py, meant for
compute-sanitizer, which this GPU pool does not allow) run as a plain GPU test: each case is checked
against the oracle."""
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_sanitize_cases_run_clean():
    sys.path.insert(0, str(ROOT / "tools"))
    import sanitize_cases

    sanitize_cases.main()
