"""Compile the reference's own unit-test files against the C++ drop-in with only the
namespace changed (source compatibility).

Each listed /root/reference/proj/tests/<name>.cpp is read, its `using namespace hadacodec;`
becomes `using namespace hadacodec::b200;`, and the result is compiled (from /tmp, nothing
of the reference is written into the repo) with tests/cpp/compat first on the include path:
`hadacodec/<header>.hpp` there maps onto include/hadacodec_b200.hpp and `doctest.h` is our
minimal harness.  The binary lands in tests/cpp/bin/ (git-ignored; it travels to the GPU box
with the snapshot, where /root/reference does not exist) and is run by
tests/test_dropin.py::test_reference_unit_tests_unchanged on a B200.

    python tests/cpp/build_ref_tests.py
"""
from __future__ import annotations

import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF_TESTS = Path("/root/reference/proj/tests")
CASES = ("test_codec", "test_spectrum", "test_colorimetry")  # codec, spectrum and colorimetry value APIs
OUT = ROOT / "tests" / "cpp" / "bin" / "ref_unit_tests"


def build() -> Path | None:
    if not REF_TESTS.is_dir():
        return None
    sys.path.insert(0, str(ROOT))
    from paper_2602_18741_b200 import build as b

    lib = b.build()
    OUT.parent.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        srcs = []
        for name in CASES:
            text = (REF_TESTS / f"{name}.cpp").read_text()
            assert "using namespace hadacodec;" in text, name
            dst = Path(tmp) / f"{name}.cpp"
            dst.write_text(text.replace("using namespace hadacodec;", "using namespace hadacodec::b200;"))
            srcs.append(str(dst))
        cmd = ["g++", "-std=c++17", "-O1", f"-I{ROOT / 'tests' / 'cpp' / 'compat'}", f"-I{ROOT / 'include'}", *srcs,
               str(ROOT / "tests" / "cpp" / "compat" / "doctest_main.cpp"), f"-L{lib.parent}", "-lhadacodec_b200",
               f"-Wl,-rpath,{lib.parent}", "-o", str(OUT)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"reference unit tests do not compile against the drop-in:\n{r.stderr[-4000:]}")
    return OUT


if __name__ == "__main__":
    print(build())
