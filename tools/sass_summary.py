"""Per-kernel SASS instruction counts of the built library (auditable ISA evidence):
tcgen05 (UTCHMMA / UTCBAR, LDTM / STTM), TMA (UBLKCP bulk copies, UTMALDG tensor loads),
the math pipes (FFMA / FFMA2 / DFMA / HFMA2) and shared-memory ops, from `cuobjdump -sass`.

    python tools/sass_summary.py [lib] > profiles/r02/sass_summary.txt
"""
from __future__ import annotations

import re
import subprocess
import sys
from collections import Counter, OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "FFMA2", "FFMA", "DFMA",
        "HFMA2", "F2F", "LDS", "STS", "LDG", "STG", "SHFL", "BAR"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
        return out if len(out) == len(names) else names
    except OSError:
        return names


def main(lib: str) -> None:
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kernels: "OrderedDict[str, Counter]" = OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            kernels[cur][m.group(1)] += 1
    names = demangle(list(kernels))
    print(f"# SASS instruction counts per kernel: {lib} (cuobjdump -sass; static counts, not executed)")
    print("# " + " ".join(f"{k:>7}" for k in KEYS) + "  kernel")
    for (mangled, cnt), name in zip(kernels.items(), names):
        if not any(cnt[k] for k in KEYS):
            continue
        short = re.sub(r"\(.*$", "", name)
        print("  " + " ".join(f"{cnt[k]:>7}" for k in KEYS) + f"  {short[:150]}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_2602_18741_b200" / "libhadacodec_b200.so"))
