"""Summarise ncu captures into profiles/<round>/ (tracked).

    python tools/summarize_ncu.py gpurun_out profiles/r01

* <round>/ncu_full_config<C>.md   key metrics of the hot kernel of config C (from
  gpurun_out/full_c<C>.ncu-rep, `ncu --set full`), with stall reasons;
* <round>/ncu_launches_default.md share of device time per kernel of the default
  bench command (gpurun_out/launches_default.csv, cold-cache serialised ncu pass);
* profiles/traffic_config<C>.json  DRAM read + write bytes per launch of the hot
  kernel, which bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ALGO_BYTES = {"1": 696 * (1 << 20), "2": 60 * 1920 * 1080, "3": 468 * 3840 * 2160, "4": 1368 * 2048 * 2048,
              "5a": 36 * 4096 * 4096, "5b": 648 * (1 << 24), "6": 27 * 1920 * 1080, "7": 6 * 4 * 256 * 256,
              # 8 (line_parse_kernel): the 264 557 378-byte codes CSV text + 8 B per code + 32 B per row
              # (id span, newline position, row flag)
              "8": 264557378 + 8 * 6 * (1 << 21) + 32 * (1 << 21),
              # 9 (line_parse_kernel): the 175 525 094-byte spectra CSV + 8 B per value (111 per curve)
              # + 32 B per row
              "9": 175525094 + 8 * 111 * (1 << 17) + 32 * (1 << 17),
              # 10 (grad_reduce_kernel): the per-pair rows it streams — 5 x 81 + 6 x 6 doubles per pair
              "10": 8 * (5 * 81 + 6 * 6) * (1 << 16)}
METRICS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "DRAM read (bytes)"),
    ("dram__bytes_write.sum", "DRAM write (bytes)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (%)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)"),
    ("sm__warps_active.avg.per_cycle_active", "active warps / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "tensor (hmma) active cycles / SM"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor memory active (%)"),
]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep: Path) -> tuple[dict, dict]:
    """(values, units) of the first profiled kernel."""
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return dict(zip(h, v)), dict(zip(h, u))


def to_bytes(d: dict, u: dict, key: str) -> float:
    return num(d.get(key, "nan")) * SCALE.get(u.get(key, "byte"), float("nan"))


def num(x: str) -> float:
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return float("nan")


def summarize_full(src: Path, dst: Path) -> None:
    for rep in sorted(src.glob("full_c*.ncu-rep")):
        cfg = rep.stem.split("_c", 1)[1]
        d, u = raw(rep)
        kern = d.get("Kernel Name", "?")
        lines = [f"# ncu --set full, config {cfg}", "", f"kernel: `{kern}`", "",
                 "| metric | value |", "|---|---|"]
        for key, label in METRICS:
            if key in d:
                lines.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(x for x in stalls.values() if x == x) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        lines += ["", "stall samples: " + ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top)]
        rd, wr = to_bytes(d, u, "dram__bytes_read.sum"), to_bytes(d, u, "dram__bytes_write.sum")
        traffic = rd + wr if rd == rd and wr == wr else None
        algo = ALGO_BYTES.get(cfg)
        lines += ["", f"algorithmic bytes per launch (SURVEY §8d): {algo}; DRAM read + write: {traffic:.0f}"
                  f" ({traffic / algo * 100:.1f}% of algorithmic; writes still in L2 at kernel end are not"
                  " counted for short kernels)" if traffic else ""]
        (dst / f"ncu_full_config{cfg}.md").write_text("\n".join(lines) + "\n")
        if traffic is not None:
            (dst.parent / f"traffic_config{cfg}.json").write_text(json.dumps(
                {"config": cfg, "kernel": kern, "dram_read_bytes": rd, "dram_write_bytes": wr,
                 "bytes_per_launch": traffic, "algorithmic_bytes": algo,
                 "note": "ncu --set full (cold cache); dram__bytes_read.sum + dram__bytes_write.sum",
                 "source": rep.name}, indent=1) + "\n")


def summarize_launches(src: Path, dst: Path) -> None:
    f = src / "launches_default.csv"
    if not f.exists():
        return
    rows = list(csv.reader(f.open()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0][:110]
            per[name][0] += 1
            per[name][1] += num(r[vi])
    total = sum(v[1] for v in per.values()) or 1.0
    lines = ["# ncu launch list of `python bench.py --steps 16 --warmup 3 --no-cpu-baseline`",
             "(`--metrics gpu__time_duration.sum --clock-control none`; cold-cache, serialised: compare shares)", "",
             "| kernel | launches | total ns | share |", "|---|---|---|---|"]
    for name, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {n} | {t:.0f} | {t / total * 100:.1f}% |")
    (dst / "ncu_launches_default.md").write_text("\n".join(lines) + "\n")


def summarize_config_launches(src: Path, dst: Path, cfgs: list) -> None:
    """launches_c<cfg>.csv (ncu --metrics gpu__time_duration.sum[,dram__bytes_*] of
    `bench.py --config <cfg> --plain`) -> ncu_launches_config<cfg>.md: per-kernel share of the step."""
    for cfg in cfgs:
        f = src / f"launches_c{cfg}.csv"
        if not f.exists():
            continue
        rows = list(csv.reader(f.open()))
        hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        h = rows[hi]
        ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        per = defaultdict(lambda: {"n": 0, "ns": 0.0, "dram": 0.0})
        for r in rows[hi + 1:]:
            name = r[ki].split("(")[0][:110]
            if r[mi] == "gpu__time_duration.sum":
                per[name]["n"] += 1
                per[name]["ns"] += num(r[vi])
            elif r[mi].startswith("dram__bytes"):
                per[name]["dram"] += num(r[vi])
        total = sum(v["ns"] for v in per.values()) or 1.0
        lines = [f"# ncu launch list of config {cfg} (`bench.py --config {cfg} --plain`)",
                 "(`gpu__time_duration.sum`, DRAM bytes; cold-cache, serialised: compare shares)", "",
                 "| kernel | launches | avg us | share | avg DRAM MB |", "|---|---|---|---|---|"]
        for name, v in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
            lines.append(f"| `{name}` | {v['n']} | {v['ns'] / max(v['n'], 1) / 1e3:.1f} | {v['ns'] / total * 100:.1f}% "
                         f"| {v['dram'] / max(v['n'], 1) / 1e6:.1f} |")
        (dst / f"ncu_launches_config{cfg}.md").write_text("\n".join(lines) + "\n")


def main() -> int:
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    dst.mkdir(parents=True, exist_ok=True)
    summarize_full(src, dst)
    summarize_launches(src, dst)
    summarize_config_launches(src, dst, sys.argv[3:])  # e.g. `... gpurun_out profiles/r01 8`
    if (src / "launches_default.csv").exists():
        (dst / "ncu_launches_default.csv").write_text((src / "launches_default.csv").read_text())
    return 0


if __name__ == "__main__":
    sys.exit(main())
