"""One `ncu --set full` report -> a markdown summary (key metrics + stall mix).

    python tools/ncu_md.py gpurun_out/chain.ncu-rep profiles/r02/ncu_full_config4.md "config 4 chain" [alg_bytes]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from summarize_ncu import METRICS, num, raw, to_bytes  # noqa: E402

EXTRA = [("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active"),
         ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe (F2F, MUFU)"),
         ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active"),
         ("idc__request_hit_rate.pct", "immediate-constant cache hit rate"),
         ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
         ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts")]


def main(rep, out, title, alg=None):
    d, u = raw(Path(rep))
    lines = [f"# ncu --set full: {title}", "", f"kernel: `{d.get('Kernel Name', '?')}`", "",
             "| metric | value |", "|---|---|"]
    seen = set()
    for key, label in list(METRICS) + EXTRA:
        if key in d and key not in seen:
            seen.add(key)
            lines.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(x for x in stalls.values() if x == x) or 1.0
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
    lines += ["", "stall samples: " + ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top)]
    rd, wr = to_bytes(d, u, "dram__bytes_read.sum"), to_bytes(d, u, "dram__bytes_write.sum")
    if alg and rd == rd:
        lines += ["", f"algorithmic bytes per launch: {int(alg)}; DRAM read + write in this (cold, single-launch) "
                  f"capture: {rd + wr:.0f} ({(rd + wr) / float(alg) * 100:.1f}%)"]
    Path(out).write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
