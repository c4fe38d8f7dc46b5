"""gpurun_out/traffic_c<cfg>.csv (tools/ncu_traffic.sh) -> profiles/traffic_config<cfg>.json:
mean dram__bytes_read.sum + dram__bytes_write.sum per launch of the hot kernel over a
steady-state window (bench.py reads bytes_per_launch into roofline.traffic)."""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
ALG = {"1": 696 * (1 << 20), "2": 60 * 2073600, "3": 468 * 8294400, "4": 1368 * 4194304, "5a": 36 * (1 << 24),
       "5b": 648 * (1 << 24)}


def main(cfgs):
    for c in cfgs:
        path = ROOT / "gpurun_out" / f"traffic_c{c}.csv"
        if not path.exists():
            continue
        rows = [r for r in csv.reader(l for l in path.read_text().splitlines() if not l.startswith("=="))]
        if not rows:
            continue
        h = rows[0]
        iname, imet, ival = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        per = {}
        for r in rows[1:]:
            if len(r) <= ival:
                continue
            key = (r[h.index("ID")], r[iname])
            per.setdefault(key, {})[r[imet]] = float(r[ival].replace(",", ""))
        launches = list(per.values())
        rd = sum(x.get("dram__bytes_read.sum", 0) for x in launches) / len(launches)
        wr = sum(x.get("dram__bytes_write.sum", 0) for x in launches) / len(launches)
        kern = list(per)[0][1]
        out = {"config": c, "kernel": kern, "launches": len(launches), "dram_read_bytes": rd, "dram_write_bytes": wr,
               "bytes_per_launch": rd + wr, "algorithmic_bytes": ALG.get(c),
               "method": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none, launches "
                         "20-35 of a back-to-back --plain run (steady state: earlier launches' dirty lines are "
                         "written back inside the window)",
               "source": f"gpurun_out/traffic_c{c}.csv (round 2)"}
        (ROOT / "profiles" / f"traffic_config{c}.json").write_text(json.dumps(out, indent=1) + "\n")
        print(c, kern[:60], f"{(rd + wr) / 1e6:.1f} MB/launch", f"alg {ALG.get(c, 0) / 1e6:.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1:] or ["1", "2", "3", "4", "5a", "5b"])
