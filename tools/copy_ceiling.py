"""Size-matched copy ceiling: how fast can ANY kernel move a config's bytes?

The bench's roofline divides by the long-copy HBM figure of MEASURED_PEAKS.json.  A single
frame of config 2 moves only ~124 MB, where launch ramp and tail are a visible share of the
kernel.  This times device-to-device copies with the same read/write volume per launch and the
same L2 rotation scheme (8 buffer sets) as bench.py, so the kernel's fraction can be read
against what a plain copy achieves at that size.

    python tools/copy_ceiling.py            # prints one JSON line per size
"""
from __future__ import annotations

import json

import torch


def time_copy(read_bytes: int, write_bytes: int, sets: int = 8, reps: int = 400) -> dict:
    # Copy `write_bytes` from a `read_bytes` source: read == write for a plain copy; for a
    # read-heavy kernel (config 2 reads 36, writes 24 B/px) we read the extra bytes with a sum.
    n_w = write_bytes // 4
    n_extra = max(0, read_bytes - write_bytes) // 4
    src = [torch.empty(n_w, dtype=torch.float32, device="cuda").uniform_() for _ in range(sets)]
    dst = [torch.empty(n_w, dtype=torch.float32, device="cuda") for _ in range(sets)]
    extra = [torch.empty(n_extra, dtype=torch.float32, device="cuda").uniform_() for _ in range(sets)] if n_extra else None
    out = torch.empty(1, device="cuda")
    stream = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        for i in range(sets):  # warm
            dst[i].copy_(src[i])
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for i in range(sets):
                dst[i].copy_(src[i])
    torch.cuda.synchronize()
    loops = reps // sets
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(loops):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    us_copy = e0.elapsed_time(e1) * 1e3 / (loops * sets)
    res = {"write_MB": write_bytes / 1e6, "copy_us": us_copy, "copy_GBs": 2 * write_bytes / us_copy / 1e3}
    if extra is not None:
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g2, stream=stream):
                for i in range(sets):
                    torch.sum(extra[i], dim=0, out=out)
        for _ in range(3):
            g2.replay()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(loops):
                g2.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        us_sum = e0.elapsed_time(e1) * 1e3 / (loops * sets)
        res.update({"extra_read_MB": n_extra * 4 / 1e6, "sum_us": us_sum})
    return res


def main() -> None:
    px = 1920 * 1080
    for name, rd, wr in (("config2_frame", 36 * px, 24 * px), ("copy_62MB", 62_208_000, 62_208_000),
                         ("copy_1GB", 1 << 30, 1 << 30)):
        r = time_copy(rd, wr)
        r["case"] = name
        print(json.dumps(r))


if __name__ == "__main__":
    main()
