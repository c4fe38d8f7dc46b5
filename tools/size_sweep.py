"""Config-2 kernel throughput vs frame size (fixed per-launch overhead vs steady state).

Times hc_shade_latent (k = 6, 8 lights, XYZ + sRGB) at 1080p, 4K and 8K with the bench's
method (CUDA graph of launches over rotating buffer sets larger than L2, CUDA events) and
prints the achieved algorithmic GB/s of each size.  If the fraction rises with size, the
1080p gap to the copy peak is launch ramp + tail, not the steady-state pipeline.

    python tools/size_sweep.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_18741_b200 import api, synth  # noqa: E402

SEED = 20260218
N, K, L = 81, 6, 8
PEAK = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]


def main() -> None:
    ctx = api.Context(0)
    E, D = synth.codec_weights(SEED, K, N)
    codec = api.Codec(ctx, E, D)
    pal = torch.from_numpy(synth.palette(SEED, 256, N)).cuda()
    pal_codes = codec.encode(pal)
    light_codes = codec.encode(torch.from_numpy(synth.lights(SEED, L, N)).cuda()).cpu().numpy()
    stream = torch.cuda.Stream()
    for name, (w, h) in {"1080p": (1920, 1080), "4k": (3840, 2160), "8k": (7680, 4320)}.items():
        P = w * h
        sets = max(2, min(8, int(1.2e9 // (P * 60)) + 1))
        bufs = []
        for s in range(sets):
            idx, cosv = api.synth_gbuffer(ctx, SEED, s * P, P, L, 256)
            out = {"xyz": ctx.empty(P, 3), "rgb": ctx.empty(P, 3)}
            bufs.append((idx, cosv, out))
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for b in bufs:
                codec.shade_latent(pal_codes, light_codes, b[0], b[1], out=b[2])
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for b in bufs:
                    codec.shade_latent(pal_codes, light_codes, b[0], b[1], out=b[2])
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        reps = max(4, int(400 * 2073600 / P) // sets)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(reps):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * sets)
        gbs = P * 60 / us / 1e3
        print(json.dumps({"size": name, "pixels": P, "us_per_frame": round(us, 2), "GBs": round(gbs, 1),
                          "frac": round(gbs / PEAK, 3), "sets": sets}))
        del bufs, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
