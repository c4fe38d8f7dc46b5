"""Probe: run the config-2 shading kernel directly on pinned host buffers (zero copy).

With UVA, pinned host memory is addressable from kernels; the tile pipeline's bulk
copies then read the G-buffer over PCIe and its bulk stores write XYZ / sRGB back to
host memory, with no copy-engine transfers and no chunk fill / drain.  Prints the
per-frame time and checks the result against the device-resident path.

    python tools/zerocopy_probe.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_18741_b200 import _lib, api, synth  # noqa: E402

SEED = 2602
N, K, L, W, H = 81, 6, 8, 1920, 1080


def main() -> None:
    ctx = api.Context(0)
    E, D = synth.codec_weights(SEED, K, N)
    codec = api.Codec(ctx, E, D)
    pal_codes = codec.encode(torch.from_numpy(synth.palette(SEED, 256, N)).cuda())
    lc = np.ascontiguousarray(codec.encode(torch.from_numpy(synth.lights(SEED, L, N)).cuda()).cpu().numpy())
    P = W * H
    idx_d, cos_d = api.synth_gbuffer(ctx, SEED, 0, P, L, 256)
    ref = codec.shade_latent(pal_codes, lc, idx_d, cos_d)
    idx_h = idx_d.cpu().pin_memory()
    cos_h = cos_d.cpu().pin_memory()
    xyz_h = torch.zeros(P, 3).pin_memory()
    rgb_h = torch.zeros(P, 3).pin_memory()
    lib = _lib.lib()

    def run():
        ctx.bind_stream()
        _lib.check(lib.hc_shade_latent(codec.h, pal_codes.data_ptr(), 256, lc.ctypes.data, L, idx_h.data_ptr(),
                                       cos_h.data_ptr(), P, None, None, xyz_h.data_ptr(), rgb_h.data_ptr()))

    run()
    torch.cuda.synchronize()
    ok = torch.equal(xyz_h, ref["xyz"].cpu()) and torch.equal(rgb_h, ref["rgb"].cpu())
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"probe": "zero-copy shade (cfg 2)", "ms_per_frame": round(ms, 4),
                      "Mpix_s": round(P / ms / 1e3, 1), "h2d_GBs": round(P * 36 / ms / 1e6, 1),
                      "d2h_GBs": round(P * 24 / ms / 1e6, 1), "matches_device": bool(ok)}))


if __name__ == "__main__":
    main()
