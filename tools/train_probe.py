"""Probe: codec training step time (gradients + losses over a batch, then Adam on the raw
weights) on the GPU at several batch sizes, against the compiled reference's gradients().

    python tools/train_probe.py
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_18741_b200 import api  # noqa: E402

N, K = 81, 6


def main() -> None:
    ctx = api.Context(0)
    rng = np.random.default_rng(0)
    re_ = rng.uniform(-0.5, 0.5, (K, N)) / np.sqrt(N)
    rd = rng.uniform(-0.5, 0.5, (N, K)) / np.sqrt(K)
    sizes = [int(a) for a in sys.argv[1:]] or [128, 1024, 8192, 65536]
    for m in sizes:
        refl = torch.from_numpy(rng.uniform(0, 1, (m, N))).cuda()
        illum = torch.from_numpy(rng.uniform(0, 1, (m, N))).cuda()
        api.codec_train_grad(ctx, re_, rd, 10.0, refl, illum)
        torch.cuda.synchronize()
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            api.codec_train_grad(ctx, re_, rd, 10.0, refl, illum)
        dt = (time.perf_counter() - t0) / reps
        print(json.dumps({"batch": m, "ms_per_step": round(dt * 1e3, 3), "M_pairs_s": round(m / dt / 1e6, 2)}))
    if len(sys.argv) > 1:
        return
    try:
        import oracle

        ref = oracle.reference(N)
        m = 128
        r = rng.uniform(0, 1, m * N)
        l = rng.uniform(0, 1, m * N)
        ge, gd, lo = np.zeros(K * N), np.zeros(N * K), np.zeros(6)
        t0 = time.perf_counter()
        for _ in range(5):
            ref.ref_codec_gradients(K, 10.0, re_.reshape(-1), rd.reshape(-1), r, l, m, np.array(api.LOSS_WEIGHTS),
                                    ge.ctypes.data, gd.ctypes.data, lo)
        dt = (time.perf_counter() - t0) / 5
        print(json.dumps({"reference_batch": m, "ms_per_step": round(dt * 1e3, 3)}))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"reference": f"unavailable: {e}"}))


if __name__ == "__main__":
    main()
