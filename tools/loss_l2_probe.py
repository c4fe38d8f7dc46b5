"""Loss kernel (config 5b) throughput with inputs resident in L2 (2^17 pairs, 85 MB < 126 MB L2)
vs streamed from HBM (2^24 pairs): separates the kernel's compute / latency limit from HBM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_18741_b200 import api, synth  # noqa: E402

ctx = api.Context(0)
E, D = synth.codec_weights(2602, 6, 81)
codec = api.Codec(ctx, E, D)
for pairs, reps in ((1 << 17, 200), (1 << 20, 50), (1 << 24, 5)):
    A = api.synth_gm_spectra(ctx, 2602, "loss.a", 0, pairs, 81)
    B = api.synth_gm_spectra(ctx, 2602, "loss.b", 0, pairs, 81)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(3):
        codec.hadamard_loss(A, B, out=out)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        codec.hadamard_loss(A, B, out=out)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / reps
    print(f"pairs={pairs:>9d}  {ms * 1e3:9.1f} us/launch  {pairs / ms / 1e6:7.2f} G pairs/s  "
          f"{pairs * 648 / ms / 1e6:7.1f} GB/s", flush=True)
    del A, B
