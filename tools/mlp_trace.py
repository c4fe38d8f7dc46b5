"""Per-phase cycle trace of mlp_kernel (HC_MLP_TRACE=1) on the config-5a texture (4096^2)."""
import os
import sys
from pathlib import Path

os.environ["HC_MLP_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2602_18741_b200 import api, synth  # noqa: E402

ctx = api.Context(0)
up = api.CodeMLP(ctx, synth.mlp_weights(2602, 6))
rgb = api.synth_uniform(ctx, 2602, "mlp.input", 0, 4096 * 4096 * 3).view(-1, 3)
for _ in range(2):
    up.forward(rgb)
torch.cuda.synchronize()
