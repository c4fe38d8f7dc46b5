"""Phase trace of the cooperative radix select (HC_SELECT_TRACE=1) on a config-6 frame."""
import os
import sys
from pathlib import Path

os.environ["HC_SELECT_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2602_18741_b200 import api, synth  # noqa: E402

ctx = api.Context(0)
E, D = synth.codec_weights(2602, 6, 81)
codec = api.Codec(ctx, E, D)
P, L = 1920 * 1080, 8
pal = torch.from_numpy(synth.palette(2602, 256, 81)).cuda()
lts = synth.lights(2602, L, 81)
idx, cosv = api.synth_gbuffer(ctx, 2602, 0, P, L, 256)
gt = codec.shade_spectral(pal, lts, idx, cosv)["rgb"]
test = codec.shade_latent(codec.encode(pal), codec.encode(torch.from_numpy(lts).cuda()).cpu().numpy(), idx, cosv)["rgb"]
for _ in range(2):
    print(api.scene_color_report(codec, gt, test))
