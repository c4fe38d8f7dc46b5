"""GPU path tracer vs the compiled reference's render (oracle/_ref): agreement statistics."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import torch  # noqa: E402

from paper_2602_18741_b200 import api, synth  # noqa: E402


def run(mode, n, k, max_depth, block, multipass=False, W=48, H=32, spp=16, seed=5):
    ctx = api.Context(0)
    E, D = synth.codec_weights(11, k, n)
    codec = api.Codec(ctx, E, D)
    scene = synth.cornell_scene(n, block)
    got = api.render(codec, scene, mode, W, H, spp, max_depth, seed, path_hashes=True, multipass=multipass)
    img = got["image"].cpu().numpy()
    hs = got["path_hashes"].cpu().numpy().view(np.uint64).reshape(-1)
    sc, keep = api.scene_struct(scene, n)
    job = api.HcRenderJob(api.RENDER_MODES[mode], W, H, spp, max_depth, seed)
    ch = img.shape[-1]
    ref = np.zeros((H, W, ch), np.float32)
    rh = np.zeros(W * H, np.uint64)
    ev = C.c_uint64()
    rc = oracle.reference(n).ref_render(C.addressof(sc), C.addressof(job), k, E, D, int(multipass), ref.reshape(-1),
                                        rh, C.byref(ev))
    exact = np.mean(np.all(img == ref, axis=-1))
    den = np.maximum(np.abs(ref), np.max(np.abs(ref), axis=-1, keepdims=True))
    rel = np.max(np.abs(img - ref) / np.maximum(den, 1e-30))
    print(f"{mode:8s} n={n} k={k} depth={max_depth:2d} block={block} mp={multipass}: rc={rc} exact_px={exact:.4f} "
          f"max_rel={rel:.2e} hash_eq={np.mean(hs == rh):.4f} evals {got['shading_evals']} vs {ev.value}")


for args in [("spectral", 81, 6, 3, False), ("latent", 81, 6, 3, True), ("rgb", 81, 6, 3, True),
             ("latent", 47, 9, -1, True), ("spectral", 47, 6, -1, True), ("latent", 81, 6, 3, True, True)]:
    run(*args)
