"""Small-shape runs of every TMA / mbarrier / TMEM kernel of the library, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers tile_pipeline / tile_pipeline_ws / tile_generic (codec round trip, latent and
naive shading at L = 8 / 32, with and without spectra), the loss (three warp groups,
in-compute barrier, ragged tile), mlp2_kernel and mlp_kernel (tcgen05 / TMEM), the
multi-bounce chain and the training step's grad_reduce_kernel (bulk-copy ring).  Each case
is checked against the oracle so a sanitizer-clean run is also a correct one."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_2602_18741_b200 import api, synth  # noqa: E402
from paper_2602_18741_b200.colorimetry import cmf_matrix, grid  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.maximum(np.abs(b), np.max(np.abs(b), axis=-1, keepdims=True)) if b.ndim > 1 else np.abs(b)
    return float(np.max(np.abs(a - b) / np.maximum(den, 1e-30))) if b.size else 0.0


def main():
    orc = oracle.oracle()
    ctx = api.Context(0)
    n = 81
    for k, L, P in ((6, 8, 64 * 5 + 7), (9, 32, 64 * 3 + 1)):
        E, D = synth.codec_weights(3, k, n)
        codec = api.Codec(ctx, E, D)
        pal = torch.from_numpy(synth.palette(3, 256, n)).cuda()
        lts = synth.lights(3, L, n)
        pc = codec.encode(pal)
        lc = codec.encode(torch.from_numpy(lts).cuda()).cpu().numpy()
        idx, cosv = api.synth_gbuffer(ctx, 3, 0, P, L, 256)
        out = codec.shade_latent(pc, lc, idx, cosv, latent=True, spectra=True)
        ref = [np.zeros((P, d), np.float32) for d in (k, n, 3, 3)]
        orc.orc_shade_latent(D, k, n, cmf_matrix(n), grid(n)[1], pc.cpu().numpy(), lc, L,
                             idx.cpu().numpy().view(np.uint32), cosv.cpu().numpy(), P, *ref)
        assert rel(out["rgb"].cpu().numpy(), ref[3]) < 1e-5 and rel(out["spectra"].cpu().numpy(), ref[1]) < 1e-5
        out2 = codec.shade_latent(pc, lc, idx, cosv)  # xyz + rgb only (config-2 kernel)
        assert rel(out2["rgb"].cpu().numpy(), ref[3]) < 1e-5
        nv = codec.shade_spectral(pal, lts, idx, cosv)
        nv2 = codec.shade_spectral(pal, lts, idx, cosv, spectra=True)
        assert rel(nv["rgb"].cpu().numpy(), nv2["rgb"].cpu().numpy()) < 1e-5
        S = api.synth_gm_spectra(ctx, 3, "codec.spectra", 0, P, n)
        rt = codec.roundtrip(S)
        rr = [np.zeros((P, d), np.float32) for d in (k, n, 3, 3)]
        orc.orc_codec_roundtrip(E, D, k, n, cmf_matrix(n), grid(n)[1], S.cpu().numpy(), P, *rr)
        assert rel(rt["rgb"].cpu().numpy(), rr[3]) < 1e-5
        A = api.synth_gm_spectra(ctx, 3, "loss.a", 0, 64 * 7 + 5, n)
        B = api.synth_gm_spectra(ctx, 3, "loss.b", 0, 64 * 7 + 5, n)
        got = float(codec.hadamard_loss(A, B).cpu().numpy()[0])
        want = orc.orc_hadamard_loss(E, D, k, n, A.cpu().numpy(), B.cpu().numpy(), 64 * 7 + 5)
        assert abs(got - want) <= 1e-5 * abs(want), (got, want)
        print(f"shade / naive / roundtrip / loss k={k} L={L}: ok", flush=True)
    # multi-bounce chain
    E, D = synth.codec_weights(3, 6, n)
    codec = api.Codec(ctx, E, D)
    pal = torch.from_numpy(synth.palette(3, 256, n)).cuda()
    ill = torch.from_numpy(synth.lights(3, 16, n, purpose="scene.illuminants")).cuda()
    pidx, iidx, tw = api.synth_chain(ctx, 3, 0, 37, 64, 256, 16)
    pc, ic = codec.encode(pal), codec.encode(ill)
    ch = codec.multibounce_latent(pc, ic, pidx, iidx, tw, latent=True)
    nch = codec.multibounce_spectral(pal, ill, pidx, iidx, tw)
    ph, ih, th = (x.cpu().numpy() for x in (pidx, iidx, tw))
    lat = np.zeros((37, 6), np.float32)
    orc.orc_chain(6, pc.cpu().numpy(), ic.cpu().numpy(), ph, ih, th, 37, 64, 4, lat)
    assert rel(ch["latent"].cpu().numpy(), lat) < 1e-5
    spec = np.zeros((37, n), np.float32)
    X, R = np.zeros((37, 3), np.float32), np.zeros((37, 3), np.float32)
    orc.orc_chain(n, pal.cpu().numpy(), ill.cpu().numpy(), ph, ih, th, 37, 64, 4, spec)
    orc.orc_spectra_to_outputs(cmf_matrix(n), grid(n)[1], n, spec, 37, X, R)
    assert rel(nch["rgb"].cpu().numpy(), R) < 1e-5
    print("chain: ok", flush=True)
    # MLP (tcgen05 / TMEM), both kernels
    w = synth.mlp_weights(3, 6, 64)
    P = 128 * 9 + 5
    rgb = api.synth_uniform(ctx, 3, "mlp.input", 0, P * 3).reshape(P, 3)
    ref = np.zeros((P, 6), np.float32)
    orc.orc_mlp_forward(rgb.cpu().numpy(), P, 64, 6, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"], w["b3"], ref)
    got = api.CodeMLP(ctx, w).forward(rgb).cpu().numpy()
    assert rel(got, ref) < 1e-2
    print("mlp: ok", flush=True)
    # training step (grad_reduce_kernel's bulk-copy ring)
    rng = np.random.default_rng(3)
    re_ = rng.uniform(-0.5, 0.5, (6, n)) / 9
    rd = rng.uniform(-0.5, 0.5, (n, 6)) / 3
    refl = torch.from_numpy(rng.uniform(0, 1, (300, n))).cuda()
    illum = torch.from_numpy(rng.uniform(0, 1, (300, n))).cuda()
    losses, ge, gd = api.codec_train_grad(ctx, re_, rd, 10.0, refl, illum)
    assert np.all(np.isfinite(ge)) and np.all(np.isfinite(gd))
    print("train: ok", flush=True)
    ctx.synchronize()
    print("sanitize cases: all ok")


if __name__ == "__main__":
    main()
