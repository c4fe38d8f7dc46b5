"""Seeded random sweep of the shading / codec entry points against the oracle: grid, code size,
light count, palette size, row count, which outputs are requested and whether the inputs and
outputs sit at 16-byte-aligned or 4-byte-offset addresses are all drawn at random, so the
combinations the hand-written parity cases do not name (generic light counts with partial
outputs, small palettes on the bulk-copy path, offset inputs with aligned outputs, ...) are hit
too.  Same tolerance as test_gpu_parity.py (1e-5 relative, row-infinity-norm denominator)."""
import numpy as np
import pytest

from conftest import rel_err
from paper_2602_18741_b200 import synth
from paper_2602_18741_b200.colorimetry import cmf_matrix, grid

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5
CASES = 48


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def _place(t: torch.Tensor, offset: int) -> torch.Tensor:
    """The same values at `offset` elements past an aligned allocation (a contiguous view)."""
    if offset == 0:
        return t
    flat = torch.empty(t.numel() + 16, dtype=t.dtype, device=t.device)
    v = flat[offset:offset + t.numel()].view(t.shape)
    v.copy_(t)
    return v


def _out(rows: int, width: int, offset: int) -> torch.Tensor:
    flat = torch.full((rows * width + 16,), float("nan"), dtype=torch.float32, device="cuda")
    return flat[offset:offset + rows * width].view(rows, width)


def _draw(rng):
    n = int(rng.choice([81, 81, 47]))
    k = int(rng.choice([3, 6, 9]))
    L = int(rng.choice([1, 2, 5, 8, 8, 13, 32, 32, 64]))
    n_pal = int(rng.choice([1, 7, 100, 256, 256]))
    P = int(rng.choice([1, 31, 64, 255, 256, 257, 1000, 4097, 12_289]))
    return n, k, L, n_pal, P


@pytest.mark.parametrize("case", range(CASES))
def test_random_shade_latent(api, ctx, orc, case):
    rng = np.random.default_rng(1000 + case)
    n, k, L, n_pal, P = _draw(rng)
    E, D = synth.codec_weights(77 + case, k, n)
    codec = api.Codec(ctx, E, D)
    pal = synth.palette(77 + case, n_pal, n)
    lts = synth.lights(77 + case, L, n)
    pal_codes = codec.encode(torch.from_numpy(pal).cuda())
    light_codes = codec.encode(torch.from_numpy(lts).cuda()).cpu().numpy()
    idx, cosv = api.synth_gbuffer(ctx, 77 + case, int(rng.integers(0, 1 << 20)), P, L, n_pal)
    off_in, off_out = int(rng.choice([0, 0, 1, 3])), int(rng.choice([0, 0, 1, 2]))
    want = {key: bool(rng.integers(0, 2)) for key in ("latent", "spectra", "xyz", "rgb")}
    if not any(want.values()):
        want["rgb"] = True
    widths = {"latent": k, "spectra": n, "xyz": 3, "rgb": 3}
    out = {key: _out(P, widths[key], off_out) if want[key] else None for key in widths}
    codec.shade_latent(_place(pal_codes, off_in), light_codes, _place(idx, off_in), _place(cosv, off_in), out=out)
    ref = [np.zeros((P, widths[key]), np.float32) for key in ("latent", "spectra", "xyz", "rgb")]
    orc.orc_shade_latent(D, k, n, cmf_matrix(n), grid(n)[1], host(pal_codes), light_codes, L,
                         host(idx).view(np.uint32), host(cosv), P, *ref)
    tag = f"case {case}: n={n} k={k} L={L} n_pal={n_pal} P={P} in+{off_in} out+{off_out}"
    for key, r in zip(("latent", "spectra", "xyz", "rgb"), ref):
        if want[key]:
            e = rel_err(host(out[key]), r)
            assert e <= TOL, f"{tag} {key}: rel err {e:.3e}"


@pytest.mark.parametrize("case", range(CASES // 2))
def test_random_shade_spectral(api, ctx, orc, case):
    rng = np.random.default_rng(5000 + case)
    n, _, L, n_pal, P = _draw(rng)
    E, D = synth.codec_weights(177 + case, 6, n)
    codec = api.Codec(ctx, E, D)
    pal = synth.palette(177 + case, n_pal, n)
    lts = synth.lights(177 + case, L, n)
    idx, cosv = api.synth_gbuffer(ctx, 177 + case, int(rng.integers(0, 1 << 20)), P, L, n_pal)
    off_in, off_out = int(rng.choice([0, 0, 1, 3])), int(rng.choice([0, 0, 1, 2]))
    spec = bool(rng.integers(0, 2))
    out = {"spectra": _out(P, n, off_out) if spec else None, "xyz": _out(P, 3, off_out), "rgb": _out(P, 3, off_out)}
    codec.shade_spectral(_place(torch.from_numpy(pal).cuda(), off_in), lts, _place(idx, off_in), _place(cosv, off_in),
                         spectra=spec, out=out)
    ref = [np.zeros((P, d), np.float32) for d in (n, 3, 3)]
    orc.orc_shade_spectral(n, cmf_matrix(n), grid(n)[1], pal, lts, L, host(idx).view(np.uint32), host(cosv), P, *ref)
    tag = f"case {case}: n={n} L={L} n_pal={n_pal} P={P} in+{off_in} out+{off_out} spectra={spec}"
    for key, r in zip(("spectra", "xyz", "rgb"), ref):
        if out[key] is not None:
            e = rel_err(host(out[key]), r)
            assert e <= TOL, f"{tag} {key}: rel err {e:.3e}"


@pytest.mark.parametrize("case", range(CASES // 2))
def test_random_roundtrip(api, ctx, orc, case):
    rng = np.random.default_rng(9000 + case)
    n, k, _, _, rows = _draw(rng)
    E, D = synth.codec_weights(277 + case, k, n)
    codec = api.Codec(ctx, E, D)
    S = api.synth_gm_spectra(ctx, 277 + case, "sweep.spectra", int(rng.integers(0, 1 << 20)), rows, n)
    off_in, off_out = int(rng.choice([0, 0, 1, 3])), int(rng.choice([0, 0, 1, 2]))
    want = {key: bool(rng.integers(0, 2)) for key in ("codes", "spectra", "xyz", "rgb")}
    if not any(want.values()):
        want["codes"] = True
    widths = {"codes": k, "spectra": n, "xyz": 3, "rgb": 3}
    out = {key: _out(rows, widths[key], off_out) if want[key] else None for key in widths}
    codec.roundtrip(_place(S, off_in), out=out)
    ref = [np.zeros((rows, widths[key]), np.float32) for key in ("codes", "spectra", "xyz", "rgb")]
    orc.orc_codec_roundtrip(E, D, k, n, cmf_matrix(n), grid(n)[1], host(S), rows, *ref)
    tag = f"case {case}: n={n} k={k} rows={rows} in+{off_in} out+{off_out}"
    for key, r in zip(("codes", "spectra", "xyz", "rgb"), ref):
        if want[key]:
            e = rel_err(host(out[key]), r)
            assert e <= TOL, f"{tag} {key}: rel err {e:.3e}"


@pytest.mark.parametrize("case", range(CASES // 2))
def test_random_chain(api, ctx, orc, case):
    """Latent chain: random k, table sizes, samples per pixel (multiples of 8: the ABI's constraint),
    pixel counts (ragged pixel quads) and throughput ranges."""
    rng = np.random.default_rng(13000 + case)
    k = int(rng.choice([3, 6, 6, 9]))
    n_pal = int(rng.choice([1, 2, 37, 100, 255, 256]))
    n_ill = int(rng.choice([1, 5, 16, 200, 256]))
    spp = 8 * int(rng.choice([1, 2, 3, 4, 8, 8, 9, 17]))
    P = int(rng.choice([1, 3, 4, 5, 127, 777, 2049]))
    E, D = synth.codec_weights(377 + case, k, 81)
    codec = api.Codec(ctx, E, D)
    pal_codes = codec.encode(torch.from_numpy(synth.palette(377 + case, n_pal, 81)).cuda())
    ill_codes = codec.encode(torch.from_numpy(synth.lights(377 + case, n_ill, 81, purpose="scene.illuminants")).cuda())
    ph = rng.integers(0, n_pal, (P, spp, 4), dtype=np.uint8)
    ih = rng.integers(0, n_ill, (P, spp), dtype=np.uint8)
    th = rng.uniform(0.0, float(rng.choice([0.5, 1.0, 1.5])), (P, spp, 4)).astype(np.float32)
    out = codec.multibounce_latent(pal_codes, ill_codes, torch.from_numpy(ph).cuda(), torch.from_numpy(ih).cuda(),
                                   torch.from_numpy(th).cuda(), latent=True)
    ctx.synchronize()
    lat = np.zeros((P, k), np.float32)
    orc.orc_chain(k, host(pal_codes), host(ill_codes), ph, ih, th, P, spp, 4, lat)
    tag = f"case {case}: k={k} n_pal={n_pal} n_ill={n_ill} spp={spp} P={P}"
    e = rel_err(host(out["latent"]), lat)
    assert e <= TOL, f"{tag} latent: rel err {e:.3e}"
    S2, X, R = np.zeros((P, 81), np.float32), np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
    orc.orc_decode(D, k, 81, lat, P, S2)
    orc.orc_spectra_to_outputs(cmf_matrix(81), grid(81)[1], 81, S2, P, X, R)
    for key, r in (("xyz", X), ("rgb", R)):
        e = rel_err(host(out[key]), r)
        assert e <= TOL, f"{tag} {key}: rel err {e:.3e}"


@pytest.mark.parametrize("case", range(CASES // 4))
def test_random_mlp_and_loss(api, ctx, orc, case):
    rng = np.random.default_rng(17000 + case)
    k = int(rng.choice([3, 6, 9]))
    P = int(rng.choice([1, 127, 128, 129, 1000, 128 * 37 + 5, 128 * 450]))
    w = synth.mlp_weights(477 + case, k, 64)
    mlp = api.CodeMLP(ctx, w)
    off = int(rng.choice([0, 0, 1, 4]))
    rgb = _place(api.synth_uniform(ctx, 477 + case, "sweep.rgb", 0, P * 3).reshape(P, 3), off)
    got = host(mlp.forward(rgb))
    ref = np.zeros((P, k), np.float32)
    orc.orc_mlp_forward(host(rgb), P, 64, k, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"], w["b3"], ref)
    e = rel_err(got, ref)
    assert e <= 1e-2 and np.all(got >= 0), f"case {case}: mlp k={k} P={P} rgb+{off}: rel err {e:.3e}"

    n = int(rng.choice([81, 81, 47]))
    pairs = int(rng.choice([1, 63, 64, 65, 1000, 64 * 50 + 1]))
    E, D = synth.codec_weights(477 + case, k, n)
    codec = api.Codec(ctx, E, D)
    A = _place(api.synth_gm_spectra(ctx, 477 + case, "sweep.a", 0, pairs, n), off)
    B = _place(api.synth_gm_spectra(ctx, 477 + case, "sweep.b", 0, pairs, n), off)
    got = float(host(codec.hadamard_loss(A, B))[0])
    want = orc.orc_hadamard_loss(E, D, k, n, host(A), host(B), pairs)
    assert got == pytest.approx(want, rel=TOL), f"case {case}: loss n={n} k={k} pairs={pairs} +{off}"


def test_random_call_sequence_on_one_context(api, ctx, orc):
    """State carried between calls (scratch buffers that grow, cached launch configurations, the
    frame pipeline's slots): one context and one codec per k serve a random sequence of host-buffer
    and device calls with sizes going up and down; every result is compared with the device path
    (bit-identical: the same kernels) and spot-checked against the oracle."""
    rng = np.random.default_rng(4711)
    codecs = {}
    for k in (6, 9, 3):
        E, D = synth.codec_weights(900 + k, k, 81)
        codecs[k] = (api.Codec(ctx, E, D), E, D)
    group = api.Group([0, 0, 0], "fused")
    group_k = None
    for step in range(40):
        k = int(rng.choice([6, 6, 9, 3]))
        codec, E, D = codecs[k]
        L = int(rng.choice([8, 8, 32, 5]))
        n_pal = int(rng.choice([256, 256, 17]))
        W, H = int(rng.choice([1, 64, 333, 1920])), int(rng.choice([1, 2, 7, 67, 300]))
        P = W * H
        pal = synth.palette(900 + step, n_pal, 81)
        lts = synth.lights(900 + step, L, 81)
        pal_codes = codec.encode(torch.from_numpy(pal).cuda())
        light_codes = codec.encode(torch.from_numpy(lts).cuda()).cpu().numpy()
        idx, cosv = api.synth_gbuffer(ctx, 900 + step, 0, P, L, n_pal)
        dev = codec.shade_latent(pal_codes, light_codes, idx, cosv)
        want_xyz, want_rgb = host(dev["xyz"]), host(dev["rgb"])
        h_pal, h_idx, h_cos = host(pal_codes), host(idx), host(cosv)
        kind = str(rng.choice(["host", "frames", "group", "roundtrip"]))
        tag = f"step {step}: {kind} k={k} L={L} n_pal={n_pal} {W}x{H}"
        if kind == "host":
            xyz, rgb = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
            codec.shade_latent_host(h_pal, light_codes, h_idx, h_cos, xyz, rgb)
            assert np.array_equal(xyz, want_xyz) and np.array_equal(rgb, want_rgb), tag
        elif kind == "frames":
            nf = int(rng.integers(1, 5))
            frames = [(h_idx, h_cos, np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)) for _ in range(nf)]
            codec.shade_latent_host_frames(h_pal, light_codes, frames)
            for f in frames:
                assert np.array_equal(f[2], want_xyz) and np.array_equal(f[3], want_rgb), tag
        elif kind == "group":
            if group_k != k:
                group.set_codec(E, D)
                group_k = k
            xyz, rgb = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
            group.shade_latent_host(h_pal, light_codes, h_idx, h_cos, W, H, xyz, rgb)
            assert np.array_equal(xyz, want_xyz) and np.array_equal(rgb, want_rgb), tag
        else:
            rows = max(1, P // 7)
            S = host(api.synth_gm_spectra(ctx, 900 + step, "seq.spectra", 0, rows, 81))
            Z, S2 = np.zeros((rows, k), np.float32), np.zeros((rows, 81), np.float32)
            X, R = np.zeros((rows, 3), np.float32), np.zeros((rows, 3), np.float32)
            codec.roundtrip_host(S, Z, S2, X, R)
            ref = [np.zeros((rows, d), np.float32) for d in (k, 81, 3, 3)]
            orc.orc_codec_roundtrip(E, D, k, 81, cmf_matrix(81), grid(81)[1], S, rows, *ref)
            for name, got, r in zip(("codes", "spectra", "xyz", "rgb"), (Z, S2, X, R), ref):
                assert rel_err(got, r) <= TOL, f"{tag} {name}"
        if step % 8 == 0:  # the device path itself against the oracle
            ref = [np.zeros((P, d), np.float32) for d in (k, 81, 3, 3)]
            orc.orc_shade_latent(D, k, 81, cmf_matrix(81), grid(81)[1], h_pal, light_codes, L,
                                 h_idx.view(np.uint32), h_cos, P, *ref)
            assert rel_err(want_xyz, ref[2]) <= TOL and rel_err(want_rgb, ref[3]) <= TOL, tag


def _metric_images(rng, P, n):
    """Linear RGB / spectra with zeros, duplicates (percentile ties), negatives and a wide range."""
    a = (rng.lognormal(-1.0, 1.5, (P, 3)) * (rng.random((P, 3)) > 0.05)).astype(np.float32)
    if rng.random() < 0.5 and P > 4:  # many exact ties around the percentile
        a[rng.integers(0, P, P // 2)] = a[0]
    if rng.random() < 0.3:
        a[rng.integers(0, P, max(1, P // 10))] *= -1.0
    b = (a * rng.normal(1.0, 0.05, (P, 3))).astype(np.float32)
    s = (rng.random((P, n)) * rng.lognormal(0.0, 1.0, (P, 1))).astype(np.float32)
    return a, b, s


@pytest.mark.parametrize("case", range(CASES // 2))
def test_random_metric_tail(api, ctx, orc, case):
    """exposure_for (an exact order statistic), the 8-bit tone map and the per-pixel MSE map are
    bit-exact; the Delta E report within 1e-12 (test_gpu_metrics.py's bars) -- at random pixel
    counts (around the radix-select block and pass boundaries), percentiles and exposures."""
    rng = np.random.default_rng(21000 + case)
    n = int(rng.choice([81, 81, 47]))
    P = int(rng.choice([1, 2, 3, 255, 256, 257, 1023, 1025, 4096, 65_537, 131_071, 262_145]))
    E, D = synth.codec_weights(577, 6, n)
    codec = api.Codec(ctx, E, D)
    a, b, s = _metric_images(rng, P, n)
    dev_ = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ybar = np.ascontiguousarray(cmf_matrix(n)[1])
    tag = f"case {case}: n={n} P={P}"
    for pct in (99.5, float(rng.uniform(0, 100)), float(rng.choice([0.0, 100.0, 50.0]))):
        assert api.exposure_for(codec, dev_(a), pct) == orc.orc_exposure_for(a, P, 3, None, grid(n)[1], pct), (tag, pct)
        assert api.exposure_for(codec, dev_(s), pct) == orc.orc_exposure_for(s, P, n, ybar, grid(n)[1], pct), (tag, pct)
    e = float(rng.choice([1.0, 0.37, 4.0, rng.uniform(0.01, 20.0)]))
    got = api.tonemap_srgb8(ctx, dev_(a), e).cpu().numpy().reshape(-1)
    want = np.zeros(P * 3, np.uint8)
    orc.orc_tonemap_srgb8(a, P, e, want)
    assert np.array_equal(got, want), f"{tag}: tone map, {int(np.sum(got != want))} bytes differ"
    mse, mean = api.error_map(codec, dev_(s), dev_(b))
    wmse = np.zeros(P, np.float32)
    wmean = orc.orc_error_map(s, n, b, 3, P, cmf_matrix(n), grid(n)[1], wmse)
    assert np.array_equal(mse.cpu().numpy(), wmse), f"{tag}: error map"
    assert mean == pytest.approx(wmean, rel=1e-12), tag
    rep = api.scene_color_report(codec, dev_(a), dev_(b))
    wrep = np.zeros(4)
    orc.orc_scene_color_report(a, 3, b, 3, P, cmf_matrix(n), grid(n)[1], wrep)
    assert rep["exposure"] == wrep[3], tag
    for key, w in (("mean_de76", wrep[0]), ("p95_de76", wrep[1]), ("mse", wrep[2])):
        assert rep[key] == pytest.approx(w, rel=1e-12), (tag, key)


@pytest.mark.parametrize("case", range(12))
def test_random_render_vs_compiled_reference(api, ctx, case):
    """The path tracer at random image sizes, sample counts, depths (fixed and
    Russian roulette), seeds and modes: images and shading-evaluation counts bit-identical to the
    compiled reference's render()."""
    import ctypes as C

    import oracle

    rng = np.random.default_rng(25000 + case)
    n = int(rng.choice([81, 47]))
    ref = oracle.reference(n)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    mode = str(rng.choice(["spectral", "latent", "rgb"]))
    k = int(rng.choice([3, 6, 9]))
    W, H = int(rng.integers(1, 70)), int(rng.integers(1, 50))
    spp = int(rng.choice([1, 2, 5, 8, 16]))
    depth = int(rng.choice([-1, 0, 1, 2, 3, 5]))
    seed = int(rng.integers(0, 1 << 31))
    block = bool(rng.integers(0, 2))
    multipass = mode == "latent" and depth >= 0 and bool(rng.integers(0, 2))
    E, D = synth.codec_weights(11 + case, k, n)
    codec = api.Codec(ctx, E, D)
    scene = synth.cornell_scene(n, block)
    got = api.render(codec, scene, mode, W, H, spp, depth, seed, multipass=multipass)
    sc, keep = api.scene_struct(scene, n)
    job = api.HcRenderJob(api.RENDER_MODES[mode], W, H, spp, depth, seed)
    ch = {"spectral": n, "latent": k, "rgb": 3}[mode]
    img = np.zeros((H, W, ch), np.float32)
    hashes = np.zeros(W * H, np.uint64)
    ev = C.c_uint64()
    rc = ref.ref_render(C.addressof(sc), C.addressof(job), k, E, D, int(multipass), img.reshape(-1), hashes,
                        C.byref(ev))
    assert rc == 0
    g = got["image"].cpu().numpy()
    tag = f"case {case}: {mode} n={n} k={k} {W}x{H} spp={spp} depth={depth} seed={seed} multipass={multipass}"
    assert g.shape == img.shape, tag
    assert np.array_equal(g, img), f"{tag}: {int(np.sum(g != img))} values differ"
    assert got["shading_evals"] == ev.value, tag


@pytest.mark.parametrize("case", range(16))
def test_random_training_step_vs_compiled_reference(api, ctx, case):
    """The codec training step at random batch sizes (around the reduction's
    30-row warps and ring slots), code sizes, betas and loss weights, with both softplus branches
    and zero rows: losses and gradients bit-identical to the compiled reference (47-sample grid,
    the grid its trainer is built for)."""
    import oracle

    ref = oracle.reference(47)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    N = 47
    rng = np.random.default_rng(29000 + case)
    k = int(rng.choice([3, 6, 9]))
    m = int(rng.choice([1, 2, 29, 30, 31, 59, 60, 61, 127, 128, 129, 999, 4097]))
    beta = float(rng.choice([1.0, 10.0, 25.0]))
    lw = tuple(float(x) for x in (rng.uniform(0, 2, 5) * (rng.random(5) > 0.3)))
    re_ = rng.uniform(-0.5, 0.5, (k, N)) / np.sqrt(N)
    rd = rng.uniform(-0.5, 0.5, (N, k)) / np.sqrt(k)
    re_[0, :3] = [40.0 / beta, -35.0 / beta, 0.0]  # beta * raw > 30 and < -30, and 0
    refl = rng.uniform(0, 1, (m, N))
    illum = rng.uniform(0, 1, (m, N)) * rng.uniform(0.5, 2.0, (m, 1))
    refl[rng.integers(0, m)] = 0.0
    losses, ge, gd = api.codec_train_grad(ctx, re_, rd, beta, torch.from_numpy(refl).cuda(),
                                          torch.from_numpy(illum).cuda(), loss_weights=lw)
    rge, rgd, rl = np.zeros(k * N), np.zeros(N * k), np.zeros(6)
    assert ref.ref_codec_gradients(k, beta, re_.reshape(-1), rd.reshape(-1), np.ascontiguousarray(refl.reshape(-1)),
                                   np.ascontiguousarray(illum.reshape(-1)), m, np.array(lw),
                                   rge.ctypes.data, rgd.ctypes.data, rl) == 0
    tag = f"case {case}: k={k} m={m} beta={beta} lw={lw}"
    assert ge.reshape(-1).tobytes() == rge.tobytes(), f"{tag}: encoder gradient"
    assert gd.reshape(-1).tobytes() == rgd.tobytes(), f"{tag}: decoder gradient"
    assert np.array(list(losses.values())).tobytes() == rl.tobytes(), f"{tag}: losses"


@pytest.mark.parametrize("case", range(CASES // 4))
def test_random_passes_and_small_entry_points(api, ctx, orc, case):
    """The k/3 three-channel passes + reassembly (bit-identical to the fused shade), encode /
    decode / spectra_to_xyz_rgb as separate calls and blockwise_hadamard, at random sizes."""
    rng = np.random.default_rng(33000 + case)
    n = int(rng.choice([81, 47]))
    k = int(rng.choice([3, 6, 9]))
    L = int(rng.choice([1, 8, 32, 11]))
    P = int(rng.choice([1, 5, 255, 257, 3001, 20_011]))
    E, D = synth.codec_weights(677 + case, k, n)
    codec = api.Codec(ctx, E, D)
    pal_codes = codec.encode(torch.from_numpy(synth.palette(677 + case, 256, n)).cuda())
    light_codes = codec.encode(torch.from_numpy(synth.lights(677 + case, L, n)).cuda()).cpu().numpy()
    idx, cosv = api.synth_gbuffer(ctx, 677 + case, 0, P, L, 256)
    fused = codec.shade_latent(pal_codes, light_codes, idx, cosv, latent=True)["latent"]
    passes = [codec.shade_latent_pass(b, pal_codes, light_codes, idx, cosv) for b in range(k // 3)]
    multi = api.reassemble(ctx, passes)
    tag = f"case {case}: n={n} k={k} L={L} P={P}"
    assert torch.equal(multi, fused), f"{tag}: passes + reassembly differ from the fused shade"

    S = api.synth_gm_spectra(ctx, 677 + case, "small.spectra", 0, P, n)
    Z = codec.encode(S)
    Zr = np.zeros((P, k), np.float32)
    orc.orc_encode(E, k, n, host(S), P, None, Zr)
    assert rel_err(host(Z), Zr) <= TOL, f"{tag}: encode"
    dec = codec.decode(torch.from_numpy(Zr).cuda(), spectra=True, xyz=True, rgb=True)
    Sr, X, R = np.zeros((P, n), np.float32), np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
    orc.orc_decode(D, k, n, Zr, P, Sr)
    orc.orc_spectra_to_outputs(cmf_matrix(n), grid(n)[1], n, Sr, P, X, R)
    for name, got, r in (("spectra", dec["spectra"], Sr), ("xyz", dec["xyz"], X), ("rgb", dec["rgb"], R)):
        assert rel_err(host(got), r) <= TOL, f"{tag}: decode {name}"
    proj = codec.spectra_to_xyz_rgb(S)
    orc.orc_spectra_to_outputs(cmf_matrix(n), grid(n)[1], n, host(S), P, X, R)
    assert rel_err(host(proj["xyz"]), X) <= TOL and rel_err(host(proj["rgb"]), R) <= TOL, f"{tag}: project"
    A = api.synth_uniform(ctx, 677 + case, "small.a", 0, P * k).reshape(P, k)
    B = api.synth_uniform(ctx, 677 + case, "small.b", 0, P * k).reshape(P, k)
    assert np.array_equal(host(api.blockwise_hadamard(ctx, A, B)), host(A) * host(B)), f"{tag}: hadamard"


@pytest.mark.parametrize("case", range(12))
def test_random_encode_decode_tools_vs_compiled_reference(api, ctx, tmp_path, case):
    """The `encode` / `decode` tools on random measurement grids (regular and
    irregular, narrower and wider than the codec's band, 1 to ~700 samples), row counts, id columns,
    value precisions, blank lines and k: output files byte-identical to the compiled reference."""
    import ctypes

    import oracle

    ref = oracle.reference(47)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    N = 47
    rng = np.random.default_rng(37000 + case)
    k = int(rng.choice([3, 6, 9]))
    re_ = rng.uniform(-0.5, 0.5, (k, N)) / np.sqrt(N)
    rd = rng.uniform(-0.5, 0.5, (N, k)) / np.sqrt(N)
    codec = api.Codec.from_raw(ctx, re_, rd, beta=10.0)
    m = int(rng.choice([1, 2, 17, 61, 95, 300, 700]))
    lo = float(rng.uniform(300, 450))
    if rng.random() < 0.5:
        wl = lo + np.arange(m) * float(rng.choice([0.5, 1.0, 2.0, 5.0, 10.0]))
    else:
        wl = np.cumsum(np.r_[lo, rng.uniform(0.3, 9.0, m - 1)]) if m > 1 else np.array([lo])
    rows = int(rng.choice([1, 2, 33, 257, 1500]))
    ids = bool(rng.integers(0, 2))
    head = (["id"] if ids else []) + ["%.9g" % w for w in wl]
    lines = [",".join(head)]
    for r in range(rows):
        v = np.clip(rng.normal(0.5, 0.3, m), 0, None) * rng.uniform(0.1, 3.0)
        cells = (["s%05d" % r] if ids else []) + ["%.*g" % (int(rng.integers(3, 17)), x) for x in v]
        lines.append(", ".join(cells) if r % 7 == 0 else ",".join(cells))
        if r % 11 == 0:
            lines.append("  ")
    data = ("\n".join(lines) + "\n").encode()
    src, codes_ref, spec_ref = tmp_path / "s.csv", tmp_path / "codes.csv", tmp_path / "dec.csv"
    src.write_bytes(data)
    err = ctypes.create_string_buffer(512)
    flat = lambda a: np.ascontiguousarray(a.reshape(-1))
    tag = f"case {case}: k={k} grid={m} samples from {lo:.1f} nm, rows={rows}, ids={ids}"
    assert ref.ref_run_encode(str(src).encode(), k, 10.0, flat(re_), flat(rd), str(codes_ref).encode(), err,
                              512) == 0, (tag, err.value)
    got = api.encode_tool(codec, data)
    assert got == codes_ref.read_bytes(), f"{tag}: encode tool output differs"
    assert ref.ref_run_decode(str(codes_ref).encode(), k, 10.0, flat(re_), flat(rd), str(spec_ref).encode(), err,
                              512) == 0, (tag, err.value)
    assert api.decode_tool(codec, got) == spec_ref.read_bytes(), f"{tag}: decode tool output differs"


@pytest.mark.parametrize("case", range(12))
def test_random_upsampler_vs_compiled_reference(api, ctx, case):
    """The reference's fp64 SiLU upsampler (upsampler.cpp:42-72, :170-190) at random widths, code
    sizes, texel counts and input ranges: codes within 1e-13 of the compiled reference (SiLU's exp
    is CUDA's), clamp counts exact."""
    import ctypes

    import oracle

    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    rng = np.random.default_rng(41000 + case)
    k = int(rng.choice([3, 6, 9, 12]))
    hidden = int(rng.choice([1, 7, 17, 32, 64, 100, 128, 257, 512]))
    P = int(rng.choice([1, 31, 32, 33, 1000, 4097]))
    clamp = bool(rng.integers(0, 2))
    lim = lambda fi, fo: np.sqrt(6.0 / (fi + fo))  # noqa: E731
    w = {"w1": rng.uniform(-lim(3, hidden), lim(3, hidden), (hidden, 3)), "b1": rng.normal(0, 0.1, hidden),
         "w2": rng.uniform(-lim(hidden, hidden), lim(hidden, hidden), (hidden, hidden)),
         "b2": rng.normal(0, 0.1, hidden),
         "w3": rng.uniform(-lim(hidden, k), lim(hidden, k), (k, hidden)), "b3": rng.normal(0, 0.1, k)}
    rgb = rng.uniform(-0.1, float(rng.choice([1.0, 1.2, 50.0])), (P, 3))
    got, n = api.Upsampler(ctx, w).forward(torch.from_numpy(rgb).cuda(), clamp=clamp)
    got = got.cpu().numpy()
    want = np.zeros((P, k))
    rn = ctypes.c_uint64(0)
    arrs = [np.ascontiguousarray(w[x].reshape(-1)) for x in api.Upsampler.KEYS]
    assert ref.ref_upsample(k, hidden, *arrs, np.ascontiguousarray(rgb.reshape(-1)), P, int(clamp),
                            want.reshape(-1), ctypes.byref(rn)) == 0
    tag = f"case {case}: k={k} hidden={hidden} P={P} clamp={clamp}"
    assert n == rn.value, f"{tag}: clamp count {n} vs {rn.value}"
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13 * max(np.abs(want).max(), 1e-300), err_msg=tag)
