"""GPU parity: every kernel of libhadacodec_b200.so (through the C ABI) against
the oracle (oracle/hc_oracle.c, pinned bit-exact to the compiled reference in
test_oracle.py) and the reference's golden fixtures.

Tolerances (BASELINE.json north_star): fp32 codes / spectra / XYZ / sRGB within
1e-5 relative, denominator max(|ref|, ||ref_row||_inf); bf16 MLP within 1e-2.
Integer work (generators, indices) bit-exact.
"""
import numpy as np
import pytest

from conftest import max_abs, rel_err
from paper_2602_18741_b200 import synth
from paper_2602_18741_b200.colorimetry import cmf_matrix, grid

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5
MLP_TOL = 1e-2
SEED = 31337


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def _codec(api, ctx, k, n=81, seed=SEED):
    E, D = synth.codec_weights(seed, k, n)
    return api.Codec(ctx, E, D), E, D


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def _check(name, got, ref, tol=TOL):
    e = rel_err(got, ref)
    print(f"{name}: max_rel={e:.3e} max_abs={max_abs(got, ref):.3e}")
    assert e <= tol, f"{name}: rel err {e:.3e} > {tol}"


# ----------------------------------------------------------------- library / generators
def test_library_is_the_cuda_path(api, ctx):
    from paper_2602_18741_b200 import _lib

    assert _lib.LIB_PATH.exists()
    assert b"sm_100a" in _lib.lib().hc_version()
    before = ctx.launches
    api.synth_uniform(ctx, 1, "x", 0, 1024)
    assert ctx.launches == before + 1


def test_device_generators_match_numpy_bit_exact(api, ctx):
    idx, cosv = api.synth_gbuffer(ctx, SEED, 1000, 4097, 8, 256)
    ri, rc = synth.gbuffer_np(SEED, 1000, 4097, 8, 256)
    assert np.array_equal(host(idx).view(np.uint32), ri)
    assert np.array_equal(host(cosv), rc)
    pidx, iidx, tw = api.synth_chain(ctx, SEED, 77, 33, 64, 256, 16)
    rp, ri2, rt = synth.chain_np(SEED, 77, 33, 64, 256, 16)
    assert np.array_equal(host(pidx), rp) and np.array_equal(host(iidx), ri2) and np.array_equal(host(tw), rt)
    u = api.synth_uniform(ctx, SEED, "mlp.input", 5, 999)
    assert np.array_equal(host(u), synth.uniform_np(SEED, "mlp.input", 5, 999))


def test_device_gm_spectra_match_host_generator(api, ctx):
    for n in (81, 47):
        dev = host(api.synth_gm_spectra(ctx, SEED, "codec.spectra", 123, 40, n))
        ref = synth.gm_spectra_ctr(SEED, "codec.spectra", 123, 40, n)
        assert max_abs(dev, ref) <= 1e-7  # double exp on device vs glibc; after the fp32 cast


# ----------------------------------------------------------------- codec (config 1)
def test_roundtrip_golden(api, ctx, golden):
    codec = api.Codec(ctx, golden["E6"], golden["D6"])
    S = torch.from_numpy(golden["c1_S"]).cuda()
    out = codec.roundtrip(S)
    for key, g in (("codes", "c1_Z"), ("spectra", "c1_S2"), ("xyz", "c1_xyz"), ("rgb", "c1_rgb")):
        _check(f"golden c1 {key}", host(out[key]), golden[g])


@pytest.mark.parametrize("n,k", [(81, 6), (81, 9), (81, 3), (47, 6), (47, 9)])
@pytest.mark.parametrize("rows", [1, 129, 20011])
def test_roundtrip_vs_oracle(api, ctx, orc, n, k, rows):
    codec, E, D = _codec(api, ctx, k, n)
    S = api.synth_gm_spectra(ctx, SEED, "codec.spectra", 0, rows, n)
    out = codec.roundtrip(S)
    Sh = host(S)
    ref = [np.zeros((rows, d), np.float32) for d in (k, n, 3, 3)]
    orc.orc_codec_roundtrip(E, D, k, n, cmf_matrix(n), grid(n)[1], Sh, rows, *ref)
    for key, r in zip(("codes", "spectra", "xyz", "rgb"), ref):
        _check(f"roundtrip n={n} k={k} rows={rows} {key}", host(out[key]), r)


def test_roundtrip_unaligned_and_partial_outputs(api, ctx, orc):
    codec, E, D = _codec(api, ctx, 6)
    rows = 1001
    buf = api.synth_gm_spectra(ctx, SEED, "codec.spectra", 0, rows + 1, 81).reshape(-1)
    S = buf[1:1 + rows * 81]  # 4-byte aligned only -> generic (non-TMA) path
    out = codec.roundtrip(S, codes=False, spectra=False)
    ref = [np.zeros((rows, d), np.float32) for d in (6, 81, 3, 3)]
    orc.orc_codec_roundtrip(E, D, 6, 81, cmf_matrix(81), grid(81)[1], host(S).reshape(rows, 81), rows, *ref)
    assert out["codes"] is None and out["spectra"] is None
    _check("unaligned xyz", host(out["xyz"]), ref[2])
    _check("unaligned rgb", host(out["rgb"]), ref[3])


def test_encode_decode_project_vs_oracle(api, ctx, orc):
    codec, E, D = _codec(api, ctx, 9)
    rows = 5003
    S = api.synth_gm_spectra(ctx, SEED, "codec.spectra", 9, rows, 81)
    Z = codec.encode(S)
    Zr = np.zeros((rows, 9), np.float32)
    orc.orc_encode(E, 9, 81, host(S), rows, None, Zr)
    _check("encode", host(Z), Zr)
    dec = codec.decode(torch.from_numpy(Zr).cuda(), spectra=True, xyz=True, rgb=True)
    Sr = np.zeros((rows, 81), np.float32)
    orc.orc_decode(D, 9, 81, Zr, rows, Sr)
    X, R = np.zeros((rows, 3), np.float32), np.zeros((rows, 3), np.float32)
    orc.orc_spectra_to_outputs(cmf_matrix(81), grid(81)[1], 81, Sr, rows, X, R)
    _check("decode spectra", host(dec["spectra"]), Sr)
    _check("decode xyz", host(dec["xyz"]), X)
    _check("decode rgb", host(dec["rgb"]), R)
    proj = codec.spectra_to_xyz_rgb(S)
    X2, R2 = np.zeros((rows, 3), np.float32), np.zeros((rows, 3), np.float32)
    orc.orc_spectra_to_outputs(cmf_matrix(81), grid(81)[1], 81, host(S), rows, X2, R2)
    _check("project xyz", host(proj["xyz"]), X2)
    _check("project rgb", host(proj["rgb"]), R2)


def test_decode_rejects_negative_codes(api, ctx):
    codec, _, _ = _codec(api, ctx, 6)
    Z = torch.tensor([[0.1, 0.2, 0.3, 0.4, 0.5, 0.6]], device="cuda")
    codec.decode(Z, check_negative=True)
    Z[0, 2] = -1e-9
    with pytest.raises(ArithmeticError):
        codec.decode(Z, check_negative=True)
    codec.decode(Z, check_negative=False)  # decode_image does not check (renderer.cpp:661-690)
    ctx.synchronize()


def test_codec_validation(api, ctx):
    E, D = synth.codec_weights(1, 6, 81)
    with pytest.raises(ValueError):
        api.Codec(ctx, E[:5], D[:, :5])  # k = 5 not a multiple of 3 (validate, codec.cpp:111-135)
    with pytest.raises(ValueError):
        api.Codec(ctx, E, D[:, :3])


def test_codec_from_raw_softplus(api, ctx, kats):
    rng = np.random.default_rng(3)
    raw_e = rng.uniform(-0.3, 0.3, (6, 47))
    raw_d = rng.uniform(-0.3, 0.3, (47, 6))
    c = api.Codec.from_raw(ctx, raw_e, raw_d, beta=10.0)
    assert np.all(c.E > 0) and np.all(c.D > 0)  # test_codec.cpp:70-79
    S = torch.rand(17, 47, device="cuda")
    Z = host(c.encode(S))
    np.testing.assert_allclose(Z, host(S).astype(np.float64) @ c.E.T.astype(np.float64), rtol=1e-5)


def test_encode_linearity(api, ctx):
    """Scaling and addition preserving (test_codec.cpp:113-137), at fp32 tolerance."""
    codec, _, _ = _codec(api, ctx, 6)
    a = api.synth_gm_spectra(ctx, 1, "a", 0, 4096, 81)
    b = api.synth_gm_spectra(ctx, 1, "b", 0, 4096, 81)
    za, zb, zs = codec.encode(a), codec.encode(b), codec.encode(a + b)
    z3 = codec.encode(a * 2.5)
    _check("linearity add", host(zs), host(za) + host(zb), 2e-6)
    _check("linearity scale", host(z3), 2.5 * host(za), 2e-6)


def test_blockwise_hadamard_kat(api, ctx, kats):
    h = kats["hadamard"]
    a = torch.tensor([h["a"]], device="cuda")
    b = torch.tensor([h["b"]], device="cuda")
    assert host(api.blockwise_hadamard(ctx, a, b)).tolist()[0] == h["expect"]
    with pytest.raises(ValueError):
        api.blockwise_hadamard(ctx, a, b[:, :3])
    blocks = api.split_blocks(np.array(h["a"]))
    assert len(blocks) == 2 and list(api.join_blocks(blocks)) == h["a"]


# ----------------------------------------------------------------- shading (configs 2 / 3)
def _scene(api, ctx, k, L, n=81):
    codec, E, D = _codec(api, ctx, k, n)
    pal = synth.palette(SEED, 256, n)
    lts = synth.lights(SEED, L, n)
    pal_d = torch.from_numpy(pal).cuda()
    pal_codes = codec.encode(pal_d)
    light_codes = host(codec.encode(torch.from_numpy(lts).cuda()))
    return codec, E, D, pal, lts, pal_d, pal_codes, light_codes


@pytest.mark.parametrize("k,L,P,spec,n", [(6, 8, 50_003, False, 81), (6, 8, 4096, True, 81),
                                          (9, 32, 20_011, True, 81), (9, 32, 777, False, 81), (3, 8, 1000, True, 81),
                                          (6, 5, 3001, True, 81), (9, 1, 1000, False, 81), (6, 64, 513, True, 81),
                                          (6, 8, 5000, True, 47), (9, 32, 3001, False, 47), (3, 8, 777, True, 47),
                                          (9, 13, 2000, True, 47)])
def test_shade_latent_vs_oracle(api, ctx, orc, k, L, P, spec, n):
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, k, L, n)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, P, L, 256)
    out = codec.shade_latent(pal_codes, light_codes, idx, cosv, latent=True, spectra=spec)
    ref = [np.zeros((P, d), np.float32) for d in (k, n, 3, 3)]
    orc.orc_shade_latent(D, k, n, cmf_matrix(n), grid(n)[1], host(pal_codes), light_codes, L,
                         host(idx).view(np.uint32), host(cosv), P, *ref)
    _check(f"latent k={k} L={L}", host(out["latent"]), ref[0])
    if spec:
        _check(f"spectra k={k} L={L}", host(out["spectra"]), ref[1])
    _check(f"xyz k={k} L={L}", host(out["xyz"]), ref[2])
    _check(f"rgb k={k} L={L}", host(out["rgb"]), ref[3])


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("k,L,P", [(6, 8, 300_007), (9, 32, 131_072), (3, 5, 1001)])
def test_shade_latent_host_buffers(api, ctx, k, L, P, pinned):
    """hc_shade_latent_host (chunked H2D -> kernel -> D2H pipeline over the aux streams,
    ragged last chunk, pinned or pageable host buffers) == the device-resident call."""
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, k, L)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 11, P, L, 256)
    dev = codec.shade_latent(pal_codes, light_codes, idx, cosv)
    if pinned:
        xyz_t, rgb_t = torch.zeros(P, 3).pin_memory(), torch.zeros(P, 3).pin_memory()
        xyz, rgb = xyz_t.numpy(), rgb_t.numpy()
    else:
        xyz, rgb = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
    codec.shade_latent_host(host(pal_codes), light_codes, host(idx), host(cosv), xyz, rgb)
    assert np.array_equal(xyz, host(dev["xyz"])) and np.array_equal(rgb, host(dev["rgb"]))


@pytest.mark.parametrize("k,L,P,nf", [(6, 8, 600_011, 3), (9, 32, 65_536, 5), (3, 5, 999, 4), (6, 8, 262_144, 1)])
def test_shade_latent_host_frames(api, ctx, k, L, P, nf):
    """hc_shade_latent_host_frames: one pipeline across a frame stream (chunk slots reused
    across frame boundaries, ragged last chunk, frames of different G-buffers, a frame
    without xyz) == one device-resident call per frame, bit for bit."""
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, k, L)
    frames, want = [], []
    for f in range(nf):
        idx, cosv = api.synth_gbuffer(ctx, SEED + f, 7 * f, P, L, 256)
        dev = codec.shade_latent(pal_codes, light_codes, idx, cosv)
        want.append((host(dev["xyz"]), host(dev["rgb"])))
        xyz = None if (f == 1 and nf > 1) else torch.zeros(P, 3).pin_memory().numpy()
        frames.append((host(idx).view(np.uint32), host(cosv), xyz, torch.zeros(P, 3).pin_memory().numpy()))
    codec.shade_latent_host_frames(host(pal_codes), light_codes, frames)
    for f in range(nf):
        if frames[f][2] is not None:
            assert np.array_equal(frames[f][2], want[f][0]), f"frame {f} xyz"
        assert np.array_equal(frames[f][3], want[f][1]), f"frame {f} rgb"


def test_roundtrip_host_buffers(api, ctx, orc):
    codec, E, D = _codec(api, ctx, 6)
    rows = 20_001
    S = host(api.synth_gm_spectra(ctx, SEED, "host.rt", 0, rows, 81))
    dev = codec.roundtrip(torch.from_numpy(S).cuda())
    Z, S2, xyz, rgb = (np.zeros((rows, d), np.float32) for d in (6, 81, 3, 3))
    codec.roundtrip_host(S, Z, S2, xyz, rgb)
    for key, got in (("codes", Z), ("spectra", S2), ("xyz", xyz), ("rgb", rgb)):
        assert np.array_equal(got, host(dev[key])), key


def test_shade_golden(api, ctx, golden):
    for tag, k, L in (("c2", 6, 8), ("c3", 9, 32)):
        codec = api.Codec(ctx, golden[f"E{k}"], golden[f"D{k}"])
        idx = torch.from_numpy(golden[f"{tag}_idx"].view(np.int32)).cuda()
        cosv = torch.from_numpy(np.ascontiguousarray(golden[f"{tag}_cos"])).cuda()
        pc = torch.from_numpy(golden[f"{tag}_palcodes"]).cuda()
        out = codec.shade_latent(pc, golden[f"{tag}_lightcodes"], idx, cosv, latent=True, spectra=True)
        for key in ("latent", "xyz", "rgb"):
            _check(f"golden {tag} {key}", host(out[key]), golden[f"{tag}_{key}"])
        _check(f"golden {tag} spectra", host(out["spectra"]), golden[f"{tag}_S2"])
        nv = codec.shade_spectral(torch.from_numpy(golden["palette"]).cuda(), golden[f"{tag}_lights"], idx, cosv,
                                  spectra=True)
        _check(f"golden {tag} naive spectra", host(nv["spectra"]), golden[f"{tag}_naive_S"])
        _check(f"golden {tag} naive xyz", host(nv["xyz"]), golden[f"{tag}_naive_xyz"])
        _check(f"golden {tag} naive rgb", host(nv["rgb"]), golden[f"{tag}_naive_rgb"])


@pytest.mark.parametrize("k,L", [(6, 8), (9, 32)])
def test_multipass_equals_fused(api, ctx, k, L):
    """render_latent_multipass == single k-channel render (renderer.hpp:103-105)."""
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, k, L)
    P = 10_007
    idx, cosv = api.synth_gbuffer(ctx, SEED, 5, P, L, 256)
    fused = codec.shade_latent(pal_codes, light_codes, idx, cosv, latent=True)["latent"]
    passes = [codec.shade_latent_pass(b, pal_codes, light_codes, idx, cosv) for b in range(k // 3)]
    multi = api.reassemble(ctx, passes)
    assert np.array_equal(host(multi), host(fused))


@pytest.mark.parametrize("L,P,spec,n", [(8, 30_001, False, 81), (32, 5000, True, 81), (8, 2048, True, 81),
                                        (3, 1001, True, 81), (17, 999, False, 81), (8, 4099, True, 47),
                                        (32, 1000, False, 47), (32, 777, False, 81), (32, 31, True, 81),
                                        (32, 40_003, True, 81)])
def test_shade_spectral_vs_oracle(api, ctx, orc, L, P, spec, n):
    codec, E, D, pal, lts, pal_d, _, _ = _scene(api, ctx, 6, L, n)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 3, P, L, 256)
    out = codec.shade_spectral(pal_d, lts, idx, cosv, spectra=spec)
    ref = [np.zeros((P, d), np.float32) for d in (n, 3, 3)]
    orc.orc_shade_spectral(n, cmf_matrix(n), grid(n)[1], pal, lts, L, host(idx).view(np.uint32), host(cosv), P,
                           *ref)
    if spec:
        _check(f"naive spectra L={L}", host(out["spectra"]), ref[0])
    _check(f"naive xyz L={L}", host(out["xyz"]), ref[1])
    _check(f"naive rgb L={L}", host(out["rgb"]), ref[2])


def test_latent_tracks_naive_on_shared_scene(api, ctx):
    """Same scene through both paths: the codec approximation error is finite and
    bounded (not a parity claim; the paper's colour comparison)."""
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, 6, 8)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, 4096, 8, 256)
    lat = host(codec.shade_latent(pal_codes, light_codes, idx, cosv)["xyz"])
    nv = host(codec.shade_spectral(pal_d, lts, idx, cosv)["xyz"])
    assert np.all(np.isfinite(lat)) and np.all(np.isfinite(nv))
    assert np.corrcoef(lat[:, 1], nv[:, 1])[0, 1] > 0.5


@pytest.mark.parametrize("L,spec", [(32, True), (32, False), (8, False)])
def test_shade_spectral_index_out_of_range_is_reported(api, ctx, L, spec):
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, 6, L)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, 1024, L, 256)
    idx[1000] = 256
    codec.shade_spectral(pal_d, lts, idx, cosv, spectra=spec)
    with pytest.raises(ValueError):
        ctx.synchronize()


def test_shade_index_out_of_range_is_reported(api, ctx):
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, 6, 8)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, 1024, 8, 256)
    idx[17] = 300
    codec.shade_latent(pal_codes[:256], light_codes, idx, cosv)
    with pytest.raises(ValueError):
        ctx.synchronize()


def test_empty_inputs(api, ctx):
    codec, E, D, pal, lts, pal_d, pal_codes, light_codes = _scene(api, ctx, 6, 8)
    idx = torch.empty(0, dtype=torch.int32, device="cuda")
    cosv = torch.empty(0, 8, device="cuda")
    before = ctx.launches
    out = codec.shade_latent(pal_codes, light_codes, idx, cosv)
    out2 = codec.roundtrip(torch.empty(0, 81, device="cuda"))
    ctx.synchronize()
    assert out["xyz"].shape == (0, 3) and out2["codes"].shape == (0, 6)
    assert ctx.launches == before


# ----------------------------------------------------------------- multi-bounce (config 4)
@pytest.mark.parametrize("spp,k,n", [(64, 6, 81), (8, 6, 81), (16, 9, 81), (32, 3, 81), (8, 3, 47), (64, 6, 47)])
def test_multibounce_vs_oracle(api, ctx, orc, spp, k, n):
    codec, E, D, pal, _, pal_d, pal_codes, _ = _scene(api, ctx, k, 8, n)
    ill = synth.lights(SEED, 16, n, purpose="scene.illuminants")
    ill_d = torch.from_numpy(ill).cuda()
    ill_codes = codec.encode(ill_d)
    P = 1237
    pidx, iidx, tw = api.synth_chain(ctx, SEED, 0, P, spp, 256, 16)
    out = codec.multibounce_latent(pal_codes, ill_codes, pidx, iidx, tw, latent=True)
    ph, ih, th = host(pidx), host(iidx), host(tw)
    lat = np.zeros((P, k), np.float32)
    orc.orc_chain(k, host(pal_codes), host(ill_codes), ph, ih, th, P, spp, 4, lat)
    _check("chain latent", host(out["latent"]), lat)
    S2 = np.zeros((P, n), np.float32)
    X, R = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
    orc.orc_decode(D, k, n, lat, P, S2)
    orc.orc_spectra_to_outputs(cmf_matrix(n), grid(n)[1], n, S2, P, X, R)
    _check("chain xyz", host(out["xyz"]), X)
    _check("chain rgb", host(out["rgb"]), R)
    nv = codec.multibounce_spectral(pal_d, ill_d, pidx, iidx, tw)
    spec = np.zeros((P, n), np.float32)
    orc.orc_chain(n, pal, ill, ph, ih, th, P, spp, 4, spec)
    orc.orc_spectra_to_outputs(cmf_matrix(n), grid(n)[1], n, spec, P, X, R)
    _check("chain naive xyz", host(nv["xyz"]), X)
    _check("chain naive rgb", host(nv["rgb"]), R)


@pytest.mark.parametrize("n_pal,n_ill,spp,k", [(100, 5, 72, 6), (256, 200, 64, 6), (1, 1, 8, 6), (37, 16, 136, 6),
                                                (100, 5, 72, 3), (37, 16, 24, 9), (100, 5, 64, 6), (255, 16, 64, 6)])
def test_multibounce_small_tables(api, ctx, orc, n_pal, n_ill, spp, k):
    """Palettes / illuminant sets smaller than the u8 index range (the k = 6 kernel range-checks
    palette indices only when n_pal < 256), large illuminant sets, and spp with a sample tail
    (spp / 8 not a multiple of the 8-sample load group)."""
    codec, E, D = _codec(api, ctx, k)
    pal = synth.palette(SEED, n_pal, 81)
    ill = synth.lights(SEED, n_ill, 81, purpose="scene.illuminants")
    pal_codes = codec.encode(torch.from_numpy(pal).cuda())
    ill_codes = codec.encode(torch.from_numpy(ill).cuda())
    P = 777
    rng = np.random.default_rng(n_pal * 1000 + spp)
    ph = rng.integers(0, n_pal, (P, spp, 4), dtype=np.uint8)
    ih = rng.integers(0, n_ill, (P, spp), dtype=np.uint8)
    th = rng.uniform(0.0, 1.5, (P, spp, 4)).astype(np.float32)
    out = codec.multibounce_latent(pal_codes, ill_codes, torch.from_numpy(ph).cuda(), torch.from_numpy(ih).cuda(),
                                   torch.from_numpy(th).cuda(), latent=True)
    ctx.synchronize()
    lat = np.zeros((P, k), np.float32)
    orc.orc_chain(k, host(pal_codes), host(ill_codes), ph, ih, th, P, spp, 4, lat)
    _check(f"chain latent n_pal={n_pal} n_ill={n_ill} spp={spp}", host(out["latent"]), lat)


@pytest.mark.parametrize("offset", [1, 16])
def test_multibounce_unaligned_records(api, ctx, orc, offset):
    """k = 6 at spp = 64 takes the bulk-copy record path only for 16-byte aligned index streams;
    an illuminant-index stream at a 1-byte offset runs the LDG path, 16 bytes the bulk-copy path
    (ragged last pixel quad in both: P % 4 == 1)."""
    codec, E, D = _codec(api, ctx, 6)
    pal_codes = codec.encode(torch.from_numpy(synth.palette(SEED, 256, 81)).cuda())
    ill_codes = codec.encode(torch.from_numpy(synth.lights(SEED, 16, 81, purpose="scene.illuminants")).cuda())
    P, spp = 1001, 64
    rng = np.random.default_rng(offset)
    ph = rng.integers(0, 256, (P, spp, 4), dtype=np.uint8)
    ih = rng.integers(0, 16, (P, spp), dtype=np.uint8)
    th = rng.uniform(0.0, 1.5, (P, spp, 4)).astype(np.float32)
    buf = torch.empty(P * spp + offset, dtype=torch.uint8, device="cuda")
    iidx = buf[offset:].view(P, spp)
    iidx.copy_(torch.from_numpy(ih))
    out = codec.multibounce_latent(pal_codes, ill_codes, torch.from_numpy(ph).cuda(), iidx,
                                   torch.from_numpy(th).cuda(), latent=True)
    ctx.synchronize()
    lat = np.zeros((P, 6), np.float32)
    orc.orc_chain(6, host(pal_codes), host(ill_codes), ph, ih, th, P, spp, 4, lat)
    _check(f"chain latent iidx offset {offset}", host(out["latent"]), lat)


@pytest.mark.parametrize("which", ["pal", "ill"])
@pytest.mark.parametrize("k", [6, 9])
def test_multibounce_index_out_of_range_is_reported(api, ctx, which, k):
    codec, E, D = _codec(api, ctx, k)
    pal_codes = codec.encode(torch.from_numpy(synth.palette(SEED, 100, 81)).cuda())
    ill_codes = codec.encode(torch.from_numpy(synth.lights(SEED, 5, 81, purpose="scene.illuminants")).cuda())
    P, spp = 300, 64
    ph = np.zeros((P, spp, 4), np.uint8)
    ih = np.zeros((P, spp), np.uint8)
    if which == "pal":
        ph[123, 17, 2] = 100
    else:
        ih[299, 63] = 5
    th = np.full((P, spp, 4), 0.5, np.float32)
    codec.multibounce_latent(pal_codes, ill_codes, torch.from_numpy(ph).cuda(), torch.from_numpy(ih).cuda(),
                             torch.from_numpy(th).cuda())
    with pytest.raises(ValueError):
        ctx.synchronize()


def test_multibounce_golden(api, ctx, golden):
    codec = api.Codec(ctx, golden["E6"], golden["D6"])
    t = {k: torch.from_numpy(np.ascontiguousarray(golden[k])).cuda()
         for k in ("c4_palcodes", "c4_illcodes", "c4_pidx", "c4_iidx", "c4_tw")}
    out = codec.multibounce_latent(t["c4_palcodes"], t["c4_illcodes"], t["c4_pidx"], t["c4_iidx"], t["c4_tw"],
                                   latent=True)
    _check("golden c4 latent", host(out["latent"]), golden["c4_latent"])
    _check("golden c4 xyz", host(out["xyz"]), golden["c4_xyz"])
    _check("golden c4 rgb", host(out["rgb"]), golden["c4_rgb"])
    nv = codec.multibounce_spectral(torch.from_numpy(golden["palette"]).cuda(),
                                    torch.from_numpy(golden["c4_ill"]).cuda(), t["c4_pidx"], t["c4_iidx"], t["c4_tw"])
    _check("golden c4 naive xyz", host(nv["xyz"]), golden["c4_naive_xyz"])
    _check("golden c4 naive rgb", host(nv["rgb"]), golden["c4_naive_rgb"])


# ----------------------------------------------------------------- loss (config 5b)
@pytest.mark.parametrize("pairs,k,n", [(29, 6, 81), (100_003, 6, 81), (70_001, 9, 81), (5000, 3, 81),
                                       (64 * 296 * 3, 6, 47), (1001, 9, 47)])
def test_hadamard_loss_vs_oracle(api, ctx, orc, pairs, k, n):
    codec, E, D = _codec(api, ctx, k, n)
    A = api.synth_gm_spectra(ctx, SEED, "loss.a", 0, pairs, n)
    B = api.synth_gm_spectra(ctx, SEED, "loss.b", 0, pairs, n)
    got = float(host(codec.hadamard_loss(A, B))[0])
    want = orc.orc_hadamard_loss(E, D, k, n, host(A), host(B), pairs)
    print(f"loss pairs={pairs}: got={got!r} want={want!r} rel={abs(got - want) / abs(want):.2e}")
    assert got == pytest.approx(want, rel=TOL)


def test_hadamard_loss_golden(api, ctx, golden):
    codec = api.Codec(ctx, golden["E6"], golden["D6"])
    got = float(host(codec.hadamard_loss(torch.from_numpy(golden["c5b_A"]).cuda(),
                                         torch.from_numpy(golden["c5b_B"]).cuda()))[0])
    assert got == pytest.approx(float(golden["c5b_loss"][0]), rel=TOL)


# ----------------------------------------------------------------- MLP (config 5a)
@pytest.mark.parametrize("k,P", [(6, 40), (6, 128 * 148 + 77), (6, 128 * 148 * 4 * 3 + 5), (9, 128 * 600),
                                 (3, 1), (9, 1000)])
def test_mlp_vs_oracle(api, ctx, orc, k, P):
    """Multiple tiles per stream, ragged tails (generic path), k in {3, 6, 9}."""
    w = synth.mlp_weights(SEED, k, 64)
    mlp = api.CodeMLP(ctx, w)
    rgb = api.synth_uniform(ctx, SEED, "mlp.input", 0, P * 3).reshape(P, 3)
    got = host(mlp.forward(rgb))
    ref = np.zeros((P, k), np.float32)
    orc.orc_mlp_forward(host(rgb), P, 64, k, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"], w["b3"], ref)
    _check(f"mlp k={k} P={P}", got, ref, MLP_TOL)
    assert np.all(got >= 0)


def test_mlp_unaligned_input_and_repeat(api, ctx, orc):
    """rgb base not 16-byte aligned (no bulk copies), and two calls give identical codes."""
    w = synth.mlp_weights(SEED, 6, 64)
    mlp = api.CodeMLP(ctx, w)
    P = 128 * 300 + 3
    buf = api.synth_uniform(ctx, SEED, "mlp.input", 0, P * 3 + 1)
    rgb = buf[1:].reshape(P, 3)
    assert rgb.data_ptr() % 16 != 0
    got = host(mlp.forward(rgb))
    ref = np.zeros((P, 6), np.float32)
    orc.orc_mlp_forward(host(rgb), P, 64, 6, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"], w["b3"], ref)
    _check("mlp unaligned", got, ref, MLP_TOL)
    rgb2 = torch.empty(P, 3, device="cuda")
    rgb2.copy_(rgb)
    a, b = host(mlp.forward(rgb2)), host(mlp.forward(rgb2))
    assert np.array_equal(a, b)
    assert np.array_equal(a, got)


def test_mlp_golden(api, ctx, golden):
    w = {k: golden[f"c5_{k}"] for k in ("w1", "b1", "w2", "b2", "w3", "b3")}
    mlp = api.CodeMLP(ctx, w)
    got = host(mlp.forward(torch.from_numpy(np.ascontiguousarray(golden["c5_rgb"])).cuda()))
    _check("golden mlp", got, golden["c5_codes"], MLP_TOL)
