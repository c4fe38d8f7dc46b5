"""GPU parity of the colour-metric tail through the C ABI against
the oracle restatement, which test_oracle.py holds bit-exact to the compiled reference's
exposure_for / tonemap_srgb8 / error_map / scene_color_report (renderer.cpp:721-802,
evaluation.cpp:122-154) and R5, the per-pixel Delta E94 of multibounce_eval
(evaluation.cpp:59-86).

Bars: exposure (an exact order statistic of bit-identical fp64 luminances), the
per-pixel MSE map, the spectral -> linear RGB conversion and the 8-bit tone map are
bit-exact; Delta E statistics go through cbrt / hypot / pow, whose CUDA and glibc
results differ by <= 2 ulp, and through a parallel fp64 sum: rel 1e-12.
"""
import numpy as np
import pytest

from paper_2602_18741_b200 import synth
from paper_2602_18741_b200.colorimetry import cmf_matrix, grid, white_xyz

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 4242
REL = 1e-12


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def _codec(api, ctx, n):
    E, D = synth.codec_weights(SEED, 6, n)
    return api.Codec(ctx, E, D)


def _images(seed, P, n):
    """Linear RGB with zeros, negatives, near-black and a wide dynamic range; spectra."""
    rng = np.random.default_rng(seed)
    a = (rng.lognormal(-1.0, 1.5, (P, 3)) * (rng.random((P, 3)) > 0.02)).astype(np.float32)
    if P >= 7:
        a[:7] = [[0, 0, 0], [1e-9, 0, 0], [-0.01, 0.02, 0.0], [5, 5, 5], [0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [2, 0, 1]]
    b = (a * rng.normal(1.0, 0.05, (P, 3))).astype(np.float32)
    s = (rng.random((P, n)) * rng.lognormal(0.0, 1.0, (P, 1))).astype(np.float32)
    s2 = (s * rng.normal(1.0, 0.03, (P, n))).astype(np.float32)
    return a, b, s, s2


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("n,P", [(81, 1), (81, 7), (81, 3001), (47, 20_011), (81, 300_007)])
def test_exposure_for_exact(api, ctx, orc, n, P):
    codec = _codec(api, ctx, n)
    a, _, s, _ = _images(SEED + P, P, n)
    ybar = np.ascontiguousarray(cmf_matrix(n)[1])
    for img, ch in ((a, 3), (s, n)):
        for pct in (99.5, 50.0, 0.0, 100.0, 37.3, 150.0):
            got = api.exposure_for(codec, dev(img), pct)
            want = orc.orc_exposure_for(img, P, ch, None if ch == 3 else ybar, grid(n)[1], pct)
            assert got == want, (ch, pct, got, want)


def test_exposure_ties_and_constant_image(api, ctx, orc):
    codec = _codec(api, ctx, 81)
    P = 10_000
    flat = np.full((P, 3), 0.25, np.float32)
    assert api.exposure_for(codec, dev(flat)) == orc.orc_exposure_for(flat, P, 3, None, 5.0, 99.5)
    dark = np.zeros((P, 3), np.float32)
    assert api.exposure_for(codec, dev(dark)) == 1.0  # ref <= 1e-12 -> 1
    neg = -np.abs(_images(1, P, 81)[0])
    assert api.exposure_for(codec, dev(neg), 99.5) == orc.orc_exposure_for(neg, P, 3, None, 5.0, 99.5)


@pytest.mark.parametrize("P", [1, 1000, 250_001])
def test_tonemap_srgb8_exact(api, ctx, orc, P):
    a = _images(SEED, P, 81)[0]
    for e in (1.0, 0.37, 4.0):
        got = api.tonemap_srgb8(ctx, dev(a), e).cpu().numpy().reshape(-1)
        want = np.zeros(P * 3, np.uint8)
        orc.orc_tonemap_srgb8(a, P, e, want)
        assert np.array_equal(got, want), int(np.sum(got != want))


@pytest.mark.parametrize("n,P", [(81, 5003), (47, 777), (81, 200_001)])
def test_error_map(api, ctx, orc, n, P):
    codec = _codec(api, ctx, n)
    a, b, s, s2 = _images(SEED + 1, P, n)
    cmf, dl = cmf_matrix(n), grid(n)[1]
    for x, cx, y, cy in ((a, 3, b, 3), (s, n, s2, n), (s, n, b, 3)):
        mse, mean = api.error_map(codec, dev(x), dev(y))
        want = np.zeros(P, np.float32)
        wmean = orc.orc_error_map(x, cx, y, cy, P, cmf, dl, want)
        assert np.array_equal(mse.cpu().numpy(), want)
        assert mean == pytest.approx(wmean, rel=REL)


@pytest.mark.parametrize("n,P", [(81, 4099), (47, 1001), (81, 300_007)])
def test_scene_color_report(api, ctx, orc, n, P):
    codec = _codec(api, ctx, n)
    a, b, s, s2 = _images(SEED + 2, P, n)
    cmf, dl = cmf_matrix(n), grid(n)[1]
    for x, cx, y, cy in ((a, 3, b, 3), (s, n, s2, n), (s, n, b, 3)):
        got = api.scene_color_report(codec, dev(x), dev(y))
        want = np.zeros(4)
        orc.orc_scene_color_report(x, cx, y, cy, P, cmf, dl, want)
        assert got["exposure"] == want[3]
        assert got["mse"] == pytest.approx(want[2], rel=REL)
        assert got["mean_de76"] == pytest.approx(want[0], rel=REL)
        assert got["p95_de76"] == pytest.approx(want[1], rel=REL)


@pytest.mark.parametrize("n,P", [(81, 1), (81, 3001), (47, 50_000)])
def test_delta_e94_report(api, ctx, orc, n, P):
    a, b, _, _ = _images(SEED + 3, P, n)
    xg, xt = (a * 40).astype(np.float32), (b * 40).astype(np.float32)
    got = api.delta_e94_report(ctx, dev(xg), dev(xt), n=n, per_pixel=True)
    de = np.zeros(P, np.float32)
    want = np.zeros(3)
    orc.orc_delta_e94_report(xg, xt, P, np.array(white_xyz(n)), de, want)
    g = got["de94"].cpu().numpy()
    assert np.max(np.abs(g - de) / np.maximum(np.abs(de), 1e-30)) <= 1.2e-7
    for key, w in zip(("mean_de94", "median_de94", "p95_de94"), want):
        assert got[key] == pytest.approx(w, rel=REL)


def test_metrics_on_latent_vs_naive_frame(api, ctx, orc):
    """The paper's quality comparison on a shaded frame: naive n = 81 render as ground truth,
    the latent (k = 6) render as test, both through the library's own shading kernels."""
    n, k, L, P = 81, 6, 8, 64 * 1920
    E, D = synth.codec_weights(SEED, k, n)
    codec = api.Codec(ctx, E, D)
    pal, lts = synth.palette(SEED, 256, n), synth.lights(SEED, L, n)
    pal_d = dev(pal)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, P, L, 256)
    lat = codec.shade_latent(codec.encode(pal_d), codec.encode(dev(lts)).cpu().numpy(), idx, cosv, spectra=True)
    nv = codec.shade_spectral(pal_d, lts, idx, cosv, spectra=True)
    got = api.scene_color_report(codec, nv["spectra"], lat["spectra"])
    want = np.zeros(4)
    orc.orc_scene_color_report(nv["spectra"].cpu().numpy(), n, lat["spectra"].cpu().numpy(), n, P, cmf_matrix(n),
                               grid(n)[1], want)
    assert got["exposure"] == want[3]
    for key, w in zip(("mean_de76", "p95_de76", "mse"), want[:3]):
        assert got[key] == pytest.approx(w, rel=REL)
    r94 = api.delta_e94_report(ctx, nv["xyz"], lat["xyz"], n=n)
    want94 = np.zeros(3)
    orc.orc_delta_e94_report(nv["xyz"].cpu().numpy(), lat["xyz"].cpu().numpy(), P, np.array(white_xyz(n)), None,
                             want94)
    assert r94["mean_de94"] == pytest.approx(want94[0], rel=REL)
    assert r94["p95_de94"] == pytest.approx(want94[2], rel=REL)


def test_metric_argument_errors(api, ctx):
    codec = _codec(api, ctx, 81)
    with pytest.raises(ValueError):
        api.exposure_for(codec, torch.zeros(10, 5, device="cuda"))
    with pytest.raises(ValueError):
        api.error_map(codec, torch.zeros(10, 3, device="cuda"), torch.zeros(11, 3, device="cuda"))
    with pytest.raises(ArithmeticError):
        api.delta_e94_report(ctx, torch.ones(4, 3, device="cuda"), torch.ones(4, 3, device="cuda"),
                             white=(1.0, 0.0, 1.0))


def test_scene_report_dev_and_preview(api, ctx, orc):
    """The stream-ordered form gives the same four numbers and the tone-mapped preview
    tonemap_srgb8(test, exposure_for(gt)) bit-exactly."""
    codec = _codec(api, ctx, 81)
    P = 100_003
    a, b, _, _ = _images(SEED + 9, P, 81)
    sync = api.scene_color_report(codec, dev(a), dev(b))
    prev = torch.empty(P, 3, dtype=torch.uint8, device="cuda")
    out = api.scene_color_report_dev(codec, dev(a), dev(b), preview=prev).cpu().numpy()
    assert list(out) == [sync["mean_de76"], sync["p95_de76"], sync["mse"], sync["exposure"]]
    want = np.zeros(P * 3, np.uint8)
    orc.orc_tonemap_srgb8(b, P, sync["exposure"], want)
    assert np.array_equal(prev.cpu().numpy().reshape(-1), want)


@pytest.mark.parametrize("n,rows,refl", [(81, 1, False), (81, 1000, False), (47, 777, False), (81, 513, True),
                                         (47, 64, True)])
def test_spectra_to_xyz_f64_matches_reference_order(api, ctx, n, rows, refl):
    """hc_spectra_to_xyz_f64 (the drop-in's by-value spectrum_to_xyz / xyz_of_reflectance):
    fp64 sums in the reference's order (colorimetry.cpp:75-101), so bit-identical to a sequential
    numpy-scalar restatement; radiance rows are the CMF rows then x dlambda, reflectance rows the
    D65-weighted rows scale * cmf * d65 (scale = 100 / sum(ybar d65))."""
    from paper_2602_18741_b200 import _lib
    from paper_2602_18741_b200.colorimetry import cmf_table

    codec = _codec(api, ctx, n)
    rng = np.random.default_rng(rows + n)
    S = rng.random((rows, n)) * rng.lognormal(0.0, 1.0, (rows, 1))
    t = cmf_table(n)
    cmf = [t["xbar"], t["ybar"], t["zbar"]]
    if refl:
        norm = 0.0
        for i in range(n):
            norm += t["ybar"][i] * t["d65"][i]
        scale = 100.0 / norm
        w = np.array([[scale * row[i] * t["d65"][i] for i in range(n)] for row in cmf])
        rows_used, mult = w, None
    else:
        w, rows_used, mult = None, np.array(cmf), grid(n)[1]
    out = torch.empty(rows, 3, dtype=torch.float64, device="cuda")
    Sd = dev(S)
    wp = None if w is None else np.ascontiguousarray(w, np.float64).ctypes.data
    rc = _lib.lib().hc_spectra_to_xyz_f64(codec.h, Sd.data_ptr(), rows, wp, out.data_ptr())
    assert rc == 0
    ctx.synchronize()
    got = out.cpu().numpy()
    for r in range(0, rows, max(1, rows // 50)):
        want = []
        for c in range(3):
            acc = 0.0
            for i in range(n):
                acc += float(rows_used[c][i]) * float(S[r, i])
            want.append(acc * mult if mult is not None else acc)
        assert list(got[r]) == want, (r, got[r], want)
