"""CPU: pin the oracle (plain-C restatement, oracle/hc_oracle.c) and the host
generators against the reference's frozen known-answer tests and against
outputs of the compiled reference (golden fixtures; oracle/_ref when built)."""
import json
import math

import numpy as np
import pytest

import oracle
from conftest import GOLD
from paper_2602_18741_b200 import synth
from paper_2602_18741_b200.colorimetry import cmf_matrix, cmf_table, grid
from paper_2602_18741_b200.rng import Rng, ctr_u64, stream_key


# ----------------------------------------------------------------- reference KATs
def test_softplus_kats(orc, kats):
    kt = kats["softplus"]
    for raw, want, rel in kt["cases"]:
        assert orc.orc_softplus(raw, kt["beta"]) == pytest.approx(want, rel=rel)
    for raw in kt["identity_exact"]:
        assert orc.orc_softplus(raw, kt["beta"]) == raw


def test_grid47_kat(kats):
    lo, step = grid(47)
    g = kats["grid47"]
    assert step == pytest.approx(g["step"], rel=1e-15)
    assert lo + step * 4 == pytest.approx(g["wl4"], rel=1e-12)
    assert lo + step * 33 == pytest.approx(g["wl33"], rel=1e-12)
    assert lo + step * 23 == g["wl23"]


def test_cmf_data_matches_reference_anchors(kats):
    t = cmf_table(47)
    a = kats["cmf_anchors47"]
    for i, x, y, z, d in a["rows"]:
        for got, want in ((t["xbar"][i], x), (t["ybar"][i], y), (t["zbar"][i], z), (t["d65"][i], d)):
            assert got == pytest.approx(want, rel=a["rel"], abs=0.0 if want else 0.0)


def test_white_point_from_shipped_rows(kats):
    t = cmf_table(47)
    norm = float(np.sum(t["ybar"] * t["d65"]))
    scale = 100.0 / norm
    white = [float(np.sum(scale * t[r] * t["d65"])) for r in ("xbar", "ybar", "zbar")]
    for got, want in zip(white, kats["white47"]["xyz"]):
        assert got == pytest.approx(want, rel=1e-12)


def test_radiance_xyz_kats(orc, kats):
    lo, step = grid(47)
    cmf = cmf_matrix(47)
    out = np.zeros(3)
    orc.orc_spectrum_to_xyz_d(cmf, step, 47, np.ones(47), out)
    np.testing.assert_allclose(out, kats["radiance_xyz47"]["ones"], rtol=1e-12)
    g = np.array(synth.gaussian_curve(550.0, 30.0, 1.0, 47))
    orc.orc_spectrum_to_xyz_d(cmf, step, 47, g, out)
    np.testing.assert_allclose(out, kats["radiance_xyz47"]["gauss_550_30_1"], rtol=1e-12)
    # the re-gridded n = 81 probe of SURVEY §8c
    orc.orc_spectrum_to_xyz_d(cmf_matrix(81), grid(81)[1], 81, np.ones(81), out)
    np.testing.assert_allclose(out, kats["survey_n81_probe"]["ones"], rtol=kats["survey_n81_probe"]["rel"])


def test_srgb_white_kat(orc, kats):
    # xyz_to_linear_rgb(srgb_reference_white) ~ (1, 1, 1) (test_colorimetry.cpp:157-165)
    from paper_2602_18741_b200.colorimetry import XYZ_TO_LINEAR_RGB

    rgb = XYZ_TO_LINEAR_RGB @ np.array(kats["srgb_white"]["white"])
    np.testing.assert_allclose(rgb, 1.0, atol=kats["srgb_white"]["tol"])


# ----------------------------------------------------------------- RNG port vs the reference
def test_rng_port_matches_reference_streams(kats):
    g = json.loads((GOLD / "ref_rng.json").read_text())
    for case in g["stream"]:
        r = Rng.stream(case["seed"], case["purpose"])
        assert [r.next_u64() for _ in range(8)] == case["u64"]
    for case in g["seed"]:
        r = Rng(case["seed"])
        assert [r.next_u64() for _ in range(8)] == case["u64"]
    for case in g["pixel_stream"]:
        r = Rng.pixel_stream(*case["args"])
        assert [r.next_u64() for _ in range(4)] == case["u64"]
    assert g["fnv1a64_hello"] == int(kats["fnv1a64_hello"]["value"], 16)


def test_counter_stream_is_splitmix_of_index():
    key = stream_key(9, "gbuffer.cos")
    v = ctr_u64(key, np.arange(5, dtype=np.uint64))
    for i in range(5):
        st = (key + i * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        r = Rng.__new__(Rng)
        from paper_2602_18741_b200.rng import splitmix64_next

        assert int(v[i]) == splitmix64_next(st)[0]
        del r


# ----------------------------------------------------------------- generators vs the reference
def test_gaussian_and_blackbody_match_reference_bit_exact():
    g = json.loads((GOLD / "ref_generators.json").read_text())
    for case in g["gaussian"]:
        assert synth.gaussian_curve(*case["args"], case["n"]) == case["values"]
    for case in g["blackbody"]:
        assert synth.blackbody_curve(case["kelvin"], case["n"]) == case["values"]


def test_glorot_init_matches_reference():
    g = json.loads((GOLD / "ref_generators.json").read_text())["glorot"][0]
    w = synth.mlp_weights(g["seed"], g["k"], g["hidden"])
    assert list(w["w1_f64"].ravel()[:16]) == g["w1_head"]
    assert list(w["w2_f64"].ravel()[:16]) == g["w2_head"]
    assert list(w["w3_f64"].ravel()[:16]) == g["w3_head"]
    assert float(w["w2_f64"].sum()) == pytest.approx(g["w2_sum"], rel=1e-12)


def test_bf16_round_matches_oracle(orc):
    x = np.random.default_rng(0).standard_normal(1000).astype(np.float32)
    ours = synth.bf16_round(x)
    theirs = np.array([orc.orc_bf16_round(float(v)) for v in x], dtype=np.float32)
    assert np.array_equal(ours, theirs)
    assert np.all(ours.view(np.uint32) & 0xFFFF == 0)


# ----------------------------------------------------------------- oracle vs golden (reference outputs)
def _cmf81():
    return cmf_matrix(81), grid(81)[1]


def test_oracle_roundtrip_bit_exact_vs_reference_golden(orc, golden):
    cmf, dl = _cmf81()
    S = golden["c1_S"]
    rows = S.shape[0]
    Z, S2, X, R = (np.zeros((rows, d), np.float32) for d in (6, 81, 3, 3))
    orc.orc_codec_roundtrip(golden["E6"], golden["D6"], 6, 81, cmf, dl, S, rows, Z, S2, X, R)
    for got, key in ((Z, "c1_Z"), (S2, "c1_S2"), (X, "c1_xyz"), (R, "c1_rgb")):
        assert np.array_equal(got, golden[key]), key


@pytest.mark.parametrize("tag,k,L", [("c2", 6, 8), ("c3", 9, 32)])
def test_oracle_shading_bit_exact_vs_reference_golden(orc, golden, tag, k, L):
    cmf, dl = _cmf81()
    idx, cosv = golden[f"{tag}_idx"], np.ascontiguousarray(golden[f"{tag}_cos"])
    P = idx.shape[0]
    pc = np.zeros((256, k), np.float32)
    lc = np.zeros((L, k), np.float32)
    orc.orc_asset_codes(golden[f"E{k}"], k, 81, golden["palette"], 256, pc)
    orc.orc_asset_codes(golden[f"E{k}"], k, 81, golden[f"{tag}_lights"], L, lc)
    assert np.array_equal(pc, golden[f"{tag}_palcodes"]) and np.array_equal(lc, golden[f"{tag}_lightcodes"])
    lat, S2, X, R = (np.zeros((P, d), np.float32) for d in (k, 81, 3, 3))
    orc.orc_shade_latent(golden[f"D{k}"], k, 81, cmf, dl, pc, lc, L, idx, cosv, P, lat, S2, X, R)
    for got, key in ((lat, "latent"), (S2, "S2"), (X, "xyz"), (R, "rgb")):
        assert np.array_equal(got, golden[f"{tag}_{key}"]), key
    SS, SX, SR = (np.zeros((P, d), np.float32) for d in (81, 3, 3))
    orc.orc_shade_spectral(81, cmf, dl, golden["palette"], golden[f"{tag}_lights"], L, idx, cosv, P, SS, SX, SR)
    for got, key in ((SS, "naive_S"), (SX, "naive_xyz"), (SR, "naive_rgb")):
        assert np.array_equal(got, golden[f"{tag}_{key}"]), key


def test_oracle_chain_bit_exact_vs_reference_golden(orc, golden):
    cmf, dl = _cmf81()
    pidx, iidx, tw = (np.ascontiguousarray(golden[k]) for k in ("c4_pidx", "c4_iidx", "c4_tw"))
    P, spp = iidx.shape
    lat = np.zeros((P, 6), np.float32)
    orc.orc_chain(6, golden["c4_palcodes"], golden["c4_illcodes"], pidx, iidx, tw, P, spp, 4, lat)
    assert np.array_equal(lat, golden["c4_latent"])
    S2 = np.zeros((P, 81), np.float32)
    X, R = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
    orc.orc_decode(golden["D6"], 6, 81, lat, P, S2)
    orc.orc_spectra_to_outputs(cmf, dl, 81, S2, P, X, R)
    assert np.array_equal(X, golden["c4_xyz"]) and np.array_equal(R, golden["c4_rgb"])
    spec = np.zeros((P, 81), np.float32)
    orc.orc_chain(81, golden["palette"], golden["c4_ill"], pidx, iidx, tw, P, spp, 4, spec)
    orc.orc_spectra_to_outputs(cmf, dl, 81, spec, P, X, R)
    assert np.array_equal(X, golden["c4_naive_xyz"]) and np.array_equal(R, golden["c4_naive_rgb"])


def test_oracle_mlp_and_loss_vs_reference_golden(orc, golden):
    rgb = np.ascontiguousarray(golden["c5_rgb"])
    P = rgb.shape[0]
    out = np.zeros((P, 6), np.float32)
    w = {k: np.ascontiguousarray(golden[f"c5_{k}"]) for k in ("w1", "b1", "w2", "b2", "w3", "b3")}
    orc.orc_mlp_forward(rgb, P, 64, 6, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"], w["b3"], out)
    assert np.array_equal(out, golden["c5_codes"])
    A, B = golden["c5b_A"], golden["c5b_B"]
    loss = orc.orc_hadamard_loss(golden["E6"], golden["D6"], 6, 81, A, B, A.shape[0])
    assert loss == golden["c5b_loss"][0]


# ----------------------------------------------------------------- live cross-check (build container only)
def test_oracle_matches_compiled_reference_random(orc, ref81):
    """Fresh seeds, all configs, bit-for-bit against oracle/_ref (needs the compiled reference)."""
    cmf, dl = _cmf81()
    seed = 77
    E, D = synth.codec_weights(seed, 6, 81)
    S = synth.gm_spectra_ctr(seed, "codec.spectra", 1000, 23, 81)
    a = [np.zeros((23, d), np.float32) for d in (6, 81, 3, 3)]
    b = [np.zeros((23, d), np.float32) for d in (6, 81, 3, 3)]
    orc.orc_codec_roundtrip(E, D, 6, 81, cmf, dl, S, 23, *a)
    ref81.ref_codec_roundtrip(E, D, 6, S, 23, *b, 1)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    loss_o = orc.orc_hadamard_loss(E, D, 6, 81, S, S[::-1].copy(), 23)
    loss_r = ref81.ref_hadamard_loss(E, D, 6, S, S[::-1].copy(), 23, 1)
    assert loss_o == loss_r
    # n = 47 grid: the unmodified reference
    ref47 = oracle.reference(47)
    E47, D47 = synth.codec_weights(seed, 9, 47)
    S47 = synth.gm_spectra_ctr(seed, "codec.spectra", 0, 11, 47)
    c = [np.zeros((11, d), np.float32) for d in (9, 47, 3, 3)]
    d_ = [np.zeros((11, d), np.float32) for d in (9, 47, 3, 3)]
    orc.orc_codec_roundtrip(E47, D47, 9, 47, cmf_matrix(47), grid(47)[1], S47, 11, *c)
    ref47.ref_codec_roundtrip(E47, D47, 9, S47, 11, *d_, 1)
    for x, y in zip(c, d_):
        assert np.array_equal(x, y)


def test_decode_rejects_negative_in_reference(ref81):
    """decode's contract (codec.cpp:56-62) that the GPU path latches as HC_EDOMAIN."""
    D = np.full((81, 6), 0.1, np.float32)
    Z = np.array([[0.1, 0.2, 0.3, 0.4, 0.5, 0.6]])
    S = np.zeros((1, 81))
    assert ref81.ref_decode_rows_d(D, 6, Z, 1, S) == 0
    Z[0, 2] = -1e-9
    assert ref81.ref_decode_rows_d(D, 6, Z, 1, S) == 1


# ----------------------------------------------------------------- colour-metric tail
def test_colour_difference_kats(orc, kats):
    c = kats["colour_differences"]
    a, b = np.array(c["a"]), np.array(c["b"])
    assert orc.orc_delta_e76(a, b) == pytest.approx(c["de76_ab"], rel=c["eps"])
    assert orc.orc_delta_e94(a, b) == pytest.approx(c["de94_ab"], rel=c["eps"])
    assert orc.orc_delta_e94(b, a) == pytest.approx(c["de94_ba"], rel=c["eps"])
    assert orc.orc_delta_e76(a, a) == 0.0 and orc.orc_delta_e94(a, a) == 0.0
    assert orc.orc_delta_e94(np.array(c["c"]), np.array(c["d"])) == pytest.approx(c["de94_cd"], rel=c["eps"])


def test_lab_and_srgb_encode_kats(orc, kats):
    k = kats["lab_near_black"]
    lab = np.zeros(3)
    orc.orc_xyz_to_lab(np.array(k["xyz"]), np.array(k["white"]), lab)
    for got, want, eps in zip(lab, k["lab"], k["eps"]):
        assert got == pytest.approx(want, rel=eps)
    t = cmf_table(47)
    norm = float(np.sum(t["ybar"] * t["d65"]))
    white = np.array([float(np.sum(100.0 / norm * t[r] * t["d65"])) for r in ("xbar", "ybar", "zbar")])
    orc.orc_xyz_to_lab(white, white, lab)
    assert lab[0] == pytest.approx(kats["lab_white47"]["L"], rel=kats["lab_white47"]["eps"])
    assert abs(lab[1]) < kats["lab_white47"]["ab_abs"] and abs(lab[2]) < kats["lab_white47"]["ab_abs"]
    for x, want, eps in kats["srgb_encode"]["cases"]:
        assert orc.orc_srgb_encode(x) == pytest.approx(want, rel=eps, abs=0.0)


def _metric_images(seed, P, n):
    """Linear-RGB-like and spectral images with negatives, zeros and a wide dynamic range."""
    rng = np.random.default_rng(seed)
    rgb_a = (rng.lognormal(-1.0, 1.5, (P, 3)) * (rng.random((P, 3)) > 0.02)).astype(np.float32)
    rgb_a[:7] = [[0, 0, 0], [1e-9, 0, 0], [-0.01, 0.02, 0.0], [5, 5, 5], [0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [2, 0, 1]]
    rgb_b = (rgb_a * rng.normal(1.0, 0.05, (P, 3))).astype(np.float32)
    spec = rng.random((P, n)).astype(np.float32) * rng.lognormal(0.0, 1.0, (P, 1)).astype(np.float32)
    spec2 = (spec * rng.normal(1.0, 0.03, (P, n))).astype(np.float32)
    return rgb_a, rgb_b, spec, spec2


@pytest.mark.parametrize("n", [47, 81])
def test_metric_tail_oracle_matches_compiled_reference(orc, n):
    """exposure_for / tonemap_srgb8 / error_map / scene_color_report / Delta E94 report:
    the C restatement against the reference's own functions (oracle/_ref)."""
    ref = oracle.reference(n)
    if ref is None:
        pytest.skip("compiled reference not built")
    P = 3001
    cmf, dl = cmf_matrix(n), grid(n)[1]
    a, b, s, s2 = _metric_images(5 + n, P, n)
    for img, ch in ((a, 3), (s, n)):
        for pct in (99.5, 50.0, 0.0, 100.0):
            got = orc.orc_exposure_for(img, P, ch, None if ch == 3 else np.ascontiguousarray(cmf[1]), dl, pct)
            assert got == ref.ref_exposure_for(img, P, ch, pct)
    e = ref.ref_exposure_for(a, P, 3, 99.5)
    u1, u2 = np.zeros(P * 3, np.uint8), np.zeros(P * 3, np.uint8)
    orc.orc_tonemap_srgb8(a, P, e, u1)
    ref.ref_tonemap_srgb8(a, P, e, u2)
    assert np.array_equal(u1, u2)
    for x, cx, y, cy in ((a, 3, b, 3), (s, n, s2, n), (s, n, b, 3)):
        m1, m2 = np.zeros(P, np.float32), np.zeros(P, np.float32)
        assert orc.orc_error_map(x, cx, y, cy, P, cmf, dl, m1) == ref.ref_error_map(x, cx, y, cy, P, m2)
        assert np.array_equal(m1, m2)
        r1, r2 = np.zeros(4), np.zeros(4)
        orc.orc_scene_color_report(x, cx, y, cy, P, cmf, dl, r1)
        ref.ref_scene_color_report(x, cx, y, cy, P, r2)
        assert np.array_equal(r1, r2), (r1, r2)
    white = np.zeros(3)
    ref.ref_white_xyz(white)
    xg = (a * 40).astype(np.float32)
    xt = (b * 40).astype(np.float32)
    d1, d2 = np.zeros(P, np.float32), np.zeros(P, np.float32)
    o1, o2 = np.zeros(3), np.zeros(3)
    orc.orc_delta_e94_report(xg, xt, P, white, d1, o1)
    ref.ref_delta_e94_report(xg, xt, P, d2, o2)
    assert np.array_equal(d1, d2) and np.array_equal(o1, o2)


def test_analytic_cmf_fit_tracks_the_tabulated_cie1931():
    """The analytic multi-lobe fit BASELINE config 1 names stays within 1.5 % of the peak of the
    tabulated CIE 1931 functions the reference uses (CmfTable), on both grids."""
    from paper_2602_18741_b200.colorimetry import cmf_analytic, cmf_matrix

    for n in (81, 47):
        fit, tab = cmf_analytic(n), cmf_matrix(n)
        for r in range(3):
            assert np.max(np.abs(fit[r] - tab[r])) <= 0.015 * tab[r].max()
        # and it is a different function (not the table under another name)
        assert np.max(np.abs(fit - tab)) > 1e-3
