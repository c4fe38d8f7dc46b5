"""GPU: the reference's RGB -> code upsampler (upsampler.cpp:42-72, :170-190) on the device in
fp64 — against the compiled reference's upsample / upsample_raw.  Tolerance: SiLU's exp on
the device is CUDA's (<= 1 ulp from glibc's), so agreement is to 1e-13 relative; the clamp
telemetry must match exactly."""
import ctypes

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def _weights(k, hidden, seed):
    rng = np.random.default_rng(seed)
    lim = lambda fi, fo: np.sqrt(6.0 / (fi + fo))  # noqa: E731  glorot (upsampler.cpp:154-167)
    return {"w1": rng.uniform(-lim(3, hidden), lim(3, hidden), (hidden, 3)), "b1": rng.normal(0, 0.1, hidden),
            "w2": rng.uniform(-lim(hidden, hidden), lim(hidden, hidden), (hidden, hidden)),
            "b2": rng.normal(0, 0.1, hidden),
            "w3": rng.uniform(-lim(hidden, k), lim(hidden, k), (k, hidden)), "b3": rng.normal(0, 0.1, k)}


@pytest.mark.parametrize("k,hidden", [(6, 128), (3, 64), (9, 200), (6, 17), (12, 512)])
@pytest.mark.parametrize("clamp", [True, False])
def test_upsample_matches_reference(api, ctx, k, hidden, clamp):
    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    w = _weights(k, hidden, k * 1000 + hidden)
    rng = np.random.default_rng(hidden)
    P = 3000
    rgb = rng.uniform(0, 1.2, (P, 3))
    rgb[:5] = [[0, 0, 0], [1, 1, 1], [1e-9, 0.5, 2.0], [0.2, 0.9, 0.0], [1e3, 1e3, 1e3]]
    got, n = api.Upsampler(ctx, w).forward(torch.from_numpy(rgb).cuda(), clamp=clamp)
    got = got.cpu().numpy()
    want = np.zeros((P, k))
    rn = ctypes.c_uint64(0)
    arrs = [np.ascontiguousarray(w[x].reshape(-1)) for x in api.Upsampler.KEYS]
    assert ref.ref_upsample(k, hidden, *arrs, np.ascontiguousarray(rgb.reshape(-1)), P, int(clamp),
                            want.reshape(-1), ctypes.byref(rn)) == 0
    assert n == rn.value
    # a 1-ulp exp difference in any hidden unit reaches every output, so entries are close
    # rather than identical
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


def test_upsampler_rejects_invalid_weights(api, ctx):
    w = _weights(6, 32, 1)
    w["w2"][3, 4] = np.nan
    with pytest.raises(ValueError, match="finite"):
        api.Upsampler(ctx, w)


@pytest.mark.parametrize("hidden,B,lam", [(32, 64, (0.3, 0.05)), (128, 64, (0.3, 0.05)), (17, 5, (0.0, 0.0)),
                                          (64, 200, (1.0, 0.5))])
def test_upsample_loss_and_gradients_match_reference(api, ctx, hidden, B, lam):
    """upsample_loss + upsample_gradients (upsampler.cpp:207-369) against the compiled
    reference: 1e-11 relative (SiLU's exp and Lab's cbrt are CUDA's)."""
    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    k = 6
    rng = np.random.default_rng(hidden + B)
    re_ = rng.uniform(-0.5, 0.5, (k, 81)) / 9.0
    rd = rng.uniform(-0.5, 0.5, (81, k)) / np.sqrt(k)
    codec = api.Codec.from_raw(ctx, re_, rd, beta=10.0)
    w = _weights(k, hidden, hidden)
    rgb = rng.uniform(0, 1, (B, 3))
    target = np.abs(rng.normal(0.3, 0.2, (B, k)))
    losses, grads = api.upsample_train_grad(ctx, w, codec, torch.from_numpy(rgb).cuda(),
                                            torch.from_numpy(target).cuda(), *lam)
    arrs = [np.ascontiguousarray(w[x].reshape(-1)) for x in api.Upsampler.KEYS]
    rl = np.zeros(4)
    rg = np.zeros(sum(a.size for a in arrs))
    assert ref.ref_upsample_train(k, hidden, *arrs, 10.0, re_.reshape(-1).copy(), rd.reshape(-1).copy(),
                                  rgb.reshape(-1).copy(), target.reshape(-1).copy(), B, lam[0], lam[1], rl,
                                  rg.ctypes.data) == 0
    np.testing.assert_allclose(list(losses.values()), rl, rtol=1e-11)
    got = np.concatenate([grads[x].reshape(-1) for x in api.Upsampler.KEYS])
    np.testing.assert_allclose(got, rg, rtol=1e-9, atol=1e-11 * np.abs(rg).max())


def test_adamw_step_matches_reference_arithmetic(api, ctx):
    rng = np.random.default_rng(4)
    p0 = rng.normal(size=5000)
    p = torch.from_numpy(p0.copy()).cuda()
    gm, gv = torch.zeros_like(p), torch.zeros_like(p)
    m, v, pw = np.zeros_like(p0), np.zeros_like(p0), p0.copy()
    for t in range(1, 5):
        g = rng.normal(size=p0.size)
        api.adamw_step(ctx, p, torch.from_numpy(g).cuda(), gm, gv, 2e-3, 1e-5, t)
        bc1, bc2 = 1.0 - 0.9 ** t, 1.0 - 0.999 ** t
        m = 0.9 * m + (1.0 - 0.9) * g
        v = 0.999 * v + (1.0 - 0.999) * g * g
        pw -= 2e-3 * ((m / bc1) / (np.sqrt(v / bc2) + 1e-8) + 1e-5 * pw)
    assert p.cpu().numpy().tobytes() == pw.tobytes()
