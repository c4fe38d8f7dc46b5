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
