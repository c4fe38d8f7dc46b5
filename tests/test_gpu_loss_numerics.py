"""Near-multiplicativity loss (config 5b) in the regime the loss is
for: codecs that are close to multiplicative on their inputs.

The reference forms the residual r_l = (D (E a (.) E b))_l - a_l b_l per wavelength and
squares it, in fp64 (forward_pair + mse_n, trainer.cpp:49-71).  When the codec is nearly
multiplicative r_l is many orders of magnitude below a_l b_l, so any formula that does not
form r_l directly at the reference's precision returns rounding noise.  These cases pin
the kernel against the oracle (orc_hadamard_loss, the same arithmetic as the reference)
where that happens:

* flat pairs with a row-normalised codec (r_l is only the fp32 quantisation of E / D);
* near-flat pairs with a band codec (residual / |a (.) b|^2 ~ 2e-5);
* the same band codec after Adam steps of the GPU training step (hc_codec_train_grad);
* per-pair values are never negative and match the oracle pair by pair.

Tolerance: 1e-5 relative on the loss (north_star's fp32 bar; the kernel is fp64).
"""
import numpy as np
import pytest

from paper_2602_18741_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5
N = 81
BETA = 10.0


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def _loss(codec, A, B):
    out = codec.hadamard_loss(torch.from_numpy(np.ascontiguousarray(A, np.float32)).cuda(),
                              torch.from_numpy(np.ascontiguousarray(B, np.float32)).cuda())
    torch.cuda.synchronize()
    return float(out.cpu().numpy()[0])


def _oracle(orc, E, D, k, A, B):
    return orc.orc_hadamard_loss(np.ascontiguousarray(E, np.float32), np.ascontiguousarray(D, np.float32), k, N,
                                 np.ascontiguousarray(A, np.float32), np.ascontiguousarray(B, np.float32), A.shape[0])


def _softplus(r):
    return np.where(BETA * r > 30.0, r, np.log1p(np.exp(np.minimum(BETA * r, 30.0))) / BETA)


def _band_raw(k, leak=-1.0):
    """Raw (softplus-parameterised) weights of a band codec: code j averages the wavelengths of
    band j and decodes to a constant over it; everything else is softplus(leak) ~ 5e-6."""
    edges = np.linspace(0, N, k + 1).round().astype(int)
    inv = lambda v: np.log(np.expm1(BETA * v)) / BETA  # noqa: E731
    re_ = np.full((k, N), leak)
    rd = np.full((N, k), leak)
    for j in range(k):
        a, b = edges[j], edges[j + 1]
        re_[j, a:b] = inv(1.0 / (b - a))
        rd[a:b, j] = inv(1.0)
    return re_, rd


def _near_flat(m, seed, amp=0.01):
    rng = np.random.default_rng(seed)
    lam = np.arange(N)
    a = rng.uniform(0.2, 0.9, (m, 1)) + amp * np.sin(lam[None, :] / 13.0 + rng.uniform(0, 6, (m, 1)))
    b = rng.uniform(0.2, 0.9, (m, 1)) + amp * np.cos(lam[None, :] / 17.0 + rng.uniform(0, 6, (m, 1)))
    return np.clip(a, 0, 1).astype(np.float32), np.clip(b, 0, 1).astype(np.float32)


def _ratio(loss, A, B):
    return loss / float(((A.astype(np.float64) * B.astype(np.float64)) ** 2).sum())


@pytest.mark.parametrize("seed", [2602, 31337])
@pytest.mark.parametrize("k", [6, 9])
def test_flat_pairs(api, ctx, orc, seed, k):
    E, D = synth.codec_weights(seed, k, N)
    codec = api.Codec(ctx, E, D)
    levels = np.array([0.3, 0.5, 0.7, 0.9, 1.0, 0.123456], np.float32)
    A = np.repeat(levels[:, None], N, axis=1)
    B = np.repeat(levels[::-1, None], N, axis=1).copy()
    want = _oracle(orc, E, D, k, A, B)
    got = _loss(codec, A, B)
    print(f"flat seed={seed} k={k}: got={got!r} want={want!r} ratio={_ratio(want, A, B):.2e}")
    assert _ratio(want, A, B) < 1e-12  # the regime: r_l is rounding-level
    assert got == pytest.approx(want, rel=TOL)


def test_flat_pairs_each_nonnegative(api, ctx, orc):
    E, D = synth.codec_weights(2602, 6, N)
    codec = api.Codec(ctx, E, D)
    for va, vb in [(0.5, 0.9), (0.3, 0.7), (1.0, 1.0), (0.0, 0.5), (1e-3, 0.25)]:
        A = np.full((1, N), va, np.float32)
        B = np.full((1, N), vb, np.float32)
        got, want = _loss(codec, A, B), _oracle(orc, E, D, 6, A, B)
        assert got >= 0.0
        assert got == pytest.approx(want, rel=TOL, abs=1e-300)


@pytest.mark.parametrize("m", [1000, 64 * 148 * 2 + 37])
def test_near_flat_band_codec(api, ctx, orc, m):
    re_, rd = _band_raw(6)
    E, D = _softplus(re_).astype(np.float32), _softplus(rd).astype(np.float32)
    codec = api.Codec(ctx, E, D)
    A, B = _near_flat(m, 5)
    want = _oracle(orc, E, D, 6, A, B)
    got = _loss(codec, A, B)
    print(f"near-flat m={m}: got={got!r} want={want!r} ratio={_ratio(want, A, B):.2e}")
    assert _ratio(want, A, B) <= 1e-3
    assert got == pytest.approx(want, rel=TOL)


def test_trained_codec(api, ctx, orc):
    """A codec after Adam steps of the GPU training step (trainer.cpp:221-411) from a band
    initialisation; residual / |a (.) b|^2 <= 1e-3 on near-flat pairs."""
    k = 6
    re_, rd = _band_raw(k)
    A, B = _near_flat(512, 11)
    params = torch.from_numpy(np.concatenate([re_.ravel(), rd.ravel()])).cuda()
    m1, v1 = torch.zeros_like(params), torch.zeros_like(params)
    refl = torch.from_numpy(A.astype(np.float64)).cuda()
    illum = torch.from_numpy(B.astype(np.float64)).cuda()
    for step in range(1, 6):
        cur = params.cpu().numpy()
        _, ge, gd = api.codec_train_grad(ctx, cur[:k * N].reshape(k, N), cur[k * N:].reshape(N, k), BETA, refl, illum)
        g = torch.from_numpy(np.concatenate([ge.ravel(), gd.ravel()])).cuda()
        api.adam_step(ctx, params, g, m1, v1, 1e-4, step)
    cur = params.cpu().numpy()
    codec = api.Codec.from_raw(ctx, cur[:k * N].reshape(k, N), cur[k * N:].reshape(N, k), beta=BETA)
    At, Bt = _near_flat(4096, 12)
    want = _oracle(orc, codec.E, codec.D, k, At, Bt)
    got = _loss(codec, At, Bt)
    print(f"trained: got={got!r} want={want!r} ratio={_ratio(want, At, Bt):.2e}")
    assert _ratio(want, At, Bt) <= 1e-3
    assert got == pytest.approx(want, rel=TOL)
