"""GPU: the codec training step — compute_losses + gradients
(trainer.cpp:108-373) and adam_step (:399-411) — bit-identical to the compiled reference."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N = 81


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


@pytest.fixture(scope="module")
def ref():
    r = oracle.reference(N)
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    return r


def _case(k, m, seed):
    rng = np.random.default_rng(seed)
    re_ = rng.uniform(-0.5, 0.5, (k, N)) / np.sqrt(N)      # init_codec_weights scales (trainer.cpp:375-390)
    rd = rng.uniform(-0.5, 0.5, (N, k)) / np.sqrt(k)
    re_[0, :3] = [4.0, -3.5, 0.0]                          # both softplus branches (beta * raw > 30)
    refl = rng.uniform(0, 1, (m, N))
    illum = rng.uniform(0, 1, (m, N)) * rng.uniform(0.5, 2.0, (m, 1))
    if m > 2:
        refl[1] = 0.0                                      # a zero product: cosine's a == 0 branch
    return re_, rd, refl, illum


LWS = [(0.5, 0.75, 1.0, 0.5, 0.0), (1.0, 1.0, 1.0, 1.0, 0.3), (0.0, 1.0, 0.0, 0.0, 0.0), (0.7, 0.0, 0.0, 2.0, 1e-3)]


@pytest.mark.parametrize("k", [3, 6, 9])
@pytest.mark.parametrize("m", [1, 128, 1000])
@pytest.mark.parametrize("lw", range(len(LWS)))
def test_losses_and_gradients_bit_identical(api, ctx, ref, k, m, lw):
    re_, rd, refl, illum = _case(k, m, 100 * k + m + lw)
    beta = 10.0
    losses, ge, gd = api.codec_train_grad(ctx, re_, rd, beta, torch.from_numpy(refl).cuda(),
                                          torch.from_numpy(illum).cuda(), loss_weights=LWS[lw])
    rge, rgd, rl = np.zeros(k * N), np.zeros(N * k), np.zeros(6)
    assert ref.ref_codec_gradients(k, beta, re_.reshape(-1), rd.reshape(-1), np.ascontiguousarray(refl.reshape(-1)),
                                   np.ascontiguousarray(illum.reshape(-1)), m, np.array(LWS[lw]),
                                   rge.ctypes.data, rgd.ctypes.data, rl) == 0
    assert ge.reshape(-1).tobytes() == rge.tobytes()
    assert gd.reshape(-1).tobytes() == rgd.tobytes()
    assert np.array(list(losses.values())).tobytes() == rl.tobytes()


def test_adam_step_bit_identical(api, ctx):
    rng = np.random.default_rng(3)
    p0 = rng.normal(size=10_000)
    st_m, st_v = np.zeros_like(p0), np.zeros_like(p0)
    p = torch.from_numpy(p0.copy()).cuda()
    gm, gv = torch.zeros_like(p), torch.zeros_like(p)
    pw = p0.copy()
    for step in range(1, 6):
        g = rng.normal(size=p0.size) * 10.0 ** rng.integers(-6, 2, p0.size)
        api.adam_step(ctx, p, torch.from_numpy(g).cuda(), gm, gv, 1e-3, step)
        # the reference's arithmetic, in numpy fp64 (trainer.cpp:399-411)
        c1 = 1.0 - 0.9 ** step
        c2 = 1.0 - 0.999 ** step
        st_m = 0.9 * st_m + (1.0 - 0.9) * g
        st_v = 0.999 * st_v + (1.0 - 0.999) * g * g
        pw -= 1e-3 * (st_m / c1) / (np.sqrt(st_v / c2) + 1e-8)
    assert p.cpu().numpy().tobytes() == pw.tobytes()
    assert gm.cpu().numpy().tobytes() == st_m.tobytes() and gv.cpu().numpy().tobytes() == st_v.tobytes()


def test_losses_only_matches_full_call(api, ctx):
    re_, rd, refl, illum = _case(6, 300, 5)
    r, l = torch.from_numpy(refl).cuda(), torch.from_numpy(illum).cuda()
    full, _, _ = api.codec_train_grad(ctx, re_, rd, 10.0, r, l)
    only, ge, gd = api.codec_train_grad(ctx, re_, rd, 10.0, r, l, grads=False)
    assert ge is None and gd is None and only == full


# ---- the reference's own trainer tests (test_trainer.cpp), on the 47-sample grid
def _fixture_weights():  # test_trainer.cpp:14-33
    re_ = np.array([[0.1 * ((j * 47 + i) % 7) - 0.2 for i in range(47)] for j in range(3)])
    rd = np.array([[0.1 * ((i * 3 + j) % 5) - 0.1 for j in range(3)] for i in range(47)])
    return re_, rd


def _fixture_batch():  # test_trainer.cpp:35-47 (math.sin / cos are the same libm calls)
    import math

    r1 = [0.5 + 0.4 * math.sin(0.3 * i) for i in range(47)]
    l1 = [0.9 - 0.3 * math.cos(0.21 * i) for i in range(47)]
    r2 = [0.2 + 0.15 * math.cos(0.17 * i + 0.5) for i in range(47)]
    l2 = [1.1 + 0.5 * math.sin(0.13 * i + 1.0) for i in range(47)]
    return (torch.tensor([r1, r2], dtype=torch.float64).cuda(), torch.tensor([l1, l2], dtype=torch.float64).cuda())


def test_losses_match_the_reference_frozen_oracle(api, ctx):
    """test_trainer.cpp:157-185: loss values frozen by the reference, at 1e-12."""
    re_, rd = _fixture_weights()
    r, l = _fixture_batch()
    lw = (0.5, 0.75, 1.0, 0.5, 0.25)
    losses, _, _ = api.codec_train_grad(ctx, re_, rd, 10.0, r, l, loss_weights=lw, grads=False)
    want = {"e2e": 119.51570838334069, "rec": 8.6159307933410965, "code": 386.44524053693732,
            "col": 1069400.7938603153, "alg": 0.88953050349034479, "total": 535153.28435560723}
    for name, v in want.items():
        assert losses[name] == pytest.approx(v, rel=1e-12), name


def test_alg_regularizer_closed_form(api, ctx):
    """test_trainer.cpp:188-200: beta = 100, every raw entry 0.5 -> loss_alg = 47 / 8."""
    r, l = _fixture_batch()
    losses, _, _ = api.codec_train_grad(ctx, np.full((3, 47), 0.5), np.full((47, 3), 0.5), 100.0, r, l, grads=False)
    assert losses["alg"] == pytest.approx(47.0 / 8.0, rel=1e-14)


def test_losses_reject_malformed_batches(api, ctx):
    """test_trainer.cpp:218-227."""
    re_, rd = _fixture_weights()
    r, l = _fixture_batch()
    with pytest.raises(ValueError):
        api.codec_train_grad(ctx, re_, rd, 10.0, r[:0], l[:0])
    with pytest.raises(ValueError):
        api.codec_train_grad(ctx, re_, rd, 10.0, r, l[:1])


@pytest.mark.parametrize("lw", [(1, 0, 0, 0, 0), (0, 1, 0, 0, 0), (0, 0, 1, 0, 0), (0, 0, 0, 1, 0), (0, 0, 0, 0, 1),
                                (0.5, 0.75, 1.0, 0.5, 0.25)])
def test_gradients_match_finite_differences(api, ctx, lw):
    """test_trainer.cpp:100-140, :229-272: central differences of the GPU total loss over a
    strided parameter subset against the GPU's analytic gradient, relative L2 <= 1e-4."""
    re0 = np.array([0.06 * (i % 7) - 0.35 for i in range(3 * 47)]).reshape(3, 47)
    rd0 = np.array([0.06 * (i % 5) - 0.30 for i in range(47 * 3)]).reshape(47, 3)
    r, l = _fixture_batch()
    _, ge, gd = api.codec_train_grad(ctx, re0, rd0, 10.0, r, l, loss_weights=lw)
    h = 1e-5
    num = den_a = den_f = 0.0
    checked = 0
    for which, raw, g in (("enc", re0, ge), ("dec", rd0, gd)):
        flat, gflat = raw.reshape(-1), g.reshape(-1)
        for i in range(0, flat.size, 3):
            tot = []
            for d in (h, -h):
                w = flat.copy()
                w[i] += d
                w = w.reshape(raw.shape)
                args = (w, rd0) if which == "enc" else (re0, w)
                tot.append(api.codec_train_grad(ctx, *args, 10.0, r, l, loss_weights=lw, grads=False)[0]["total"])
            fd = (tot[0] - tot[1]) / (2.0 * h)
            num += (gflat[i] - fd) ** 2
            den_a += gflat[i] ** 2
            den_f += fd ** 2
            checked += 1
    assert checked >= 64
    assert np.sqrt(num) / max(1e-12, np.sqrt(max(den_a, den_f))) <= 1e-4
