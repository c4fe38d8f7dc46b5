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
