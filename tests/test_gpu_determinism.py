"""Run-to-run determinism of the mbarrier / TMA / TMEM pipelines: compute-sanitizer's racecheck
is closed on this GPU pool (profiles/r02/sanitizer_closed.txt), so races are looked for the other
way round — a missing wait or an early buffer re-use shows up as outputs that differ between
identical launches.  Each hot-path kernel runs REPS times on the same inputs at sizes that wrap
its shared-memory ring many times per CTA (several tiles per CTA on all 148 SMs) while another
stream keeps the memory system busy; every output must be bit-identical to the first run's."""
import numpy as np
import pytest

from paper_2602_18741_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 90210
REPS = 12


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def _repeat(name, call):
    """call() -> dict / tensor of device outputs (fresh buffers every time)."""
    noise_stream = torch.cuda.Stream()
    junk = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    first = None
    for rep in range(REPS):
        with torch.cuda.stream(noise_stream):  # concurrent traffic: 256 MB of writes + reads
            junk.add_(1.0)
        out = call()
        out = out if isinstance(out, dict) else {"out": out}
        torch.cuda.synchronize()
        got = {k: v.clone() for k, v in out.items() if v is not None}
        if first is None:
            first = got
            continue
        for k, v in got.items():
            same = torch.equal(v.view(torch.int32) if v.dtype == torch.float32 else v.view(torch.int64),
                               first[k].view(torch.int32) if v.dtype == torch.float32 else first[k].view(torch.int64))
            assert same, f"{name}.{k}: run {rep} differs from run 0"


def _scene(api, ctx, k, L, n=81):
    E, D = synth.codec_weights(SEED, k, n)
    codec = api.Codec(ctx, E, D)
    pal = torch.from_numpy(synth.palette(SEED, 256, n)).cuda()
    lights = synth.lights(SEED, L, n)
    return codec, pal, lights, codec.encode(pal), codec.encode(torch.from_numpy(lights).cuda()).cpu().numpy()


@pytest.mark.parametrize("k,L,P", [(6, 8, 1920 * 1080), (9, 32, 600_011), (3, 8, 300_007)])
def test_shade_is_deterministic(api, ctx, k, L, P):
    codec, pal, lights, pal_codes, light_codes = _scene(api, ctx, k, L)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, P, L, 256)
    _repeat(f"shade_latent k={k} L={L}",
            lambda: codec.shade_latent(pal_codes, light_codes, idx, cosv, latent=True, spectra=(L == 32)))
    _repeat(f"shade_spectral L={L}", lambda: codec.shade_spectral(pal, lights, idx, cosv, spectra=(L == 32)))


def test_roundtrip_is_deterministic(api, ctx):
    codec, *_ = _scene(api, ctx, 6, 8)
    S = api.synth_gm_spectra(ctx, SEED, "det.spectra", 0, 400_003, 81)
    _repeat("roundtrip", lambda: codec.roundtrip(S))


@pytest.mark.parametrize("k", [6, 3, 9])
def test_chain_is_deterministic(api, ctx, k):
    codec, pal, lights, pal_codes, _ = _scene(api, ctx, k, 16)
    ill = torch.from_numpy(lights).cuda()
    ill_codes = codec.encode(ill)
    pidx, iidx, tw = api.synth_chain(ctx, SEED, 0, 150_001, 64, 256, 16)
    _repeat(f"multibounce_latent k={k}", lambda: codec.multibounce_latent(pal_codes, ill_codes, pidx, iidx, tw))
    if k == 6:
        _repeat("multibounce_spectral", lambda: codec.multibounce_spectral(pal, ill, pidx[:20_000], iidx[:20_000],
                                                                            tw[:20_000]))


@pytest.mark.parametrize("k", [6, 9])
def test_mlp_is_deterministic(api, ctx, k):
    mlp = api.CodeMLP(ctx, synth.mlp_weights(SEED, k=k))
    rgb = api.synth_uniform(ctx, SEED, "det.rgb", 0, 3 * (2_000_000 + 77))
    _repeat(f"mlp k={k}", lambda: mlp.forward(rgb))


def test_loss_is_deterministic(api, ctx):
    codec, *_ = _scene(api, ctx, 6, 8)
    A = api.synth_gm_spectra(ctx, SEED, "det.a", 0, 500_009, 81)
    B = api.synth_gm_spectra(ctx, SEED, "det.b", 0, 500_009, 81)
    _repeat("hadamard_loss", lambda: codec.hadamard_loss(A, B))
