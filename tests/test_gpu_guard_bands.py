"""Out-of-bounds writes: every output of the hot-path entry points is placed inside a larger
device buffer filled with a sentinel bit pattern; after the call the bands on both sides must be
untouched and the output must equal the one written into a plain buffer.

compute-sanitizer is closed on this GPU pool (profiles/r02/sanitizer_closed.txt), so this is the
library's own bounds check on the writes of the TMA bulk-store, vector-store and generic tile
paths: ragged row counts (1, 129, 20011: a lone row, one full tile + 1, many tiles + a ragged
tail), 16-byte-aligned and 4-byte-offset outputs (the bulk-copy path and the generic path)."""
import numpy as np
import pytest

from paper_2602_18741_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 424242
GUARD = 4096  # floats on each side
SENTINEL = 0x7FC0DEAD  # a quiet NaN payload no kernel produces
ROWS = (1, 129, 20011)


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


class Guarded:
    """A float32 [rows, width] output inside a sentinel-filled buffer, `offset` floats past a
    16-byte-aligned position."""

    def __init__(self, rows: int, width: int, offset: int):
        self.n = rows * width
        self.lo = GUARD + offset
        self.big = torch.full((2 * GUARD + self.n + 8,), SENTINEL, dtype=torch.int32, device="cuda")
        self.view = self.big.view(torch.float32)[self.lo:self.lo + self.n].view(rows, width)
        assert self.view.data_ptr() % 16 == (4 * offset) % 16

    def check(self, name: str, plain: torch.Tensor, exact: bool):
        torch.cuda.synchronize()
        before, after = self.big[:self.lo], self.big[self.lo + self.n:]
        assert bool((before == SENTINEL).all()), f"{name}: wrote before the output"
        assert bool((after == SENTINEL).all()), f"{name}: wrote past the output"
        got, want = self.view.cpu().numpy(), plain.cpu().numpy()
        assert not np.any(got.view(np.int32) == SENTINEL), f"{name}: output words left unwritten"
        if exact:
            assert np.array_equal(got, want), f"{name}: differs from the plain-buffer run"
        else:  # the generic (unaligned) tile path may order its FMAs differently
            den = np.maximum(np.abs(want), np.max(np.abs(want), axis=-1, keepdims=True))
            assert float(np.max(np.abs(got - want) / np.maximum(den, 1e-30))) <= 1e-5, name


def _run(name, widths, rows, offset, call):
    """call(out_dict_or_None) -> dict of outputs; widths: {key: width}."""
    plain = call(None)
    guarded = {k: Guarded(rows, w, offset) for k, w in widths.items()}
    call({k: g.view for k, g in guarded.items()})
    for k, g in guarded.items():
        g.check(f"{name}.{k} rows={rows} offset={offset}", plain[k], exact=offset == 0)


def _scene(api, ctx, k, L, n=81):
    E, D = synth.codec_weights(SEED, k, n)
    codec = api.Codec(ctx, E, D)
    pal = torch.from_numpy(synth.palette(SEED, 256, n)).cuda()
    lights = synth.lights(SEED, L, n)
    pal_codes = codec.encode(pal)
    light_codes = codec.encode(torch.from_numpy(lights).cuda()).cpu().numpy()
    return codec, pal, lights, pal_codes, light_codes


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("rows", ROWS)
def test_roundtrip_outputs_stay_in_bounds(api, ctx, rows, offset):
    for k in (6, 9):
        E, D = synth.codec_weights(SEED, k, 81)
        codec = api.Codec(ctx, E, D)
        S = api.synth_gm_spectra(ctx, SEED, "guard.spectra", 0, rows, 81)
        _run(f"roundtrip k={k}", {"codes": k, "spectra": 81, "xyz": 3, "rgb": 3}, rows, offset,
             lambda out: codec.roundtrip(S, out=out))


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("rows", ROWS)
@pytest.mark.parametrize("k,L", [(6, 8), (9, 32), (3, 8)])
def test_shade_outputs_stay_in_bounds(api, ctx, k, L, rows, offset):
    codec, pal, lights, pal_codes, light_codes = _scene(api, ctx, k, L)
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, rows, L, 256)
    _run(f"shade_latent k={k} L={L}", {"latent": k, "spectra": 81, "xyz": 3, "rgb": 3}, rows, offset,
         lambda out: codec.shade_latent(pal_codes, light_codes, idx, cosv, latent=True, spectra=True, out=out))
    _run(f"shade_latent(xyz, rgb) k={k} L={L}", {"xyz": 3, "rgb": 3}, rows, offset,
         lambda out: codec.shade_latent(pal_codes, light_codes, idx, cosv,
                                        out=None if out is None else {**out, "latent": None, "spectra": None}))
    _run(f"shade_spectral L={L}", {"spectra": 81, "xyz": 3, "rgb": 3}, rows, offset,
         lambda out: codec.shade_spectral(pal, lights, idx, cosv, spectra=True, out=out))
    _run(f"shade_spectral(xyz, rgb) L={L}", {"xyz": 3, "rgb": 3}, rows, offset,
         lambda out: codec.shade_spectral(pal, lights, idx, cosv,
                                          out=None if out is None else {**out, "spectra": None}))


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("rows,spp", [(1, 64), (129, 64), (1031, 64), (257, 24)])
@pytest.mark.parametrize("k", [6, 3, 9])
def test_chain_outputs_stay_in_bounds(api, ctx, k, rows, spp, offset):
    codec, pal, lights, pal_codes, _ = _scene(api, ctx, k, 16)
    ill = torch.from_numpy(lights).cuda()
    ill_codes = codec.encode(ill)
    pidx, iidx, tw = api.synth_chain(ctx, SEED, 0, rows, spp, 256, 16)
    _run(f"multibounce_latent k={k} spp={spp}", {"latent": k, "xyz": 3, "rgb": 3}, rows, offset,
         lambda out: codec.multibounce_latent(pal_codes, ill_codes, pidx, iidx, tw, latent=True, out=out))
    if k == 6 and spp in (8, 16, 32, 64):  # the naive chain is compiled for these sample counts
        _run(f"multibounce_spectral spp={spp}", {"xyz": 3, "rgb": 3}, rows, offset,
             lambda out: codec.multibounce_spectral(pal, ill, pidx, iidx, tw, out=out))


@pytest.mark.parametrize("offset", [0, 2])  # k = 6 stores float2: 8-byte-aligned codes
@pytest.mark.parametrize("rows", ROWS)
@pytest.mark.parametrize("k", [6, 9])
def test_mlp_output_stays_in_bounds(api, ctx, k, rows, offset):
    mlp = api.CodeMLP(ctx, synth.mlp_weights(SEED, k=k))
    rgb = api.synth_uniform(ctx, SEED, "guard.rgb", 0, rows * 3)
    plain = mlp.forward(rgb)
    g = Guarded(rows, k, offset)
    mlp.forward(rgb, out=g.view)
    g.check(f"mlp k={k} rows={rows} offset={offset}", plain, exact=True)
