"""GPU path tracer (render / render_latent_multipass, renderer.cpp:437-659)
against the reference's own render() compiled in oracle/_ref, through the C ABI.

Bars: images and shading-evaluation counts bit-identical to the reference (same
streams, same fp64 geometry / fp32 channel arithmetic, no contraction, correctly rounded
sin / cos); per-pixel path hashes identical across our render modes (the reference's
contract, renderer.hpp:66-70) and equal to the reference's wherever glibc's sin / cos
is correctly rounded (glibc is within 1 ulp; ~0.16 % of its results are not the
correctly rounded value), which here is >= 90 % of pixels.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2602_18741_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def _reference(api, scene, n, k, E, D, mode, W, H, spp, depth, seed, multipass=False):
    ref = oracle.reference(n)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    sc, keep = api.scene_struct(scene, n)
    job = api.HcRenderJob(api.RENDER_MODES["latent" if multipass else mode], W, H, spp, depth, seed)
    ch = {"spectral": n, "latent": k, "rgb": 3}["latent" if multipass else mode]
    img = np.zeros((H, W, ch), np.float32)
    hashes = np.zeros(W * H, np.uint64)
    ev = C.c_uint64()
    rc = ref.ref_render(C.addressof(sc), C.addressof(job), k, E, D, int(multipass), img.reshape(-1), hashes,
                        C.byref(ev))
    assert rc == 0
    return img, hashes, ev.value


@pytest.mark.parametrize("mode,n,k,depth,block,multipass", [
    ("spectral", 81, 6, 3, False, False), ("latent", 81, 6, 3, True, False), ("rgb", 81, 6, 3, True, False),
    ("latent", 47, 9, -1, True, False), ("spectral", 47, 6, -1, True, False), ("latent", 81, 6, 3, True, True),
    ("latent", 81, 3, 0, True, False), ("rgb", 47, 6, 1, False, False), ("latent", 47, 9, 2, True, True)])
def test_render_bit_exact_vs_reference(api, ctx, mode, n, k, depth, block, multipass):
    E, D = synth.codec_weights(11, k, n)
    codec = api.Codec(ctx, E, D)
    scene = synth.cornell_scene(n, block)
    W, H, spp, seed = 40, 24, 8, 5
    got = api.render(codec, scene, mode, W, H, spp, depth, seed, path_hashes=True, multipass=multipass)
    fast = api.render(codec, scene, mode, W, H, spp, depth, seed, multipass=multipass)  # sample-parallel path
    img, hashes, evals = _reference(api, scene, n, k, E, D, mode, W, H, spp, depth, seed, multipass)
    for r in (got, fast):
        g = r["image"].cpu().numpy()
        assert g.shape == img.shape
        assert np.array_equal(g, img), f"{int(np.sum(g != img))} values differ"
        assert r["shading_evals"] == evals
    eq = np.mean(got["path_hashes"].cpu().numpy().view(np.uint64).reshape(-1) == hashes)
    print(f"{mode} n={n} k={k} depth={depth}: path-hash agreement {eq:.4f}")
    assert eq >= 0.9


def test_path_hashes_identical_across_modes_and_multipass_equals_single(api, ctx):
    """renderer.hpp:66-70 (geometry never touches channel data) and :103-105 (multipass ==
    single k-channel latent render at fixed depth)."""
    n, k = 81, 6
    E, D = synth.codec_weights(3, k, n)
    codec = api.Codec(ctx, E, D)
    scene = synth.cornell_scene(n, True)
    runs = {m: api.render(codec, scene, m, 32, 20, 4, 3, 9, path_hashes=True) for m in ("spectral", "latent", "rgb")}
    mp = api.render(codec, scene, "latent", 32, 20, 4, 3, 9, path_hashes=True, multipass=True)
    h = [r["path_hashes"].cpu().numpy() for r in list(runs.values()) + [mp]]
    assert all(np.array_equal(h[0], x) for x in h[1:])
    assert np.array_equal(runs["latent"]["image"].cpu().numpy(), mp["image"].cpu().numpy())
    assert runs["spectral"]["shading_evals"] == runs["latent"]["shading_evals"] * n // (k // 3)


def test_render_rejects_invalid_jobs_and_scenes(api, ctx):
    n = 81
    E, D = synth.codec_weights(3, 6, n)
    codec = api.Codec(ctx, E, D)
    scene = synth.cornell_scene(n)
    with pytest.raises(ValueError):
        api.render(codec, scene, "spectral", 0, 8, 1, 3)
    with pytest.raises(ValueError):
        api.render(codec, scene, "spectral", 8, 8, 1, -2)
    bad = dict(scene, wall_material=[1, 2, 0, 0, 7, -1])
    with pytest.raises(ValueError):
        api.render(codec, bad, "latent", 8, 8, 1, 3)
    bad = dict(scene, objects=[dict(scene["objects"][0], material=5)])
    with pytest.raises(ValueError):
        api.render(codec, bad, "rgb", 8, 8, 1, 3)
    bad = dict(scene, lights=[dict(scene["lights"][0], edge_u=(0.0, 0.0, 0.0))])
    with pytest.raises(ValueError):
        api.render(codec, bad, "spectral", 8, 8, 1, 3)
