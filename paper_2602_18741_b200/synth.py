"""Seeded synthetic inputs for BASELINE.json's five configs.

Small assets (codec E / D, palettes, light SPDs, MLP weights) are drawn on the
host with the reference's own generators, restated:
  gaussian_curve   spectrum.cpp:97-105
  blackbody_curve  dataset.cpp:503-516 (Planck, c2 = 1.4387768775e7 nm K,
                   zeroed outside 400-700 nm, unit peak)
  Rng / streams    rng.cpp:32-81
  Glorot init      init_upsampler_weights, upsampler.cpp:146-168
Large per-pixel arrays (G-buffers, chain samples, textures, spectrum batches)
come from counter streams keyed by ``stream_key(seed, purpose)``, generated on
the device by ``hc_synth_*`` (or here in numpy for small CPU-side cases); the
values depend only on the global element index, never on sharding.
"""
from __future__ import annotations

import math

import numpy as np

from .colorimetry import grid
from .rng import Rng, ctr_u24, ctr_u64, stream_key

BLACKBODY_C2_NM_K = 1.4387768775e7


def gaussian_curve(center: float, sigma: float, amp: float, n: int) -> list[float]:
    lo, step = grid(n)
    out = []
    for i in range(n):
        d = ((lo + step * i) - center) / sigma
        out.append(amp * math.exp(-0.5 * d * d))
    return out


def blackbody_curve(kelvin: float, n: int) -> list[float]:
    lo, step = grid(n)
    s = []
    for i in range(n):
        lam = lo + step * i
        x = BLACKBODY_C2_NM_K / (lam * kelvin)
        v = 1.0 / (math.pow(lam / 560.0, 5.0) * math.expm1(x))
        if lam < 400.0 or lam > 700.0:  # zero_outside_active_band (spectrum.cpp:90-95)
            v = 0.0
        s.append(v)
    peak = max(s)
    if peak > 0.0:
        alpha = 1.0 / peak
        s = [alpha * v for v in s]
    return s


def gm_spectrum(rng: Rng, n: int) -> list[float]:
    """Sum of 1-4 Gaussians (centre U[380,780], sigma U[10,100], amp U[0,1]), clipped to [0,1]."""
    m = 1 + rng.index(4)
    comps = [(rng.uniform(380.0, 780.0), rng.uniform(10.0, 100.0), rng.uniform(0.0, 1.0)) for _ in range(m)]
    acc = [0.0] * n
    for c, s, a in comps:
        g = gaussian_curve(c, s, a, n)
        acc = [x + y for x, y in zip(acc, g)]
    return [min(max(v, 0.0), 1.0) for v in acc]


def gm_spectra_ctr(seed: int, purpose: str, first: int, count: int, n: int) -> np.ndarray:
    """Host twin of hc_synth_gm_spectra: item i uses Rng(ctr(key, first + i))."""
    key = stream_key(seed, purpose)
    seeds = ctr_u64(key, np.arange(first, first + count, dtype=np.uint64))
    return np.array([gm_spectrum(Rng(int(s)), n) for s in seeds], dtype=np.float32).reshape(count, n)


def palette(seed: int, count: int = 256, n: int = 81, purpose: str = "scene.palette") -> np.ndarray:
    rng = Rng.stream(seed, purpose)
    return np.array([gm_spectrum(rng, n) for _ in range(count)], dtype=np.float32)


def light_spd(rng: Rng, n: int) -> list[float]:
    """Coin flip: blackbody T ~ U[2000, 10000] K, or 1-3 Gaussian peaks sigma U[5, 20] nm; unit peak."""
    if rng.uniform() < 0.5:
        return blackbody_curve(rng.uniform(2000.0, 10000.0), n)
    m = 1 + rng.index(3)
    comps = [(rng.uniform(380.0, 780.0), rng.uniform(5.0, 20.0), rng.uniform(0.0, 1.0)) for _ in range(m)]
    acc = [0.0] * n
    for c, s, a in comps:
        g = gaussian_curve(c, s, a, n)
        acc = [x + y for x, y in zip(acc, g)]
    peak = max(acc)
    if peak > 0.0:
        alpha = 1.0 / peak
        acc = [alpha * v for v in acc]
    return acc


def lights(seed: int, count: int, n: int = 81, purpose: str = "scene.lights") -> np.ndarray:
    rng = Rng.stream(seed, purpose)
    return np.array([light_spd(rng, n) for _ in range(count)], dtype=np.float32)


def codec_weights(seed: int, k: int, n: int = 81) -> tuple[np.ndarray, np.ndarray]:
    """E (k x n) and D (n x k): U[0,1) draws, each row normalised to sum 1, stored f32."""

    def mat(purpose: str, rows: int, cols: int) -> np.ndarray:
        rng = Rng.stream(seed, purpose)
        m = np.array([[rng.uniform() for _ in range(cols)] for _ in range(rows)], dtype=np.float64)
        return (m / m.sum(axis=1, keepdims=True)).astype(np.float32)

    return mat("codec.E", k, n), mat("codec.D", n, k)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 values."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def mlp_weights(seed: int, k: int = 6, hidden: int = 64) -> dict:
    """init_upsampler_weights (upsampler.cpp:146-168) Glorot draws from stream
    'upsampler.init' (w1 h x 3, w2 h x h, w3 k x h), biases U[-0.1, 0.1] from
    'upsampler.bias' (b1, b2, b3).  Weights rounded to bf16 (tensor-core operands)."""
    rng = Rng.stream(seed, "upsampler.init")

    def glorot(fan_in: int, fan_out: int, count: int) -> np.ndarray:
        lim = math.sqrt(6.0 / (fan_in + fan_out))
        return np.array([rng.uniform(-lim, lim) for _ in range(count)], dtype=np.float64)

    w1 = glorot(3, hidden, hidden * 3).reshape(hidden, 3)
    w2 = glorot(hidden, hidden, hidden * hidden).reshape(hidden, hidden)
    w3 = glorot(hidden, k, k * hidden).reshape(k, hidden)
    rb = Rng.stream(seed, "upsampler.bias")
    b1 = np.array([rb.uniform(-0.1, 0.1) for _ in range(hidden)])
    b2 = np.array([rb.uniform(-0.1, 0.1) for _ in range(hidden)])
    b3 = np.array([rb.uniform(-0.1, 0.1) for _ in range(k)])
    # Biases are drawn bf16-representable: layer 1's bias rides the tensor-core
    # operand (constant-1 input column), so all three are kept on the bf16 grid.
    return {
        "w1": bf16_round(w1), "b1": bf16_round(b1),
        "w2": bf16_round(w2), "b2": bf16_round(b2),
        "w3": bf16_round(w3), "b3": bf16_round(b3),
        "w1_f64": w1, "w2_f64": w2, "w3_f64": w3,
    }


# ----------------------------------------------------------------- per-element arrays (numpy twins)
def gbuffer_np(seed: int, first: int, P: int, L: int, n_pal: int) -> tuple[np.ndarray, np.ndarray]:
    ki, kc = stream_key(seed, "gbuffer.idx"), stream_key(seed, "gbuffer.cos")
    idx = (ctr_u64(ki, np.arange(first, first + P, dtype=np.uint64)) % np.uint64(n_pal)).astype(np.uint32)
    cosv = ctr_u24(kc, np.arange(first * L, (first + P) * L, dtype=np.uint64)).reshape(P, L)
    return idx, cosv


def chain_np(seed: int, first: int, P: int, spp: int, n_pal: int, n_ill: int):
    kp, ki, kt = (stream_key(seed, p) for p in ("chain.pidx", "chain.iidx", "chain.tw"))
    g4 = np.arange(first * spp * 4, (first + P) * spp * 4, dtype=np.uint64)
    g1 = np.arange(first * spp, (first + P) * spp, dtype=np.uint64)
    pidx = (ctr_u64(kp, g4) % np.uint64(n_pal)).astype(np.uint8).reshape(P, spp, 4)
    tw = ctr_u24(kt, g4).reshape(P, spp, 4)
    iidx = (ctr_u64(ki, g1) % np.uint64(n_ill)).astype(np.uint8).reshape(P, spp)
    return pidx, iidx, tw


def uniform_np(seed: int, purpose: str, first: int, count: int) -> np.ndarray:
    return ctr_u24(stream_key(seed, purpose), np.arange(first, first + count, dtype=np.uint64))


def cornell_scene(n: int, block: bool = False) -> dict:
    """The reference render benchmark's enclosed test scene (benchmarks/bm_render.cpp:14-36):
    grey / red / green walls, open front, a grey sphere and a ceiling area light; with
    `block`, a second (axis-aligned box) object exercises hit_block (renderer.cpp:342-381)."""
    grey = [0.7] * n
    red = gaussian_curve(620.0, 60.0, 0.6, n)
    green = gaussian_curve(540.0, 60.0, 0.6, n)
    scene = {
        "materials": [grey, red, green],
        "wall_material": [1, 2, 0, 0, 0, -1],
        "objects": [{"kind": "sphere", "center": (0.35, 0.4, -0.3), "radius": 0.4, "material": 0}],
        "lights": [{"corner": (-0.25, 1.999, -0.25), "edge_u": (0.5, 0.0, 0.0), "edge_v": (0.0, 0.0, 0.5),
                    "spd": [1.0] * n, "scale": 12.0}],
    }
    if block:
        scene["objects"].append({"kind": "block", "box_min": (-0.7, 0.0, -0.6), "box_max": (-0.2, 0.9, -0.1),
                                 "material": 1})
        scene["lights"].append({"corner": (0.9, 1.2, 0.5), "edge_u": (0.0, 0.0, -0.3), "edge_v": (0.0, -0.3, 0.0),
                                "spd": gaussian_curve(580.0, 80.0, 1.0, n), "scale": 3.0})
    return scene
