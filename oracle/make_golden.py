"""Generate package data and golden fixtures from the COMPILED REFERENCE.

Runs only in the build container (needs /root/reference and `make -C oracle ref`).
Outputs (committed):
  (checks) paper_2602_18741_b200/data/cmf_n{47,81}.json against CmfTable of the compiled reference
          (the files themselves are written by tools/make_cmf_tables.py from the CIE tables)
  tests/golden/ref_rng.json                      Rng streams / pixel streams / FNV (rng.cpp)
  tests/golden/ref_generators.json               gaussian_curve / blackbody_curve / Glorot init
  tests/golden/ref_small_cases.npz               small seeded cases of every config, outputs
                                                 computed by the reference shim (oracle/_ref)

    python oracle/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2602_18741_b200 import synth  # noqa: E402
from paper_2602_18741_b200.colorimetry import grid  # noqa: E402

DATA = ROOT / "paper_2602_18741_b200" / "data"
GOLD = ROOT / "tests" / "golden"


def cmf_files() -> None:
    """The package CMF rows (tools/make_cmf_tables.py: CIE tables + an in-repo resampler) must equal
    CmfTable of the compiled reference bit for bit (colorimetry.cpp:45-61)."""
    for n in (47, 81):
        ref = oracle.reference(n)
        t = np.zeros(7 * n)
        ref.ref_cmf_table(t)
        t = t.reshape(7, n)
        lo, step = ref.ref_lambda_min(), ref.ref_lambda_step()
        assert (lo, step) == grid(n), (lo, step, grid(n))
        d = json.loads((DATA / f"cmf_n{n}.json").read_text())
        for i, key in enumerate(("xbar", "ybar", "zbar", "d65")):
            assert d[key] == [float(v) for v in t[i]], f"cmf_n{n}.json {key} differs from the reference CmfTable"


def rng_file() -> None:
    ref = oracle.reference(81)
    out = {"stream": [], "seed": [], "pixel_stream": []}
    for seed, purpose in [(0, "codec.E"), (7, "scene.palette"), (123456789, "upsampler.init"),
                          (2**63 + 5, "gbuffer.idx")]:
        buf = np.zeros(8, dtype=np.uint64)
        ref.ref_rng_stream_u64(seed, purpose.encode(), 8, buf)
        out["stream"].append({"seed": seed, "purpose": purpose, "u64": [int(v) for v in buf]})
    for seed in (0, 1, 0xDEADBEEF):
        buf = np.zeros(8, dtype=np.uint64)
        ref.ref_rng_seed_u64(seed, 8, buf)
        out["seed"].append({"seed": seed, "u64": [int(v) for v in buf]})
    for args in [(0, 1, 2, 3, 0), (42, 1919, 1079, 63, 1)]:
        buf = np.zeros(4, dtype=np.uint64)
        ref.ref_pixel_stream_u64(*args, 4, buf)
        out["pixel_stream"].append({"args": list(args), "u64": [int(v) for v in buf]})
    out["fnv1a64_hello"] = int(ref.ref_fnv1a64(b"hello", 5))
    GOLD.mkdir(parents=True, exist_ok=True)
    (GOLD / "ref_rng.json").write_text(json.dumps(out, indent=1) + "\n")


def generators_file() -> None:
    out = {"gaussian": [], "blackbody": [], "glorot": []}
    for n in (47, 81):
        ref = oracle.reference(n)
        for c, s, a in [(550.0, 30.0, 1.0), (412.5, 7.25, 0.8), (700.0, 99.0, 0.3)]:
            buf = np.zeros(n)
            ref.ref_gaussian_curve(c, s, a, buf)
            out["gaussian"].append({"n": n, "args": [c, s, a], "values": [float(v) for v in buf]})
        for T in (2000.0, 5777.0, 9999.5):
            buf = np.zeros(n)
            ref.ref_blackbody_curve(T, buf)
            out["blackbody"].append({"n": n, "kelvin": T, "values": [float(v) for v in buf]})
    ref = oracle.reference(81)
    k, h, seed = 6, 64, 11
    w1, w2, w3 = np.zeros(h * 3), np.zeros(h * h), np.zeros(k * h)
    ref.ref_init_upsampler(k, h, seed, w1, w2, w3)
    out["glorot"].append({"k": k, "hidden": h, "seed": seed, "w1_head": [float(v) for v in w1[:16]],
                          "w2_head": [float(v) for v in w2[:16]], "w3_head": [float(v) for v in w3[:16]],
                          "w1_sum": float(w1.sum()), "w2_sum": float(w2.sum()), "w3_sum": float(w3.sum())})
    (GOLD / "ref_generators.json").write_text(json.dumps(out, indent=1) + "\n")


def small_cases() -> None:
    """Every config at a tiny size; inputs from the repo's generators, outputs from oracle/_ref."""
    seed = 2602
    ref = oracle.reference(81)
    n = 81
    z: dict[str, np.ndarray] = {}
    for k in (6, 9):
        E, D = synth.codec_weights(seed, k, n)
        z[f"E{k}"], z[f"D{k}"] = E, D
    # config 1: 37 spectra (ragged), k = 6
    S = synth.gm_spectra_ctr(seed, "codec.spectra", 0, 37, n)
    Z, S2, X, R = (np.zeros((37, d), np.float32) for d in (6, n, 3, 3))
    ref.ref_codec_roundtrip(z["E6"], z["D6"], 6, S, 37, Z, S2, X, R, 1)
    z.update(c1_S=S, c1_Z=Z, c1_S2=S2, c1_xyz=X, c1_rgb=R)
    # configs 2/3: palette + lights, G-buffer of 50 px
    pal = synth.palette(seed, 256, n)
    z["palette"] = pal
    for tag, k, L, P in (("c2", 6, 8, 50), ("c3", 9, 32, 22)):
        lt = synth.lights(seed, L, n)
        idx, cosv = synth.gbuffer_np(seed, 0, P, L, 256)
        pc = np.zeros((256, k), np.float32)
        lc = np.zeros((L, k), np.float32)
        ref.ref_asset_codes(z[f"E{k}"], k, pal, 256, pc)
        ref.ref_asset_codes(z[f"E{k}"], k, lt, L, lc)
        lat, S2, X, R = (np.zeros((P, d), np.float32) for d in (k, n, 3, 3))
        ref.ref_shade_latent(z[f"E{k}"], z[f"D{k}"], k, pc, lc, L, idx, np.ascontiguousarray(cosv), P,
                             lat, S2, X, R, 1)
        SS, SX, SR = (np.zeros((P, d), np.float32) for d in (n, 3, 3))
        ref.ref_shade_spectral(pal, lt, L, idx, np.ascontiguousarray(cosv), P, SS, SX, SR, 1)
        z.update({f"{tag}_lights": lt, f"{tag}_idx": idx, f"{tag}_cos": cosv, f"{tag}_palcodes": pc,
                  f"{tag}_lightcodes": lc, f"{tag}_latent": lat, f"{tag}_S2": S2, f"{tag}_xyz": X,
                  f"{tag}_rgb": R, f"{tag}_naive_S": SS, f"{tag}_naive_xyz": SX, f"{tag}_naive_rgb": SR})
    # config 4: 6 px x 16 spp, depth 4, 16 illuminants
    P, spp = 6, 16
    ill = synth.lights(seed, 16, n, purpose="scene.illuminants")
    pc = np.zeros((256, 6), np.float32)
    ic = np.zeros((16, 6), np.float32)
    ref.ref_asset_codes(z["E6"], 6, pal, 256, pc)
    ref.ref_asset_codes(z["E6"], 6, ill, 16, ic)
    pidx, iidx, tw = synth.chain_np(seed, 0, P, spp, 256, 16)
    lat, X, R = (np.zeros((P, d), np.float32) for d in (6, 3, 3))
    ref.ref_multibounce_latent(z["E6"], z["D6"], 6, pc, ic, np.ascontiguousarray(pidx), np.ascontiguousarray(iidx),
                               np.ascontiguousarray(tw), P, spp, 4, lat, X, R, 1)
    SX, SR = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
    ref.ref_multibounce_spectral(pal, ill, np.ascontiguousarray(pidx), np.ascontiguousarray(iidx),
                                 np.ascontiguousarray(tw), P, spp, 4, SX, SR, 1)
    z.update(c4_ill=ill, c4_palcodes=pc, c4_illcodes=ic, c4_pidx=pidx, c4_iidx=iidx, c4_tw=tw, c4_latent=lat,
             c4_xyz=X, c4_rgb=R, c4_naive_xyz=SX, c4_naive_rgb=SR)
    # config 5a: MLP on 40 texels; 5b: loss on 29 pairs
    w = synth.mlp_weights(seed, 6, 64)
    rgb = synth.uniform_np(seed, "mlp.input", 0, 40 * 3).reshape(40, 3)
    out = np.zeros((40, 6), np.float32)
    ref.ref_mlp_forward(np.ascontiguousarray(rgb), 40, 64, 6, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"],
                        w["b3"], out, 1)
    z.update({f"c5_{key}": w[key] for key in ("w1", "b1", "w2", "b2", "w3", "b3")})
    z.update(c5_rgb=rgb, c5_codes=out)
    A = synth.gm_spectra_ctr(seed, "loss.a", 0, 29, n)
    B = synth.gm_spectra_ctr(seed, "loss.b", 0, 29, n)
    loss = ref.ref_hadamard_loss(z["E6"], z["D6"], 6, A, B, 29, 1)
    z.update(c5b_A=A, c5b_B=B, c5b_loss=np.array([loss]))
    np.savez_compressed(GOLD / "ref_small_cases.npz", **z)


def main() -> int:
    if not oracle.REFERENCE_CORE.is_dir():
        print("reference sources not present; nothing to generate", file=sys.stderr)
        return 1
    oracle.build(with_reference=True)
    cmf_files()
    rng_file()
    generators_file()
    small_cases()
    print("wrote", DATA, GOLD)
    return 0


if __name__ == "__main__":
    sys.exit(main())
