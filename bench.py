#!/usr/bin/env python
"""hadacodec-b200 benchmark (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1|2|3|4|5a|5b|6|7|8|9|10] [--all] [--no-cpu-baseline]

Default workload = BASELINE.json configs[1] ("config 2"): 1920x1080 G-buffer,
k = 6 (2 RGB passes), 8 lights, latent Hadamard shade + reassembly + decode
folded to XYZ and linear sRGB; metric Mpixel/s.  A step is one frame per GPU
(weak scaling: rank r renders rows [r*1080, (r+1)*1080) of an N-frame-tall
image; no collective on the data path).  Inputs are resident in HBM, rotated
over enough buffer sets that one rotation exceeds 2x the 126 MB L2, and the K
steps are replayed from a CUDA graph (a 19 us ideal frame is launch-bound
otherwise); timing = CUDA events on the launching stream, max over ranks.

e2e: the same frame through the reference-facing host-buffer C-ABI call
(hc_shade_latent_host): pinned host G-buffer in, XYZ + sRGB out, copies inside
the timed region.

cpu_baseline / --impl reference: the reference's own CPU implementation
(oracle/_ref: the reference core compiled from its sources + the G-buffer
restatement) on the host's cores; see DESIGN.md.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

from paper_2602_18741_b200.colorimetry import cmf_analytic

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"
METRIC = BASELINE["metric"]
SEED = 2602
N_SPEC = 81

# Per-config shape, algorithmic bytes per unit and unit names.
CONFIGS = {
    "1": dict(name="codec round trip N=2^20, n=81, k=6 -> codes+spectra+XYZ+sRGB", units=1 << 20, k=6,
              unit="M spectra/s", bytes_per_unit=696, rot=2, cmf="analytic"),
    "2": dict(name="1920x1080 G-buffer, k=6 (2 RGB passes), 8 lights, latent shade -> XYZ+sRGB",
              W=1920, H=1080, k=6, L=8, unit="Mpixel/s", bytes_per_unit=60, rot=8),
    "3": dict(name="3840x2160 G-buffer, k=9 (3 RGB passes), 32 lights, latent shade -> spectra(81)+sRGB",
              W=3840, H=2160, k=9, L=32, unit="Mpixel/s", bytes_per_unit=468, rot=2),
    "4": dict(name="2048x2048, 64 spp, depth 4, k=6 multi-bounce accumulate -> XYZ+sRGB",
              W=2048, H=2048, k=6, spp=64, unit="Mpixel/s", bytes_per_unit=1368, rot=1),
    "5a": dict(name="4096x4096 RGB -> code MLP 3-64-64-6 (bf16 tcgen05)", W=4096, H=4096, k=6,
               unit="Mpixel/s", bytes_per_unit=36, flops_per_unit=9344, rot=2),
    "5b": dict(name="Hadamard near-multiplicativity loss, 2^24 pairs, n=81, k=6", units=1 << 24, k=6,
               unit="M pairs/s", bytes_per_unit=648, rot=1),
    # SURVEY §8f row 1 (the next row): the colour-metric tail of a config-2 frame.
    "6": dict(name="1920x1080 colour-metric tail: scene_color_report(naive n=81 sRGB, latent k=6 sRGB) "
                   "+ tonemap_srgb8 preview of the latent frame", W=1920, H=1080, k=6, L=8, unit="Mpixel/s",
              bytes_per_unit=27, rot=8, dtype="f64"),
    # the reference's path tracer, latent k = 6 (naive: spectral n = 81).
    # Units are pixel-samples; the algorithmic bytes are the image writes (k floats per pixel
    # over spp samples), so the HBM fraction is ~0: the tracer is fp64 / latency bound.
    # codes CSV on the device — write_codes_csv (%.17g) then read_codes_csv
    # (exact strtod) of 2^21 rows x k = 6 codes; algorithmic bytes per code: 4 B float in, the
    # ~20 B of text written and read back, 8 B double out.
    "8": dict(name="codes CSV round trip on the device: write_codes_csv (%.17g) + read_codes_csv (exact "
                   "strtod), 2^21 rows x k=6", units=(1 << 21) * 6, rows=1 << 21, k=6, unit="M codes/s",
              bytes_per_unit=52, rot=1, graph=False, dtype="f64"),
    # the reference's `encode` tool (tools/main.cpp:285-308) on the device —
    # read_spectra_csv of 2^17 curves measured on a 4 nm 360-800 grid (111 samples, %.9g), resample
    # onto the 81-sample grid + zero outside 400-700 + fp64 encode (k = 6), write_codes_csv
    # (%.17g); algorithmic bytes per curve: its ~1.2 KB of input text + ~120 B of output text.
    "9": dict(name="encode tool on the device: spectra CSV (2^17 curves x 111 samples, 4 nm) -> resample + "
                   "fp64 encode (k=6) -> codes CSV", units=1 << 17, rows=1 << 17, m=111, k=6, unit="M curves/s",
              bytes_per_unit=1330, rot=1, graph=False, dtype="f64"),
    # the codec training objective — compute_losses + gradients
    # (trainer.cpp:108-373), bit-identical — over one batch of 2^16 (reflectance, illumination)
    # pairs, k = 6, default LossWeights; algorithmic bytes per pair: its two 81-sample curves.
    "10": dict(name="codec training objective: losses + analytic gradients (bit-identical fp64) over 2^16 "
                    "pairs, k=6, n=81", units=1 << 16, m=1 << 16, k=6, unit="M pairs/s", bytes_per_unit=2 * 81 * 8,
               rot=1, graph=False, dtype="f64"),
    "7": dict(name="Cornell box path trace (bm_render scene + block + 2nd light), 256x256, 64 spp, depth 3, "
                   "latent k=6 (naive: spectral n=81)", W=256, H=256, spp=64, depth=3, k=6,
              unit="M samples/s", bytes_per_unit=6 * 4 / 64, rot=1, graph=False, dtype="f64"),
}


# fp32-issue bound of the naive n = 81 paths: lane-ops per unit at 148 SMs x 128
# fp32 lanes x the max SM clock (1.965 GHz).
FP32_LANE_OPS_PER_S = 148 * 128 * 1.965e9
NAIVE_BOUND = {"2": {"lane_ops_per_unit": 981, "lane_ops_per_s": FP32_LANE_OPS_PER_S},
               "3": {"lane_ops_per_unit": 2925, "lane_ops_per_s": FP32_LANE_OPS_PER_S},
               "4": {"lane_ops_per_unit": 62460, "lane_ops_per_s": FP32_LANE_OPS_PER_S}}


# ---------------------------------------------------------------------------- helpers
def peaks() -> dict:
    if PEAKS_PATH.exists():
        d = json.loads(PEAKS_PATH.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """NVML sampling of SM clock + clocks-event reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz = sorted(s[0] for s in self.samples)
        bits = 0
        for _, r in self.samples:
            bits |= r
        reasons = [name for bit, name in self.REASONS.items() if bits & bit and name != "gpu_idle"]
        return {"sm_mhz": mhz[len(mhz) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def emit(obj: dict) -> None:
    print(json.dumps(obj), flush=True)


# ---------------------------------------------------------------------------- config 9 inputs
TOOL_GRID = (360.0, 4.0)  # the measured grid of the encode-tool input: 360, 364, ..., 800 nm


def tool_raw_weights(k: int) -> tuple:
    """Raw codec weights (CodecWeights, softplus beta = 10) for the encode tool, k x 81 / 81 x k."""
    from paper_2602_18741_b200 import synth

    re_ = (synth.uniform_np(SEED, "tool.raw_enc", 0, k * N_SPEC) - 0.5) / np.sqrt(N_SPEC)
    rd = (synth.uniform_np(SEED, "tool.raw_dec", 0, N_SPEC * k) - 0.5) / np.sqrt(N_SPEC)
    return np.ascontiguousarray(re_, np.float64), np.ascontiguousarray(rd, np.float64)


def tool_spectra_text_np(rows: int, m: int) -> bytes:
    """A spectra CSV (ids s<r>, %.9g) of `rows` seeded curves on TOOL_GRID, formatted on the host."""
    from paper_2602_18741_b200 import synth

    lo, step = TOOL_GRID
    v = synth.uniform_np(SEED, "tool.spectra", 0, rows * m).reshape(rows, m).astype(np.float64)
    head = "id," + ",".join("%.9g" % (lo + step * i) for i in range(m))
    lines = [head] + ["s%d," % r + ",".join("%.9g" % x for x in row) for r, row in enumerate(v)]
    return ("\n".join(lines) + "\n").encode()


# ---------------------------------------------------------------------------- CPU reference
def cpu_reference_run(cfg_key: str, budget_s: float, threads: int = 0, rank: int = 0, min_reps: int = 1) -> dict:
    """Time the reference's CPU implementation (oracle/_ref) on its per-step workload
    (the full frame for configs 2 / 3, a bounded sample otherwise) for >= budget_s and
    >= min_reps steps."""
    case = cpu_reference_case(cfg_key, threads, rank)
    return time_cpu_case(case, budget_s, min_reps)


def time_cpu_case(case: dict, budget_s: float, min_reps: int = 1, warmup: int = 1) -> dict:
    run = case["run"]
    for _ in range(warmup):
        run()
    t0 = time.perf_counter()
    reps = 0
    while True:
        run()
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s and reps >= min_reps:
            break
    value = case["P"] * reps / el / 1e6
    return {"value": value, "unit": case["unit"], "cores": case["cores"], "kind": "reference",
            "sample": case["sample"], "seconds": round(el, 3), "units_per_rep": case["P"], "reps": reps,
            "step_s": el / reps, "cpu": _cpu_model()}


def cpu_reference_case(cfg_key: str, threads: int = 0, rank: int = 0) -> dict:
    """The reference's CPU implementation of one step of config `cfg_key` (oracle/_ref: the
    reference core compiled from its sources, plus the G-buffer restatement SURVEY §8c R1)."""
    import oracle
    from paper_2602_18741_b200 import synth

    ref = oracle.reference(81)
    if ref is None:
        raise RuntimeError("oracle/_ref not built (python __graft_entry__.py build)")
    cfg = CONFIGS[cfg_key]
    nthreads = threads if threads > 0 else ref.ref_thread_count()
    k = cfg["k"]
    E, D = synth.codec_weights(SEED, k, N_SPEC)

    if cfg_key in ("2", "3"):
        L = cfg["L"]
        W, H = cfg["W"], cfg["H"]
        pal = synth.palette(SEED, 256, N_SPEC)
        lts = synth.lights(SEED, L, N_SPEC)
        pc = np.zeros((256, k), np.float32)
        lc = np.zeros((L, k), np.float32)
        ref.ref_asset_codes(E, k, pal, 256, pc)
        ref.ref_asset_codes(E, k, lts, L, lc)
        P = W * H  # the whole frame, as the GPU arm's step
        idx, cosv = synth.gbuffer_np(SEED, rank * H * W, P, L, 256)
        cosv = np.ascontiguousarray(cosv)
        outs = {"xyz": np.zeros((P, 3), np.float32), "rgb": np.zeros((P, 3), np.float32)}
        spec = np.zeros((P, N_SPEC), np.float32) if cfg_key == "3" else None

        def run():
            ref.ref_shade_latent(E, D, k, pc, lc, L, idx, cosv, P, None, spec,
                                 None if cfg_key == "3" else outs["xyz"], outs["rgb"], nthreads)

        sample = (f"the full {W}x{H} frame per step (R1 latent shade + decode_image + image_to_linear_rgb, "
                  f"{nthreads} threads)")
    elif cfg_key == "1":
        P = 1 << 14
        S = synth.gm_spectra_ctr(SEED, "codec.spectra", 0, 2048, N_SPEC)
        S = np.ascontiguousarray(np.tile(S, (P // 2048, 1)))
        bufs = [np.zeros((P, d), np.float32) for d in (k, N_SPEC, 3, 3)]

        def run():
            ref.ref_codec_roundtrip(E, D, k, S, P, *bufs, nthreads)

        sample = f"{P} spectra (encode/decode_image/image_to_linear_rgb)"
    elif cfg_key == "4":
        spp = cfg["spp"]
        P = 2048 * 2
        pal = synth.palette(SEED, 256, N_SPEC)
        ill = synth.lights(SEED, 16, N_SPEC, purpose="scene.illuminants")
        pc = np.zeros((256, k), np.float32)
        ic = np.zeros((16, k), np.float32)
        ref.ref_asset_codes(E, k, pal, 256, pc)
        ref.ref_asset_codes(E, k, ill, 16, ic)
        pidx, iidx, tw = (np.ascontiguousarray(a) for a in synth.chain_np(SEED, 0, P, spp, 256, 16))
        X, R = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)

        def run():
            ref.ref_multibounce_latent(E, D, k, pc, ic, pidx, iidx, tw, P, spp, 4, None, X, R, nthreads)

        sample = f"{P} px x {spp} spp (2 rows)"
    elif cfg_key == "5a":
        from paper_2602_18741_b200.synth import mlp_weights

        w = mlp_weights(SEED, 6, 64)
        P = 4096 * 8
        rgb = np.ascontiguousarray(synth.uniform_np(SEED, "mlp.input", 0, P * 3).reshape(P, 3))
        out = np.zeros((P, 6), np.float32)

        def run():
            ref.ref_mlp_forward(rgb, P, 64, 6, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"], w["b3"], out, nthreads)

        sample = f"{P} texels (8 rows)"
    elif cfg_key == "8":
        import ctypes as C
        import tempfile

        rows = 1 << 15
        Zs = np.exp(synth.uniform_np(SEED, "csv.codes", 0, rows * k) * 20.0 - 10.0).astype(np.float32)
        tmp = tempfile.mkdtemp()
        path = (tmp + "/codes.csv").encode()
        buf_codes = np.zeros(rows * k, np.float64)
        ids = C.create_string_buffer(rows * 24 + 4096)
        r_rows, r_k = C.c_int64(), C.c_int()
        P = rows * k
        nthreads = 1

        def run():
            ref.ref_write_codes_csv(path, Zs, rows, k, 0)
            ref.ref_read_codes_csv(path, C.byref(r_rows), C.byref(r_k), buf_codes, buf_codes.size, ids, len(ids))

        sample = f"{rows} rows x k={k}: the reference's write_codes_csv + read_codes_csv (single-threaded, /tmp file)"
    elif cfg_key == "10":
        m = 2048
        raw_e, raw_d = tool_raw_weights(k)
        refl = synth.uniform_np(SEED, "train.refl", 0, m * N_SPEC).astype(np.float64)
        illum = synth.uniform_np(SEED, "train.illum", 0, m * N_SPEC).astype(np.float64) * 2.0
        ge, gd, lo = np.zeros(k * N_SPEC), np.zeros(N_SPEC * k), np.zeros(6)
        lw = np.array([0.5, 0.75, 1.0, 0.5, 0.0])
        P = m
        nthreads = 1

        def run():
            ref.ref_codec_gradients(k, 10.0, raw_e, raw_d, refl, illum, m, lw, ge.ctypes.data, gd.ctypes.data, lo)

        sample = f"{m} pairs: the reference's gradients() + compute_losses() (single-threaded)"
    elif cfg_key == "9":
        import ctypes as C
        import tempfile

        rows, m = 2048, cfg["m"]
        raw_e, raw_d = tool_raw_weights(k)
        text = tool_spectra_text_np(rows, m)
        tmp = tempfile.mkdtemp()
        src, dst = (tmp + "/spectra.csv").encode(), (tmp + "/codes.csv").encode()
        with open(src, "wb") as f:
            f.write(text)
        err = C.create_string_buffer(256)
        P = rows
        nthreads = 1

        def run():
            if ref.ref_run_encode(src, k, 10.0, raw_e, raw_d, dst, err, 256) != 0:
                raise RuntimeError(err.value.decode())

        sample = (f"{rows} curves x {m} samples: the reference's encode tool steps (read_spectra_csv, resample, "
                  "encode, write_codes_csv; single-threaded, /tmp files)")
    elif cfg_key == "7":
        import ctypes as C

        from paper_2602_18741_b200 import api as _api

        scene = synth.cornell_scene(N_SPEC, block=True)
        sc, keep = _api.scene_struct(scene, N_SPEC)
        W = H = 64
        spp = 16
        job = _api.HcRenderJob(1, W, H, spp, cfg["depth"], SEED + rank)
        img = np.zeros(W * H * k, np.float32)
        ev = C.c_uint64()
        P = W * H * spp

        def run():
            ref.ref_render(C.addressof(sc), C.addressof(job), k, E, D, 0, img, None, C.byref(ev))

        sample = f"{W}x{H} px x {spp} spp latent render of the reference (render_compiled's thread pool)"
    elif cfg_key == "6":
        # the reference's own scene_color_report + tonemap_srgb8 (single-threaded as written)
        L, W = cfg["L"], cfg["W"]
        pal = synth.palette(SEED, 256, N_SPEC)
        lts = synth.lights(SEED, L, N_SPEC)
        pc = np.zeros((256, k), np.float32)
        lc = np.zeros((L, k), np.float32)
        ref.ref_asset_codes(E, k, pal, 256, pc)
        ref.ref_asset_codes(E, k, lts, L, lc)
        P = 64 * W
        idx, cosv = synth.gbuffer_np(SEED, rank * cfg["H"] * W, P, L, 256)
        cosv = np.ascontiguousarray(cosv)
        gt, test = np.zeros((P, 3), np.float32), np.zeros((P, 3), np.float32)
        ref.ref_shade_spectral(pal, lts, L, idx, cosv, P, None, None, gt, nthreads)
        ref.ref_shade_latent(E, D, k, pc, lc, L, idx, cosv, P, None, None, None, test, nthreads)
        rep, u8 = np.zeros(4), np.zeros(P * 3, np.uint8)
        nthreads = 1

        def run():
            ref.ref_scene_color_report(gt, 3, test, 3, P, rep)
            ref.ref_tonemap_srgb8(test, P, rep[3], u8)

        sample = f"{P} px (64 rows): scene_color_report + tonemap_srgb8 of the reference (single-threaded)"
    else:  # 5b
        P = 1 << 15
        A = synth.gm_spectra_ctr(SEED, "loss.a", 0, 1024, N_SPEC)
        B = synth.gm_spectra_ctr(SEED, "loss.b", 0, 1024, N_SPEC)
        A = np.ascontiguousarray(np.tile(A, (P // 1024, 1)))
        B = np.ascontiguousarray(np.tile(B, (P // 1024, 1)))

        def run():
            ref.ref_hadamard_loss(E, D, k, A, B, P, nthreads)

        sample = f"{P} pairs"

    return {"run": run, "P": P, "sample": sample, "cores": nthreads, "unit": cfg["unit"]}


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_dict(key: str) -> dict:
    """The workload description both arms print (identical, so the driver can match them)."""
    cfg = CONFIGS[key]
    d = {"workload": cfg["name"], "config_id": key}
    for f in ("W", "H", "units", "k", "L", "spp", "cmf"):
        if f in cfg:
            d[f] = cfg[f]
    return d


def metric_name(key: str) -> str:
    return METRIC if key == "2" else f"{CONFIGS[key]['unit']} config {key}"


def run_reference_arm(args) -> int:
    """The reference's own CPU implementation of the step (oracle/_ref, all host threads):
    W untimed warm-up steps, then exactly K timed steps, each the same workload as one
    GPU-arm step (the full frame for the default config).  Rank 0 only."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    case = cpu_reference_case(args.config)
    for _ in range(args.warmup):
        case["run"]()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        case["run"]()
    el = time.perf_counter() - t0
    value = case["P"] * args.steps / el / 1e6
    line = {"metric": metric_name(args.config), "value": value, "unit": cfg["unit"], "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": cfg.get("dtype", "bf16" if args.config == "5a" else "f32"), "data": "synthetic",
            "config": config_dict(args.config), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": cfg["unit"], "cores": case["cores"], "kind": "reference",
                             "sample": case["sample"], "cpu": _cpu_model()},
            "e2e": {"value": value, "unit": cfg["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# ---------------------------------------------------------------------------- GPU arm
class Workload:
    """Builds the per-rank inputs of one config and a step() closure over buffer set i."""

    def __init__(self, api, ctx, cfg_key: str, rank: int, naive: bool = False, world: int = 1,
                 strong: bool = False):
        import torch
        from paper_2602_18741_b200 import synth

        self.cfg = cfg = CONFIGS[cfg_key]
        self.key = cfg_key
        k = cfg["k"]
        E, D = synth.codec_weights(SEED, k, N_SPEC)
        # config 1 projects with the analytic multi-lobe CIE 1931 fit BASELINE.json names; the
        # other configs with the reference's tabulated CmfTable rows
        cmf = cmf_analytic(N_SPEC) if cfg.get("cmf") == "analytic" else None
        self.codec = codec = api.Codec(ctx, E, D, cmf=cmf)
        self.sets = []
        self.extra = {}  # workload facts added to the JSON line's config
        R = cfg["rot"]
        from paper_2602_18741_b200.sharding import row_band

        def span(total_rows: int, width: int) -> tuple[int, int]:
            # weak: rank r owns rows [r*H, (r+1)*H) of an N-frame-tall image;
            # strong: one frame split into row bands (sharding.row_band).
            if strong:
                b = row_band(rank, world, total_rows, width)
                return b.first_pixel, b.pixels
            return rank * total_rows * width, total_rows * width
        if cfg_key in ("2", "3"):
            W, H, L = cfg["W"], cfg["H"], cfg["L"]
            first, P = span(H, W)
            pal = synth.palette(SEED, 256, N_SPEC)
            lts = synth.lights(SEED, L, N_SPEC)
            self.pal_d = torch.from_numpy(pal).cuda()
            self.lts = lts
            self.pal_codes = codec.encode(self.pal_d)  # compile_scene: assets encoded once
            self.light_codes = codec.encode(torch.from_numpy(lts).cuda()).cpu().numpy()
            spec = cfg_key == "3"
            for r in range(R):
                idx, cosv = api.synth_gbuffer(ctx, SEED + r, first, P, L, 256)
                outs = {"xyz": None if spec else ctx.empty(P, 3), "rgb": ctx.empty(P, 3),
                        "spectra": ctx.empty(P, N_SPEC) if spec else None, "latent": None}
                self.sets.append((idx, cosv, outs))
            self.units = P

            def step(i):
                idx, cosv, outs = self.sets[i % R]
                if naive:
                    codec.shade_spectral(self.pal_d, self.lts, idx, cosv, out=outs)
                else:
                    codec.shade_latent(self.pal_codes, self.light_codes, idx, cosv, out=outs)
            self.step = step
        elif cfg_key == "6":
            W, H, L = cfg["W"], cfg["H"], cfg["L"]
            first, P = span(H, W)
            pal = synth.palette(SEED, 256, N_SPEC)
            lts = synth.lights(SEED, L, N_SPEC)
            pal_d = torch.from_numpy(pal).cuda()
            pal_codes = codec.encode(pal_d)
            light_codes = codec.encode(torch.from_numpy(lts).cuda()).cpu().numpy()
            for r in range(R):  # ground truth = naive n = 81 render, test = latent render of the same frame
                idx, cosv = api.synth_gbuffer(ctx, SEED + r, first, P, L, 256)
                gt = codec.shade_spectral(pal_d, lts, idx, cosv)["rgb"]
                test = codec.shade_latent(pal_codes, light_codes, idx, cosv, xyz=False)["rgb"]
                self.sets.append((gt, test, ctx.empty(4, dtype=torch.float64),
                                  torch.empty(P, 3, dtype=torch.uint8, device="cuda")))
                del idx, cosv
            self.units = P

            def step(i):
                gt, test, out, prev = self.sets[i % R]
                api.scene_color_report_dev(codec, gt, test, out=out, preview=prev)
            self.step = step
        elif cfg_key == "8":
            rows, k = cfg["rows"], cfg["k"]
            Z = api.synth_uniform(ctx, SEED + rank, "csv.codes", 0, rows * k).reshape(rows, k)
            Z = torch.exp(Z * 20.0 - 10.0)  # codes across many decades
            self.units = rows * k
            self.sets.append({"rgb": None})
            length = C_int64()
            api._check(api._lib.lib().hc_codes_csv_write(ctx.h, Z.data_ptr(), rows, k, 0, None, 0,
                                                        api.C.byref(length)))
            self.text = torch.empty(length.value, dtype=torch.uint8, device="cuda")
            self.extra = {"text_bytes": length.value}
            self.codes = torch.empty(rows, k, dtype=torch.float64, device="cuda")
            self.ids = torch.empty(rows, 2, dtype=torch.int64, device="cuda")

            def step(i):
                lib = api._lib.lib()
                ln, kk, rr = C_int64(), api.C.c_int(), C_int64()
                ctx.bind_stream()
                api._check(lib.hc_codes_csv_write(ctx.h, Z.data_ptr(), rows, k, 0, self.text.data_ptr(),
                                                  self.text.numel(), api.C.byref(ln)))
                api._check(lib.hc_codes_csv_read(ctx.h, self.text.data_ptr(), ln.value, api.C.byref(kk),
                                                 api.C.byref(rr), self.codes.data_ptr(), self.ids.data_ptr(), rows))
            self.step = step
        elif cfg_key == "10":
            m, k = cfg["m"], cfg["k"]
            self.raw_e, self.raw_d = tool_raw_weights(k)
            self.raw_e = self.raw_e.reshape(k, N_SPEC)
            self.raw_d = self.raw_d.reshape(N_SPEC, k)
            base = api.synth_uniform(ctx, SEED + rank, "train.refl", 0, m * N_SPEC).reshape(m, N_SPEC)
            self.refl = base.double().contiguous()
            self.illum = (api.synth_uniform(ctx, SEED + rank, "train.illum", 0, m * N_SPEC).reshape(m, N_SPEC)
                          .double() * 2.0).contiguous()
            self.units = m
            self.sets.append({"rgb": None})

            def step(i):
                api.codec_train_grad(ctx, self.raw_e, self.raw_d, 10.0, self.refl, self.illum)
            self.step = step
        elif cfg_key == "9":
            rows, m, k = cfg["rows"], cfg["m"], cfg["k"]
            lib = api._lib.lib()
            raw_e, raw_d = tool_raw_weights(k)
            self.codec = api.Codec.from_raw(ctx, raw_e.reshape(k, N_SPEC), raw_d.reshape(N_SPEC, k), beta=10.0)
            vals = api.synth_uniform(ctx, SEED + rank, "tool.spectra", 0, rows * m).reshape(rows, m).double()
            lo, step = TOOL_GRID
            self.src_wl = np.array([lo + step * i for i in range(m)], np.float64)
            ln = C_int64()  # setup: the input file (ids s0, s1, ...), written by the device writer
            api._check(lib.hc_spectra_csv_write(ctx.h, vals.data_ptr(), 1, rows, m, api._np_ptr(self.src_wl), 1, None,
                                                None, b"s", 0, None, 0, api.C.byref(ln)))
            self.text = torch.empty(ln.value, dtype=torch.uint8, device="cuda")
            api._check(lib.hc_spectra_csv_write(ctx.h, vals.data_ptr(), 1, rows, m, api._np_ptr(self.src_wl), 1, None,
                                                None, b"s", 0, self.text.data_ptr(), ln.value, api.C.byref(ln)))
            self.vals = torch.empty(rows, m, dtype=torch.float64, device="cuda")
            self.spans = torch.empty(rows, 2, dtype=torch.int64, device="cuda")
            self.codes = torch.empty(rows, k, dtype=torch.float64, device="cuda")
            self.wl = np.zeros(m, np.float64)
            self.units = rows
            self.sets.append({"rgb": None})
            gl, gs = api.grid(N_SPEC)
            self.out = None

            def step(i):
                hid, mm, rr, olen = api.C.c_int(), api.C.c_int(), C_int64(), C_int64()
                ctx.bind_stream()
                api._check(lib.hc_spectra_csv_read(ctx.h, self.text.data_ptr(), self.text.numel(), api.C.byref(hid),
                                                   api._np_ptr(self.wl), m, api.C.byref(mm), api.C.byref(rr),
                                                   self.vals.data_ptr(), self.spans.data_ptr(), rows))
                api._check(lib.hc_encode_resampled_f64(self.codec.h, api._np_ptr(self.wl), m, self.vals.data_ptr(),
                                                       rows, gl, gs, 1, self.codes.data_ptr()))
                if self.out is None:
                    api._check(lib.hc_codes_csv_write_ids(ctx.h, self.codes.data_ptr(), 1, rows, k,
                                                          self.text.data_ptr(), self.spans.data_ptr(), None, 0, None,
                                                          0, api.C.byref(olen)))
                    self.out = torch.empty(olen.value, dtype=torch.uint8, device="cuda")
                api._check(lib.hc_codes_csv_write_ids(ctx.h, self.codes.data_ptr(), 1, rows, k, self.text.data_ptr(),
                                                      self.spans.data_ptr(), None, 0, self.out.data_ptr(),
                                                      self.out.numel(), api.C.byref(olen)))
            self.extra = {"text_bytes_in": int(self.text.numel())}
            self.step = step
        elif cfg_key == "7":
            W, H, spp, depth = cfg["W"], cfg["H"], cfg["spp"], cfg["depth"]
            scene = synth.cornell_scene(N_SPEC, block=True)
            mode = "spectral" if naive else "latent"
            self.units = W * H * spp
            self.sets.append({"rgb": None})

            def step(i):  # weak scaling: every rank renders its own frame (seed per rank)
                api.render(codec, scene, mode, W, H, spp, depth, seed=SEED + rank)
            self.step = step
        elif cfg_key == "1":
            first, P = span(cfg["units"], 1)
            for r in range(R):
                S = api.synth_gm_spectra(ctx, SEED + r, "codec.spectra", first, P, N_SPEC)
                outs = {"codes": ctx.empty(P, k), "spectra": ctx.empty(P, N_SPEC), "xyz": ctx.empty(P, 3),
                        "rgb": ctx.empty(P, 3)}
                self.sets.append((S, outs))
            self.units = P

            def step(i):
                S, outs = self.sets[i % R]
                codec.roundtrip(S, out=outs)
            self.step = step
        elif cfg_key == "4":
            W, H, spp = cfg["W"], cfg["H"], cfg["spp"]
            first, P = span(H, W)
            pal = synth.palette(SEED, 256, N_SPEC)
            ill = synth.lights(SEED, 16, N_SPEC, purpose="scene.illuminants")
            self.pal_d = torch.from_numpy(pal).cuda()
            self.ill_d = torch.from_numpy(ill).cuda()
            self.pal_codes = codec.encode(self.pal_d)
            self.ill_codes = codec.encode(self.ill_d)
            for r in range(R):
                pidx, iidx, tw = api.synth_chain(ctx, SEED + r, first, P, spp, 256, 16)
                outs = {"xyz": ctx.empty(P, 3), "rgb": ctx.empty(P, 3), "latent": None}
                self.sets.append((pidx, iidx, tw, outs))
            self.units = P

            def step(i):
                pidx, iidx, tw, outs = self.sets[i % R]
                if naive:
                    codec.multibounce_spectral(self.pal_d, self.ill_d, pidx, iidx, tw, out=outs)
                else:
                    codec.multibounce_latent(self.pal_codes, self.ill_codes, pidx, iidx, tw, out=outs)
            self.step = step
        elif cfg_key == "5a":
            W, H = cfg["W"], cfg["H"]
            first, P = span(H, W)
            w = synth.mlp_weights(SEED, 6, 64)
            self.mlp = api.CodeMLP(ctx, w)
            for r in range(R):
                rgb = api.synth_uniform(ctx, SEED + r, "mlp.input", first * 3, P * 3).reshape(P, 3)
                self.sets.append((rgb, ctx.empty(P, 6)))
            self.units = P

            def step(i):
                rgb, out = self.sets[i % R]
                self.mlp.forward(rgb, out=out)
            self.step = step
        else:  # 5b
            first, P = span(cfg["units"], 1)
            A = api.synth_gm_spectra(ctx, SEED, "loss.a", first, P, N_SPEC)
            B = api.synth_gm_spectra(ctx, SEED, "loss.b", first, P, N_SPEC)
            self.sum = ctx.empty(1, dtype=torch.float64)
            self.sets.append((A, B))
            self.units = P

            def step(i):
                codec.hadamard_loss(A, B, out=self.sum)
            self.step = step
        self.R = R


class StepReplayer:
    """Replays exactly n steps of a workload from CUDA graphs, so any --steps is honoured
    exactly: up to MAX_NODES steps are one graph of exactly n steps (the buffer rotation runs
    through it, and every launch overlaps its predecessor's tail by programmatic dependent
    launch -- at 22 us per step the gap between two graph launches is visible); longer runs
    replay a chunk graph (a whole number of buffer rotations) plus one graph of the remainder.
    Configs whose step cannot be captured (host-side setup / synchronisation inside the
    call) run the steps as plain library calls."""

    MAX_NODES = 512

    def __init__(self, torch, wl, warmup: int, stream, max_steps: int):
        self.torch, self.wl, self.stream = torch, wl, stream
        from paper_2602_18741_b200 import api as _api

        self.api = _api
        self.graph = wl.cfg.get("graph", True)
        R = wl.R
        ctx = wl.codec.ctx
        with torch.cuda.stream(stream):
            for i in range(max(warmup, R if self.graph else 1)):
                wl.step(i)
            torch.cuda.synchronize()
            l0 = ctx.launches
            wl.step(0)
            torch.cuda.synchronize()
            self.per_step = ctx.launches - l0
        self.graphs = {}
        self.chunk = max(R, self.MAX_NODES // max(1, self.per_step) // R * R)  # steps per chunk graph
        if self.graph:
            self.prepare(R)

    def _capture(self, n: int):
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            with torch.cuda.graph(g, stream=self.stream):
                for i in range(n):
                    self.wl.step(i)
            g.replay()
        torch.cuda.synchronize()
        return g

    def _parts(self, n: int):
        """(graph size, replays) pairs that add up to exactly n steps."""
        if n <= self.chunk:
            return [(n, 1)] if n else []
        parts = [(self.chunk, n // self.chunk)]
        if n % self.chunk:
            parts.append((n % self.chunk, 1))
        return parts

    def prepare(self, n: int) -> None:
        """Capture the graphs n steps need (outside any timed region)."""
        if not self.graph:
            return
        for size, _ in self._parts(n):
            if size not in self.graphs:
                self.graphs[size] = self._capture(size)

    def run(self, n: int) -> None:
        """Issue exactly n steps on the stream (no synchronisation)."""
        if not self.graph:
            for i in range(n):
                self.wl.step(i)
            return
        self.prepare(n)  # (timed callers prepare beforehand; a no-op then)
        for size, reps in self._parts(n):
            for _ in range(reps):
                self.graphs[size].replay()


def C_int64():
    import ctypes

    return ctypes.c_int64()


def _max_over_ranks(torch, dist, world: int, v: float) -> float:
    if world == 1:
        return v
    t = torch.tensor([v], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_steps(torch, dist, world: int, rep: StepReplayer, steps: int, stream, clocks=None) -> tuple[float, float]:
    """Exactly `steps` steps between two CUDA events on the launching stream, bracketed by
    a barrier + synchronize on both sides; (ms max over ranks, host wall seconds)."""
    rep.prepare(steps)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cm = clocks if clocks is not None else _NullCtx()
    with cm:
        w0 = time.perf_counter()
        with torch.cuda.stream(stream):
            if rep.graph:
                # A ~200 us spin kernel ahead of the start event: the device is still busy while the
                # host enqueues the graph, so the event interval starts when the first step can start
                # instead of containing the host's graph-launch latency (visible at --steps 20).
                rep.api.spin(rep.wl.codec.ctx, 400_000)
            e0.record(stream)
            rep.run(steps)
            e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    barrier()
    return _max_over_ranks(torch, dist, world, e0.elapsed_time(e1)), wall


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def roofline_record(cfg: dict, units: int, kernel_us: float) -> dict:
    pk = peaks()
    if "flops_per_unit" in cfg:
        achieved = units * cfg["flops_per_unit"] / (kernel_us * 1e-6) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16_tflops"], "traffic": None,
                "peak_source": f"{pk['source']} bf16_tflops (burst)", "flops_per_unit": cfg["flops_per_unit"],
                "units_per_launch": units, "kernel_us": kernel_us}
    achieved = units * cfg["bytes_per_unit"] / (kernel_us * 1e-6) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": None, "peak_source": f"{pk['source']} hbm_gbs",
            "bytes_per_unit": cfg["bytes_per_unit"], "units_per_launch": units, "kernel_us": kernel_us}


def _traffic(key: str):
    """ncu DRAM bytes per launch of the dominant kernel (profiles/traffic_config<key>.json:
    dram__bytes_read.sum + dram__bytes_write.sum, steady-state window of back-to-back launches)."""
    path = ROOT / "profiles" / f"traffic_config{key}.json"
    if path.exists():
        try:
            d = json.loads(path.read_text())
            return d.get("bytes_per_launch"), d
        except Exception:  # noqa: BLE001
            pass
    return None, None


def parity_gbuffer(wl, rows_stride: int = 1) -> dict:
    """Set 0 of a config 2 / 3 workload against the reference (oracle/_ref, R1 restatement over
    the reference's decode_image / image_to_linear_rgb) on the same inputs: every
    `rows_stride`-th row of the frame.  Tolerance (north_star): 1e-5 relative, denominator
    max(|ref|, ||ref_row||_inf)."""
    import oracle

    ref = oracle.reference(81)
    cfg = wl.cfg
    k, L, W = cfg["k"], cfg["L"], cfg["W"]
    idx, cosv, outs = wl.sets[0]
    P = wl.units
    rows = np.arange(0, P // W, rows_stride)
    sel = (rows[:, None] * W + np.arange(W)[None, :]).reshape(-1)
    h_idx = idx.cpu().numpy().view(np.uint32)[sel].copy()
    h_cos = np.ascontiguousarray(cosv.cpu().numpy()[sel])
    m = sel.size
    E, D = wl.codec.E, wl.codec.D
    spec = cfg["W"] == 3840
    r_spec = np.zeros((m, N_SPEC), np.float32) if spec else None
    r_xyz = None if spec else np.zeros((m, 3), np.float32)
    r_rgb = np.zeros((m, 3), np.float32)
    ref.ref_shade_latent(E, D, k, wl.pal_codes.cpu().numpy(), wl.light_codes, L, h_idx, h_cos, m, None, r_spec,
                         r_xyz, r_rgb, 0)
    res = {"rows": f"every {rows_stride}th row" if rows_stride > 1 else "full frame", "pixels": int(m),
           "tol": 1e-5, "checker": "oracle/_ref (the reference compiled from its sources)"}
    worst = 0.0
    for name, want in (("spectra", r_spec), ("xyz", r_xyz), ("rgb", r_rgb)):
        if want is None:
            continue
        got = outs[name].cpu().numpy()[sel]
        rel, mabs = rel_err_rows(got, want), float(np.max(np.abs(got.astype(np.float64) - want)))
        res[name] = {"max_rel": rel, "max_abs": mabs}
        worst = max(worst, rel)
    res["pass"] = bool(worst <= 1e-5)
    return res


def parity_naive_gbuffer(wn, rows_stride: int = 16) -> dict:
    """The naive n = 81 path (config 2 / 3 ground truth) on set 0 against the reference's
    spectral shading (oracle/_ref, R1 at C = n) on every `rows_stride`-th row."""
    import oracle

    ref = oracle.reference(81)
    cfg = wn.cfg
    L, W = cfg["L"], cfg["W"]
    idx, cosv, outs = wn.sets[0]
    P = wn.units
    rows = np.arange(0, P // W, rows_stride)
    sel = (rows[:, None] * W + np.arange(W)[None, :]).reshape(-1)
    h_idx = idx.cpu().numpy().view(np.uint32)[sel].copy()
    h_cos = np.ascontiguousarray(cosv.cpu().numpy()[sel])
    m = sel.size
    spec = outs.get("spectra") is not None
    r_spec = np.zeros((m, N_SPEC), np.float32) if spec else None
    r_xyz = np.zeros((m, 3), np.float32)
    r_rgb = np.zeros((m, 3), np.float32)
    ref.ref_shade_spectral(np.ascontiguousarray(wn.pal_d.cpu().numpy()), np.ascontiguousarray(wn.lts, np.float32), L,
                           h_idx, h_cos, m, r_spec, r_xyz, r_rgb, 0)
    res = {}
    for name, want in (("naive spectra", r_spec), ("naive xyz", r_xyz), ("naive rgb", r_rgb)):
        key = name.split()[1]
        if want is None or outs.get(key) is None:
            continue
        got = outs[key].cpu().numpy()[sel]
        res[name] = {"max_rel": rel_err_rows(got, want), "max_abs": float(np.max(np.abs(got.astype(np.float64) - want))),
                     "rows": f"every {rows_stride}th row", "pixels": int(m)}
    return res


def rel_err_rows(got, ref) -> float:
    """max |got - ref| / max(|ref|, ||ref_row||_inf), chunked for large arrays."""
    worst = 0.0
    n = ref.shape[0]
    step = max(1, (1 << 24) // max(1, ref.shape[1] if ref.ndim > 1 else 1))
    for a in range(0, n, step):
        g = np.asarray(got[a:a + step], np.float64)
        r = np.asarray(ref[a:a + step], np.float64)
        row = np.max(np.abs(r), axis=-1, keepdims=True) if r.ndim > 1 else np.abs(r)
        den = np.maximum(np.maximum(np.abs(r), row), 1e-30)
        if r.size:
            worst = max(worst, float(np.max(np.abs(g - r) / den)))
    return worst


def nccl_record(world: int, rank: int) -> dict | None:
    """What NCCL reported at communicator init (NCCL_DEBUG=INFO, subsystem INIT, logged to a
    per-process file): the version and the rank count of the communicator it built."""
    import re

    import torch

    path = os.environ.get("NCCL_DEBUG_FILE", "")
    rec = {"backend": "nccl", "world": world}
    try:
        v = torch.cuda.nccl.version()
        rec["version"] = ".".join(map(str, v)) if isinstance(v, tuple) else str(v)
    except Exception:  # noqa: BLE001
        pass
    if path:
        f = Path(path.replace("%h", os.uname().nodename).replace("%p", str(os.getpid())))
        if f.exists():
            txt = f.read_text(errors="replace")
            n = re.findall(r"nranks\s*[= ]\s*(\d+)", txt, re.I)
            if n:
                rec["comm_nranks"] = int(n[-1])
            rec["init_lines"] = len([ln for ln in txt.splitlines() if "Init" in ln or "init" in ln])
    return rec


def run_ours(args) -> int:
    import torch
    import torch.distributed as dist
    from paper_2602_18741_b200 import api

    rank, world, local = dist_env()
    if world > 1:
        # NCCL's own account of the communicator (version, nranks) goes to a per-process
        # file, read back into the JSON line (nccl_record); stdout stays one JSON line.
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/hc_bench_nccl.%h.%p.log")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()  # the communicator exists (and is logged) before the timed region
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cfg = CONFIGS[args.config]
    stream = torch.cuda.Stream()
    strong = args.scaling == "strong"
    with torch.cuda.stream(stream):
        ctx = api.Context(dev)
        wl = Workload(api, ctx, args.config, rank, world=world, strong=strong)
    torch.cuda.synchronize()
    steps = args.steps

    if args.plain:
        # Profiling mode (ncu): plain stream launches, no graph, no extras, no JSON contract.
        with torch.cuda.stream(stream):
            for i in range(args.warmup + args.steps):
                wl.step(i)
        torch.cuda.synchronize()
        if args.naive_plain:
            with torch.cuda.stream(stream):
                wn = Workload(api, ctx, args.config, rank, naive=True, world=world, strong=strong)
                for i in range(args.steps):
                    wn.step(i)
            torch.cuda.synchronize()
        print(json.dumps({"plain": True, "config": args.config, "steps": args.steps, "launches": ctx.launches}))
        return 0

    rep = StepReplayer(torch, wl, args.warmup, stream, steps)
    rep.prepare(steps)
    with torch.cuda.stream(stream):  # the W warm-up steps again through the replay path
        rep.run(min(args.warmup, max(steps, 1)))
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps, CUDA events on the launching stream, max over ranks
    clocks = ClockSampler(dev)
    ms, t_wall = time_steps(torch, dist, world, rep, steps, stream, clocks)
    launches_timed = rep.per_step * steps  # graph replays do not pass through the host counter
    ms_per_step = ms / steps
    # per-step distribution after the timed region (does not perturb it): groups of R steps
    R = wl.R
    nrep = 8
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(nrep + 1)]
    with torch.cuda.stream(stream):
        evs[0].record(stream)
        for j in range(nrep):
            rep.run(R)
            evs[j + 1].record(stream)
    torch.cuda.synchronize()
    per = np.array([evs[j].elapsed_time(evs[j + 1]) / R for j in range(nrep)])
    dist_ms = {"p10": float(np.percentile(per, 10)), "p50": float(np.median(per)),
               "p90": float(np.percentile(per, 90)), "groups": nrep, "steps_per_group": R}
    value = wl.units * world * steps / (ms / 1e3) / 1e6

    kernel_us = ms_per_step * 1e3 / max(1, rep.per_step) if rep.per_step <= 1 else ms_per_step * 1e3
    roof = roofline_record(cfg, wl.units, kernel_us)
    roof["traffic"], tr = _traffic(args.config)
    if tr:
        roof["traffic_note"] = tr.get("method")

    extra = {}
    # ---- naive n = 81 comparison on the same inputs
    if args.config in ("2", "3", "4", "7") and not args.no_naive:
        with torch.cuda.stream(stream):
            wn = Workload(api, ctx, args.config, rank, naive=True, world=world, strong=strong)
        nsteps = steps if args.config not in ("4", "7") else wn.R
        nrep_ = StepReplayer(torch, wn, 1, stream, nsteps)
        nms, _ = time_steps(torch, dist, world, nrep_, nsteps, stream)
        extra["naive_n81"] = {"value": wn.units * world * nsteps / (nms / 1e3) / 1e6, "unit": cfg["unit"],
                              "ms_per_step": nms / nsteps, "steps": nsteps}
        nb = NAIVE_BOUND.get(args.config)
        if nb:
            nb_ms = wn.units * nb["lane_ops_per_unit"] / nb["lane_ops_per_s"] * 1e3
            extra["naive_n81"]["roofline"] = {
                "bound": "fp32 issue", "lane_ops_per_unit": nb["lane_ops_per_unit"],
                "ideal_ms_per_step": nb_ms, "frac": nb_ms / (nms / nsteps),
                "peak": f"148 SMs x 128 fp32 lanes x {nb['lane_ops_per_s'] / 148 / 128 / 1e9:.3f} GHz"}
        extra["speedup_latent_vs_naive"] = (nms / nsteps) / ms_per_step
        del wn, nrep_

    # ---- gather of the sRGB band to rank 0 (compute + gather), N > 1 only
    if world > 1 and args.config in ("2", "3", "4"):
        from paper_2602_18741_b200.sharding import gather_rows, row_band

        H = cfg["H"]
        band = row_band(rank, world, H * world if not strong else H, cfg["W"])
        gsteps = min(steps, 20)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for i in range(gsteps):
                wl.step(i)
                gather_rows(wl.sets[i % R][-1]["rgb"], band, H * world if not strong else H)
            e1.record(stream)
        torch.cuda.synchronize()
        gms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1))
        extra["with_gather"] = {"value": wl.units * world * gsteps / (gms / 1e3) / 1e6, "unit": cfg["unit"],
                                "ms_per_step": gms / gsteps,
                                "gathered": "linear-sRGB row bands -> rank 0 (sharding.gather_rows, NCCL)"}
        if args.gather == "fused" and args.config == "2":
            # Opt-in: no gather step -- every rank's shade kernel stores its sRGB band straight into
            # rank 0's frame through NVLink peer memory (sharding.PeerFrame, CUDA IPC mapping); one
            # frame per buffer-rotation slot.  Not the default: this run has one GPU, so the path is
            # covered by the two-process test on one device only (tests/test_gpu_group.py).
            from paper_2602_18741_b200.sharding import PeerFrame

            rows_all = H * world if not strong else H
            frames = [PeerFrame(band, rows_all, device=dev) for _ in range(R)]

            def fused_step(i):
                idx, cosv, outs = wl.sets[i % R]
                wl.codec.shade_latent(wl.pal_codes, wl.light_codes, idx, cosv,
                                      out={**outs, "rgb": frames[i % R].local})

            with torch.cuda.stream(stream):
                for i in range(R):
                    fused_step(i)
            dist.barrier()
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                e0.record(stream)
                for i in range(gsteps):
                    fused_step(i)
                e1.record(stream)
            torch.cuda.synchronize()
            dist.barrier()
            fms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1))
            ok = True
            if rank == 0:  # rank 0's own band of the last frame equals its device-buffer result
                last = (gsteps - 1) % R
                ok = bool(torch.equal(frames[last].local, wl.sets[last][-1]["rgb"]))
            extra["with_gather_fused"] = {
                "value": wl.units * world * gsteps / (fms / 1e3) / 1e6, "unit": cfg["unit"],
                "ms_per_step": fms / gsteps, "rank0_band_matches": ok,
                "gathered": "each rank's shade kernel stores its sRGB band into rank 0's frame through peer "
                            "memory (sharding.PeerFrame: CUDA IPC mapping, no gather step, plain launches)"}
            for f in frames:
                f.close()

    # ---- config 5b across ranks: the per-rank fp64 partial sums are all-reduced (the one exchange
    # step this path has); compute + all-reduce per step, N > 1 only
    if world > 1 and args.config == "5b":
        from paper_2602_18741_b200.sharding import reduce_loss

        gsteps = min(steps, 20)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for i in range(gsteps):
                wl.step(i)
                reduce_loss(wl.sum)
            e1.record(stream)
        torch.cuda.synchronize()
        ams = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1))
        extra["with_allreduce"] = {"value": wl.units * world * gsteps / (ams / 1e3) / 1e6, "unit": cfg["unit"],
                                   "ms_per_step": ams / gsteps, "total_loss": float(wl.sum.item()),
                                   "reduced": "per-rank fp64 partial sums -> total on every rank "
                                              "(sharding.reduce_loss: one NCCL all-reduce of one double)"}

    # ---- e2e through the host-buffer C-ABI call (config 2)
    e2e = None
    if args.config == "2":
        e2e, ok1, ok2 = e2e_config2(torch, dist, world, wl, stream, steps)
        extra["e2e_matches_device"] = ok1
        extra["e2e_stream_matches_device"] = ok2

    # ---- parity of the timed outputs against the reference (config 2: the full frame)
    if args.config in ("2", "3") and rank == 0 and not args.no_parity:
        try:
            extra["parity"] = parity_gbuffer(wl, 1 if args.config == "2" else 16)
        except Exception as e:  # noqa: BLE001
            extra["parity"] = {"unavailable": str(e)}

    # ---- the k = 9 path (config 3: 4K, 32 lights, full spectra written) beside config 2
    if args.config == "2" and not args.no_k9:
        n_in = wl.units
        del wl, rep
        torch.cuda.empty_cache()
        with torch.cuda.stream(stream):
            w3 = Workload(api, ctx, "3", rank, world=world, strong=strong)
        torch.cuda.synchronize()
        s3 = max(4, min(steps, 20))
        r3 = StepReplayer(torch, w3, 3, stream, s3)
        ms3, _ = time_steps(torch, dist, world, r3, s3, stream)
        c3 = CONFIGS["3"]
        k9 = {"config": config_dict("3"), "value": w3.units * world * s3 / (ms3 / 1e3) / 1e6,
              "unit": c3["unit"], "steps": s3, "ms_per_step": ms3 / s3,
              "roofline": roofline_record(c3, w3.units, ms3 / s3 * 1e3)}
        k9["roofline"]["traffic"], _ = _traffic("3")
        if not args.no_naive:
            with torch.cuda.stream(stream):
                wn3 = Workload(api, ctx, "3", rank, naive=True, world=world, strong=strong)
            rn3 = StepReplayer(torch, wn3, 1, stream, wn3.R)
            nms3, _ = time_steps(torch, dist, world, rn3, wn3.R, stream)
            k9["naive_n81"] = {"value": wn3.units * world * wn3.R / (nms3 / 1e3) / 1e6, "unit": c3["unit"],
                               "ms_per_step": nms3 / wn3.R}
            k9["speedup_latent_vs_naive"] = (nms3 / wn3.R) / (ms3 / s3)
            del wn3, rn3
        if rank == 0 and not args.no_parity:
            try:
                k9["parity"] = parity_gbuffer(w3, 16)
            except Exception as e:  # noqa: BLE001
                k9["parity"] = {"unavailable": str(e)}
        extra["k9"] = k9
        del w3, r3
        wl_units = n_in
    else:
        wl_units = wl.units

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the contract: rank 0 at N = 1 only
        try:
            c = cpu_reference_run(args.config, budget_s=args.cpu_seconds)
            cpu = {k_: c[k_] for k_ in ("value", "unit", "cores", "kind", "sample", "seconds", "cpu", "reps")}
            if cpu["cores"] > 1:  # the single-thread rate beside the all-core one
                old = os.environ.get("HADACODEC_THREADS")
                os.environ["HADACODEC_THREADS"] = "1"
                try:
                    one = cpu_reference_run(args.config, budget_s=max(2.0, args.cpu_seconds / 4), threads=1)
                finally:
                    if old is None:
                        os.environ.pop("HADACODEC_THREADS", None)
                    else:
                        os.environ["HADACODEC_THREADS"] = old
                cpu["single_thread_value"] = one["value"]
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": cfg["unit"], "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": metric_name(args.config),
            "value": value, "unit": cfg["unit"], "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": cfg.get("dtype", "bf16" if args.config == "5a" else "f32"),
            "data": "synthetic (seeded, DESIGN.md Inputs)",
            "config": config_dict(args.config),
            "units_per_gpu": wl_units,
            "method": {
                "l2": (f"{R} rotating input/output buffer sets ({'each' if R == 1 else 'rotation'} > 2x 126 MB L2)"
                       if cfg.get("graph", True) else "compute-bound step (no L2 rotation needed)"),
                "timing": ("CUDA graphs (one graph of exactly K steps up to 512 launches, else chunk graphs + the "
                           "remainder) replaying exactly K steps; CUDA "
                           "events on the launching stream, the start event queued behind a 200 us spin kernel so "
                           "the host's graph-launch latency is outside the interval; max over ranks"
                           if cfg.get("graph", True) else
                           "K library calls (host-side setup included); CUDA events; max over ranks"),
                "parallelism": (f"row bands, {args.scaling} scaling, {world} rank(s), one process per GPU, "
                                "no data-path collective")},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches_timed),
            "ms_per_step_dist": dist_ms,
            "clocks": clocks.summary(),
            "wall_s_timed": t_wall,
        }
        if world > 1:
            line["nccl"] = nccl_record(world, rank)
        line.update(extra)
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e_config2(torch, dist, world, wl, stream, steps):
    """Config 2 end to end through the reference-facing host-buffer C-ABI calls: pinned host
    G-buffer in, XYZ + sRGB out, every frame's H2D and D2H inside the timed region."""
    cfg = wl.cfg
    P = wl.units
    idx, cosv, _ = wl.sets[0]
    h_idx = torch.empty(P, dtype=torch.int32, pin_memory=True)
    h_cos = torch.empty(P, cfg["L"], pin_memory=True)
    h_idx.copy_(idx)
    h_cos.copy_(cosv)
    h_pal = wl.pal_codes.cpu().numpy()
    h_xyz = torch.empty(P, 3, pin_memory=True)
    h_rgb = torch.empty(P, 3, pin_memory=True)
    ni, nc, nx, nr = h_idx.numpy(), h_cos.numpy(), h_xyz.numpy(), h_rgb.numpy()
    with torch.cuda.stream(stream):
        for _ in range(3):
            wl.codec.shade_latent_host(h_pal, wl.light_codes, ni, nc, nx, nr)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        esteps = max(5, min(steps, 50))
        t0 = time.perf_counter()
        for _ in range(esteps):
            wl.codec.shade_latent_host(h_pal, wl.light_codes, ni, nc, nx, nr)
        el = time.perf_counter() - t0
    el = _max_over_ranks(torch, dist, world, el)
    single = {"value": P * world * esteps / el / 1e6, "ms_per_step": el / esteps * 1e3,
              "api": "hc_shade_latent_host, one synchronous call per frame"}
    dev_rgb = wl.sets[0][2]["rgb"].cpu().numpy()
    ok1 = bool(np.array_equal(dev_rgb, nr))
    # Frame stream through hc_shade_latent_host_frames (one pipeline across frames); two
    # pinned input / output sets alternate.
    idx1, cosv1, _ = wl.sets[1]
    h_idx1 = torch.empty(P, dtype=torch.int32, pin_memory=True)
    h_cos1 = torch.empty(P, cfg["L"], pin_memory=True)
    h_idx1.copy_(idx1)
    h_cos1.copy_(cosv1)
    h_xyz1 = torch.empty(P, 3, pin_memory=True)
    h_rgb1 = torch.empty(P, 3, pin_memory=True)
    sets_h = [(ni, nc, nx, nr), (h_idx1.numpy(), h_cos1.numpy(), h_xyz1.numpy(), h_rgb1.numpy())]
    frames = [sets_h[f % 2] for f in range(esteps)]
    with torch.cuda.stream(stream):
        wl.codec.shade_latent_host_frames(h_pal, wl.light_codes, frames[:4])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        wl.codec.shade_latent_host_frames(h_pal, wl.light_codes, frames)
        el2 = time.perf_counter() - t0
    el2 = _max_over_ranks(torch, dist, world, el2)
    ok2 = bool(np.array_equal(wl.sets[1][2]["rgb"].cpu().numpy(), sets_h[1][3]) and np.array_equal(dev_rgb, nr))
    e2e = {"value": P * world * esteps / el2 / 1e6, "unit": cfg["unit"],
           "h2d_bytes_per_step": int(h_idx.numel() * 4 + h_cos.numel() * 4),
           "d2h_bytes_per_step": int(h_xyz.numel() * 4 + h_rgb.numel() * 4), "ms_per_step": el2 / esteps * 1e3,
           "steps": esteps,
           "api": f"hc_shade_latent_host_frames (pinned host buffers, {esteps} frames per call)",
           "single_frame": single}
    return e2e, ok1, ok2


# ---------------------------------------------------------------------------- full-size parity
VERIFY_CONFIGS = ("1", "2", "3", "4", "5a", "5b")


def _cmp(name: str, got, want, tol: float) -> dict:
    got = np.asarray(got)
    want = np.asarray(want)
    if got.shape != want.shape:
        return {"name": name, "pass": False, "error": f"shape {got.shape} vs {want.shape}"}
    rel = rel_err_rows(got, want)
    mabs = 0.0
    for a in range(0, want.shape[0], 1 << 20):
        mabs = max(mabs, float(np.max(np.abs(np.asarray(got[a:a + (1 << 20)], np.float64) - want[a:a + (1 << 20)]))))
    return {"name": name, "max_rel": rel, "max_abs": mabs, "tol": tol, "pass": bool(rel <= tol)}


def verify_config(key: str, rank: int = 0) -> dict:
    """One step of config `key` at BASELINE size on the GPU (the bench's own inputs: buffer
    set 0, seed SEED), against the reference on the host (oracle/_ref, all threads) on the
    same inputs.  Config 4 checks every 16th row; the others the full output."""
    import torch

    import oracle
    from paper_2602_18741_b200 import api, synth

    ref = oracle.reference(81)
    if ref is None:
        raise RuntimeError("oracle/_ref not built")
    torch.cuda.set_device(0)
    cfg = CONFIGS[key]
    t0 = time.perf_counter()
    ctx = api.Context(0)
    wl = Workload(api, ctx, key, rank)
    wl.step(0)
    torch.cuda.synchronize()
    k = cfg["k"]
    E, D = wl.codec.E, wl.codec.D
    checks = []
    if key in ("2", "3"):
        par = parity_gbuffer(wl, 1)
        for name in ("spectra", "xyz", "rgb"):
            if name in par:
                checks.append({"name": name, **par[name], "tol": 1e-5, "pass": par[name]["max_rel"] <= 1e-5})
        # the naive n = 81 ground truth at full size too (every 16th row checked)
        wn = Workload(api, ctx, key, rank, naive=True)
        wn.step(0)
        torch.cuda.synchronize()
        for name, r in parity_naive_gbuffer(wn, 16).items():
            checks.append({"name": name, **r, "tol": 1e-5, "pass": r["max_rel"] <= 1e-5})
        del wn
        sample = f"full {cfg['W']}x{cfg['H']} frame (naive: every 16th row)"
    elif key == "1":
        S, outs = wl.sets[0]
        P = wl.units
        hS = S.cpu().numpy()
        want = {"codes": np.zeros((P, k), np.float32), "spectra": np.zeros((P, N_SPEC), np.float32),
                "xyz": np.zeros((P, 3), np.float32), "rgb": np.zeros((P, 3), np.float32)}
        # codes and spectra: the compiled reference; XYZ / sRGB: the oracle's restatement of
        # image_to_linear_rgb with the analytic CMF rows the config names (the reference's
        # CmfTable is tabulated)
        ref.ref_codec_roundtrip(E, D, k, hS, P, want["codes"], want["spectra"], None, None, 0)
        orc = oracle.oracle()
        junk = [np.zeros((P, d), np.float32) for d in (k, N_SPEC)]
        orc.orc_codec_roundtrip(E, D, k, N_SPEC, cmf_analytic(N_SPEC), 5.0, hS, P, junk[0], junk[1], want["xyz"],
                                want["rgb"])
        for name in ("codes", "spectra", "xyz", "rgb"):
            checks.append(_cmp(name, outs[name].cpu().numpy(), want[name], 1e-5))
        sample = f"all {P} spectra (XYZ / sRGB with the analytic CMF fit)"
    elif key == "4":
        pidx, iidx, tw, outs = wl.sets[0]
        W, H, spp = cfg["W"], cfg["H"], cfg["spp"]
        rows = np.arange(0, H, 16)
        sel = torch.from_numpy((rows[:, None] * W + np.arange(W)[None, :]).reshape(-1)).cuda()
        m = sel.numel()
        h_p = np.ascontiguousarray(pidx.reshape(wl.units, -1)[sel].cpu().numpy())
        h_i = np.ascontiguousarray(iidx.reshape(wl.units, -1)[sel].cpu().numpy())
        h_t = np.ascontiguousarray(tw.reshape(wl.units, -1)[sel].cpu().numpy())
        pal = synth.palette(SEED, 256, N_SPEC)
        ill = synth.lights(SEED, 16, N_SPEC, purpose="scene.illuminants")
        pc, ic = np.zeros((256, k), np.float32), np.zeros((16, k), np.float32)
        ref.ref_asset_codes(E, k, pal, 256, pc)
        ref.ref_asset_codes(E, k, ill, 16, ic)
        X, R = np.zeros((m, 3), np.float32), np.zeros((m, 3), np.float32)
        ref.ref_multibounce_latent(E, D, k, pc, ic, h_p, h_i, h_t, m, spp, 4, None, X, R, 0)
        checks.append(_cmp("xyz", outs["xyz"][sel].cpu().numpy(), X, 1e-5))
        checks.append(_cmp("rgb", outs["rgb"][sel].cpu().numpy(), R, 1e-5))
        # the naive n = 81 chain (ground truth) on the same samples
        nv = wl.codec.multibounce_spectral(torch.from_numpy(pal).cuda(), torch.from_numpy(ill).cuda(), pidx, iidx, tw)
        torch.cuda.synchronize()
        Xn, Rn = np.zeros((m, 3), np.float32), np.zeros((m, 3), np.float32)
        ref.ref_multibounce_spectral(pal, ill, h_p, h_i, h_t, m, spp, 4, Xn, Rn, 0)
        checks.append(_cmp("naive xyz", nv["xyz"][sel].cpu().numpy(), Xn, 1e-5))
        checks.append(_cmp("naive rgb", nv["rgb"][sel].cpu().numpy(), Rn, 1e-5))
        del nv
        sample = f"every 16th row ({m} px x {spp} spp; latent and naive)"
    elif key == "5a":
        rgb, out = wl.sets[0]
        P = wl.units
        w = synth.mlp_weights(SEED, 6, 64)
        want = np.zeros((P, 6), np.float32)
        ref.ref_mlp_forward(rgb.cpu().numpy(), P, 64, 6, w["w1"], w["b1"], w["w2"], w["b2"], w["w3"], w["b3"], want,
                            0)
        checks.append(_cmp("codes", out.cpu().numpy(), want, 1e-2))
        sample = f"all {P} texels (bf16 tolerance 1e-2)"
    else:  # 5b
        A, B = wl.sets[0]
        P = wl.units
        got = float(wl.sum.cpu().numpy()[0])
        hA, hB = A.cpu().numpy(), B.cpu().numpy()
        want = ref.ref_hadamard_loss(E, D, k, hA, hB, P, 0)
        del hA, hB
        rel = abs(got - want) / abs(want)
        checks.append({"name": "loss", "got": got, "want": want, "max_rel": rel, "tol": 1e-5, "pass": rel <= 1e-5})
        sample = f"all {P} pairs"
    res = {"verify": key, "workload": cfg["name"], "sample": sample, "checks": checks,
           "pass": all(c["pass"] for c in checks), "seconds": round(time.perf_counter() - t0, 1),
           "checker": "oracle/_ref (the reference compiled from its sources; SURVEY §8c R1-R4 restatements on "
                      "top of its primitives), all host threads"}
    del wl
    torch.cuda.empty_cache()
    return res


def run_verify(args) -> int:
    keys = [c.strip() for c in args.verify_configs.split(",") if c.strip()]
    ok = True
    for key in keys:
        r = verify_config(key)
        ok &= r["pass"]
        emit(r)
    return 0 if ok else 1


def spawn_ranks(n: int, argv: list) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on this node, rendezvous on 127.0.0.1; rank 0 prints the line."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="2")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: one frame per GPU (default); strong: one frame split into row bands")
    ap.add_argument("--gather", choices=("nccl", "fused"), default="nccl",
                    help="N > 1: 'fused' adds a with_gather_fused record (bands stored straight into rank 0's "
                         "frame through peer memory) next to the NCCL gather")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-naive", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-k9", action="store_true", help="default config: skip the config 3 (k = 9) sub-record")
    ap.add_argument("--no-parity", action="store_true", help="skip the parity record against the reference")
    ap.add_argument("--verify", action="store_true",
                    help="full-size parity of the configs' outputs against the reference (no timing)")
    ap.add_argument("--verify-configs", default=",".join(VERIFY_CONFIGS))
    ap.add_argument("--plain", action="store_true", help="profiling mode: plain launches only")
    ap.add_argument("--naive-plain", action="store_true", help="with --plain: also run the naive path")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.verify:
        return spawn_ranks(args.gpus, sys.argv[1:] if argv is None else list(argv))
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.verify:
        return run_verify(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
