"""ORACLE / TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes front-ends for
  * ``lib/libhc_oracle.so`` — the plain-C restatement (hc_oracle.c), and
  * ``_ref/libhcref{47,81}.so`` — the reference core compiled from
    /root/reference by ``make -C oracle ref`` plus ``ref_shim.cpp``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this package, and only as the checker / baseline — never on the product
path (the product fails loudly without its CUDA library).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "lib" / "libhc_oracle.so"
REF_LIB = {47: HERE / "_ref" / "libhcref47.so", 81: HERE / "_ref" / "libhcref81.so"}
REFERENCE_CORE = Path("/root/reference/proj/core")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build(with_reference: bool | None = None) -> None:
    """Compile the C restatement, and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if with_reference is None:
        with_reference = REFERENCE_CORE.is_dir()
    if with_reference:
        subprocess.run(["make", "-s", "-j", str(os.cpu_count() or 4), "-C", str(HERE), "ref"], check=True)


def _opt(a):
    return None if a is None else a


class _Lib:
    def __init__(self, path: Path, sigs: dict):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle` / `make -C oracle ref`)")
        self.lib = C.CDLL(str(path))
        for name, (res, args) in sigs.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args


def _nullable(ptype):
    """ndpointer that also accepts None (-> NULL)."""

    class _N(ptype):  # type: ignore[misc, valid-type]
        @classmethod
        def from_param(cls, obj):
            if obj is None:
                return None
            return ptype.from_param(obj)

    return _N


_f32n = _nullable(_f32p)
_f64n = _nullable(_f64p)

_ORACLE_SIGS = {
    "orc_softplus": (C.c_double, [C.c_double, C.c_double]),
    "orc_encode": (None, [_f32p, C.c_int, C.c_int, _f32p, C.c_int64, _f64n, _f32n]),
    "orc_decode": (None, [_f32p, C.c_int, C.c_int, _f32p, C.c_int64, _f32p]),
    "orc_spectra_to_outputs": (None, [_f64p, C.c_double, C.c_int, _f32p, C.c_int64, _f32n, _f32n]),
    "orc_spectrum_to_xyz_d": (None, [_f64p, C.c_double, C.c_int, _f64p, _f64p]),
    "orc_codec_roundtrip": (None, [_f32p, _f32p, C.c_int, C.c_int, _f64p, C.c_double, _f32p, C.c_int64,
                                   _f32n, _f32n, _f32n, _f32n]),
    "orc_asset_codes": (None, [_f32p, C.c_int, C.c_int, _f32p, C.c_int64, _f32p]),
    "orc_shade_latent": (None, [_f32p, C.c_int, C.c_int, _f64p, C.c_double, _f32p, _f32p, C.c_int, _u32p,
                                _f32p, C.c_int64, _f32n, _f32n, _f32n, _f32n]),
    "orc_shade_spectral": (None, [C.c_int, _f64p, C.c_double, _f32p, _f32p, C.c_int, _u32p, _f32p,
                                  C.c_int64, _f32n, _f32n, _f32n]),
    "orc_chain": (None, [C.c_int, _f32p, _f32p, _u8p, _u8p, _f32p, C.c_int64, C.c_int, C.c_int, _f32p]),
    "orc_bf16_round": (C.c_float, [C.c_float]),
    "orc_mlp_forward": (None, [_f32p, C.c_int64, C.c_int, C.c_int, _f32p, _f32p, _f32p, _f32p, _f32p,
                               _f32p, _f32p]),
    "orc_hadamard_loss": (C.c_double, [_f32p, _f32p, C.c_int, C.c_int, _f32p, _f32p, C.c_int64]),
    # colour-metric tail
    "orc_percentile_nearest_rank": (C.c_double, [_f64p, C.c_int64, C.c_double]),
    "orc_luminance": (None, [_f32p, C.c_int64, C.c_int, _f64n, C.c_double, _f64p]),
    "orc_exposure_for": (C.c_double, [_f32p, C.c_int64, C.c_int, _f64n, C.c_double, C.c_double]),
    "orc_srgb_encode": (C.c_double, [C.c_double]),
    "orc_tonemap_srgb8": (None, [_f32p, C.c_int64, C.c_double, _u8p]),
    "orc_image_to_linear_rgb": (None, [_f32p, C.c_int64, C.c_int, _f64p, C.c_double, _f32p]),
    "orc_error_map": (C.c_double, [_f32p, C.c_int, _f32p, C.c_int, C.c_int64, _f64p, C.c_double, _f32n]),
    "orc_xyz_to_lab": (None, [_f64p, _f64p, _f64p]),
    "orc_delta_e76": (C.c_double, [_f64p, _f64p]),
    "orc_delta_e94": (C.c_double, [_f64p, _f64p]),
    "orc_scene_color_report": (None, [_f32p, C.c_int, _f32p, C.c_int, C.c_int64, _f64p, C.c_double, _f64p]),
    "orc_delta_e94_report": (None, [_f32p, _f32p, C.c_int64, _f64p, _f32n, _f64p]),
}

_REF_SIGS = {
    "ref_grid_n": (C.c_int, []),
    "ref_lambda_min": (C.c_double, []),
    "ref_lambda_step": (C.c_double, []),
    "ref_wavelength_at": (C.c_double, [C.c_int]),
    "ref_cmf_table": (None, [_f64p]),
    "ref_white_xyz": (None, [_f64p]),
    "ref_spectrum_to_xyz_d": (None, [_f64p, _f64p]),
    "ref_xyz_to_linear_rgb_d": (None, [_f64p, _f64p]),
    "ref_softplus": (C.c_double, [C.c_double, C.c_double]),
    "ref_rng_stream_u64": (None, [C.c_uint64, C.c_char_p, C.c_int, _u64p]),
    "ref_rng_seed_u64": (None, [C.c_uint64, C.c_int, _u64p]),
    "ref_pixel_stream_u64": (None, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_int, _u64p]),
    "ref_fnv1a64": (C.c_uint64, [C.c_char_p, C.c_int64]),
    "ref_gaussian_curve": (None, [C.c_double, C.c_double, C.c_double, _f64p]),
    "ref_blackbody_curve": (None, [C.c_double, _f64p]),
    "ref_init_upsampler": (None, [C.c_int, C.c_int, C.c_uint64, _f64p, _f64p, _f64p]),
    "ref_encode_rows_d": (None, [_f32p, C.c_int, _f32p, C.c_int64, _f64p, C.c_int]),
    "ref_decode_rows_d": (C.c_int, [_f32p, C.c_int, _f64p, C.c_int64, _f64p]),
    "ref_codec_roundtrip": (None, [_f32p, _f32p, C.c_int, _f32p, C.c_int64, _f32n, _f32n, _f32n, _f32n, C.c_int]),
    "ref_decode_image": (None, [_f32p, _f32p, C.c_int, _f32p, C.c_int64, _f32n, _f32n, _f32n, C.c_int]),
    "ref_spectra_to_outputs": (None, [_f32p, C.c_int64, _f32n, _f32n, C.c_int]),
    "ref_asset_codes": (None, [_f32p, C.c_int, _f32p, C.c_int64, _f32p]),
    "ref_shade_latent": (None, [_f32p, _f32p, C.c_int, _f32p, _f32p, C.c_int, _u32p, _f32p, C.c_int64,
                                _f32n, _f32n, _f32n, _f32n, C.c_int]),
    "ref_shade_spectral": (None, [_f32p, _f32p, C.c_int, _u32p, _f32p, C.c_int64, _f32n, _f32n, _f32n, C.c_int]),
    "ref_multibounce_latent": (None, [_f32p, _f32p, C.c_int, _f32p, _f32p, _u8p, _u8p, _f32p, C.c_int64,
                                      C.c_int, C.c_int, _f32n, _f32n, _f32n, C.c_int]),
    "ref_multibounce_spectral": (None, [_f32p, _f32p, _u8p, _u8p, _f32p, C.c_int64, C.c_int, C.c_int,
                                        _f32n, _f32n, C.c_int]),
    "ref_mlp_forward": (None, [_f32p, C.c_int64, C.c_int, C.c_int, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p,
                               _f32p, C.c_int]),
    "ref_hadamard_loss": (C.c_double, [_f32p, _f32p, C.c_int, _f32p, _f32p, C.c_int64, C.c_int]),
    "ref_thread_count": (C.c_int, []),
    # colour-metric tail
    "ref_exposure_for": (C.c_double, [_f32p, C.c_int64, C.c_int, C.c_double]),
    "ref_tonemap_srgb8": (None, [_f32p, C.c_int64, C.c_double, _u8p]),
    "ref_error_map": (C.c_double, [_f32p, C.c_int, _f32p, C.c_int, C.c_int64, _f32n]),
    "ref_scene_color_report": (None, [_f32p, C.c_int, _f32p, C.c_int, C.c_int64, _f64p]),
    "ref_xyz_to_lab": (None, [_f64p, _f64p, _f64p]),
    "ref_delta_e76": (C.c_double, [_f64p, _f64p]),
    "ref_delta_e94": (C.c_double, [_f64p, _f64p]),
    "ref_srgb_encode": (C.c_double, [C.c_double]),
    "ref_delta_e94_report": (None, [_f32p, _f32p, C.c_int64, _f32n, _f64p]),
    # formats
    "ref_write_codes_csv": (C.c_int, [C.c_char_p, _f32p, C.c_int64, C.c_int, C.c_uint64]),
    "ref_save_codec_weights": (C.c_int, [C.c_char_p, C.c_int, C.c_double, _f64p, _f64p, C.c_uint64, _f64p, C.c_int]),
    "ref_load_codec_weights": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), _f64p, _f64p,
                                         C.c_int64, C.c_char_p, C.c_int64]),
    "ref_write_raw_image": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, _f32p]),
    "ref_read_raw_image": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), _f32p,
                                     C.c_int64, C.c_char_p, C.c_int64]),
    "ref_write_ppm": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_int64]),
    "ref_read_ppm": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_char_p, C.c_int64, C.c_char_p,
                               C.c_int64]),
    "ref_codec_gradients": (C.c_int, [C.c_int, C.c_double, _f64p, _f64p, _f64p, _f64p, C.c_int64, _f64p,
                                      C.c_void_p, C.c_void_p, _f64p]),
    "ref_upsample": (C.c_int, [C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, C.c_int64, C.c_int,
                               _f64p, C.POINTER(C.c_uint64)]),
    "ref_save_upsampler_weights": (C.c_int, [C.c_char_p, C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p,
                                             C.c_int]),
    "ref_upsample_train": (C.c_int, [C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, C.c_double, _f64p,
                                     _f64p, _f64p, _f64p, C.c_int64, C.c_double, C.c_double, _f64p, C.c_void_p]),
    "ref_run_encode": (C.c_int, [C.c_char_p, C.c_int, C.c_double, _f64p, _f64p, C.c_char_p, C.c_char_p, C.c_int64]),
    "ref_run_decode": (C.c_int, [C.c_char_p, C.c_int, C.c_double, _f64p, _f64p, C.c_char_p, C.c_char_p, C.c_int64]),
    "ref_write_spectra_csv": (C.c_int, [C.c_char_p, _f64p, C.c_int64, C.c_char_p, C.c_void_p]),
    "ref_read_spectra_csv": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), _f64p, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int64), _f64p, C.c_int64, C.c_char_p, C.c_int64]),
    "ref_write_codes_csv_ids": (C.c_int, [C.c_char_p, _f64p, C.c_int64, C.c_int, C.c_char_p,
                                          np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")]),
    "ref_read_codes_csv": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int), _f64p, C.c_int64,
                                     C.c_char_p, C.c_int64]),
    # path tracer
    "ref_render": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _f32n, _f32n, C.c_int, _f32p,
                             _nullable(np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")),
                             C.POINTER(C.c_uint64)]),
}

_oracle = None
_refs: dict = {}


def oracle() -> "C.CDLL":
    """The C restatement (always available once `make -C oracle` ran)."""
    global _oracle
    if _oracle is None:
        if not ORACLE_LIB.exists():
            build(with_reference=False)
        _oracle = _Lib(ORACLE_LIB, _ORACLE_SIGS).lib
    return _oracle


def reference(n: int = 81):
    """The compiled reference for grid n (47 = unchanged, 81 = re-gridded); None if not built."""
    if n not in _refs:
        p = REF_LIB[n]
        _refs[n] = _Lib(p, _REF_SIGS).lib if p.exists() else None
    return _refs[n]


def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
