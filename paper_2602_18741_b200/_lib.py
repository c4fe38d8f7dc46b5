"""ctypes binding of the in-tree C ABI (include/hadacodec_b200.h).

Loading fails loudly when ``libhadacodec_b200.so`` is missing: there is no CPU
fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# HC_LIB overrides the library path (tuning sweeps load variant builds from tools/bin/).
LIB_PATH = Path(os.environ.get("HC_LIB") or Path(__file__).resolve().parent / "libhadacodec_b200.so")

HC_OK, HC_EINVAL, HC_EDOMAIN, HC_ECUDA, HC_ENOMEM, HC_EUNSUPPORTED = range(6)

vp = C.c_void_p
i32, i64, u64, f64 = C.c_int, C.c_int64, C.c_uint64, C.c_double

SIGNATURES: dict[str, tuple] = {
    "hc_last_error": (C.c_char_p, []),
    "hc_version": (C.c_char_p, []),
    "hc_ctx_create": (i32, [i32, vp, C.POINTER(vp)]),
    "hc_ctx_destroy": (i32, [vp]),
    "hc_ctx_set_stream": (i32, [vp, vp]),
    "hc_ctx_synchronize": (i32, [vp]),
    "hc_ctx_launch_count": (i64, [vp]),
    "hc_codec_create": (i32, [vp, i32, i32, vp, vp, vp, f64, C.POINTER(vp)]),
    "hc_codec_create_raw": (i32, [vp, i32, i32, f64, vp, vp, vp, f64, C.POINTER(vp)]),
    "hc_codec_create_f64": (i32, [vp, i32, i32, vp, vp, vp, C.c_double, C.POINTER(vp)]),
    "hc_codec_destroy": (i32, [vp]),
    "hc_codec_dims": (i32, [vp, C.POINTER(i32), C.POINTER(i32)]),
    "hc_codec_xyz_projection": (i32, [vp, vp]),
    "hc_encode": (i32, [vp, vp, i64, vp]),
    "hc_decode": (i32, [vp, vp, i64, vp, vp, vp, i32]),
    "hc_roundtrip": (i32, [vp, vp, i64, vp, vp, vp, vp]),
    "hc_spectra_to_xyz_rgb": (i32, [vp, vp, i64, vp, vp]),
    "hc_blockwise_hadamard": (i32, [vp, vp, vp, i64, i32, vp]),
    "hc_shade_latent": (i32, [vp, vp, i32, vp, i32, vp, vp, i64, vp, vp, vp, vp]),
    "hc_shade_latent_pass": (i32, [vp, i32, vp, i32, vp, i32, vp, vp, i64, vp]),
    "hc_reassemble": (i32, [vp, vp, i32, i64, vp]),
    "hc_shade_spectral": (i32, [vp, vp, i32, vp, i32, vp, vp, i64, vp, vp, vp]),
    "hc_multibounce_latent": (i32, [vp, vp, i32, vp, i32, vp, vp, vp, i64, i32, vp, vp, vp]),
    "hc_multibounce_spectral": (i32, [vp, vp, i32, vp, i32, vp, vp, vp, i64, i32, vp, vp]),
    "hc_mlp_create": (i32, [vp, i32, i32, vp, vp, vp, vp, vp, vp, C.POINTER(vp)]),
    "hc_mlp_destroy": (i32, [vp]),
    "hc_mlp_forward": (i32, [vp, vp, i64, vp]),
    "hc_hadamard_loss": (i32, [vp, vp, vp, i64, vp]),
    "hc_row_band": (i32, [i32, i32, i64, C.POINTER(i64), C.POINTER(i64)]),
    "hc_group_create": (i32, [vp, i32, i32, C.POINTER(vp)]),
    "hc_group_destroy": (i32, [vp]),
    "hc_group_size": (i32, [vp]),
    "hc_group_nccl_version": (i32, []),
    "hc_group_codec_create": (i32, [vp, i32, i32, vp, vp, vp, f64]),
    "hc_group_shade_latent_host": (i32, [vp, vp, i32, vp, i32, vp, vp, i64, i64, vp, vp]),
    "hc_ipc_alloc": (i32, [i32, i64, C.POINTER(vp), vp]),
    "hc_ipc_open": (i32, [i32, vp, C.POINTER(vp)]),
    "hc_ipc_close": (i32, [i32, vp]),
    "hc_ipc_free": (i32, [i32, vp]),
    "hc_exposure_for": (i32, [vp, vp, i64, i32, f64, C.POINTER(f64)]),
    "hc_tonemap_srgb8": (i32, [vp, vp, i64, f64, vp]),
    "hc_error_map": (i32, [vp, vp, i32, vp, i32, i64, vp, C.POINTER(f64)]),
    "hc_scene_color_report": (i32, [vp, vp, i32, vp, i32, i64, vp]),
    "hc_scene_color_report_dev": (i32, [vp, vp, i32, vp, i32, i64, vp, vp]),
    "hc_delta_e94_report": (i32, [vp, vp, vp, i64, vp, vp, vp]),
    "hc_spectra_to_xyz_f64": (i32, [vp, vp, i64, vp, vp]),
    "hc_format_g17": (i32, [vp, vp, i64, vp, vp]),
    "hc_codes_csv_write": (i32, [vp, vp, i64, i32, u64, vp, i64, C.POINTER(i64)]),
    "hc_codes_csv_write_ids": (i32, [vp, vp, i32, i64, i32, vp, vp, C.c_char_p, u64, vp, i64, C.POINTER(i64)]),
    "hc_spectra_csv_write": (i32, [vp, vp, i32, i64, i32, vp, i32, vp, vp, C.c_char_p, u64, vp, i64,
                                   C.POINTER(i64)]),
    "hc_spectra_csv_read": (i32, [vp, vp, i64, C.POINTER(i32), vp, i32, C.POINTER(i32), C.POINTER(i64), vp, vp,
                                  i64]),
    "hc_encode_resampled_f64": (i32, [vp, vp, i32, vp, i64, C.c_double, C.c_double, i32, vp]),
    "hc_decode_f64": (i32, [vp, vp, i64, vp, C.POINTER(i64)]),
    "hc_encode_f64": (i32, [vp, vp, i64, vp]),
    "hc_codec_effective_f64": (i32, [vp, vp, vp]),
    "hc_codec_train_grad": (i32, [vp, i32, i32, C.c_double, vp, vp, vp, C.c_double, vp, vp, i64, vp, vp, vp, vp]),
    "hc_adam_step": (i32, [vp, vp, vp, vp, vp, i64, C.c_double, i64]),
    "hc_upsampler_create": (i32, [vp, i32, i32, vp, vp, vp, vp, vp, vp, C.POINTER(vp)]),
    "hc_upsampler_destroy": (i32, [vp]),
    "hc_upsample_f64": (i32, [vp, vp, i64, i32, vp, C.POINTER(C.c_uint64)]),
    "hc_upsample_train_grad": (i32, [vp, i32, i32, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, i64, C.c_double,
                                     C.c_double, vp, vp]),
    "hc_adamw_step": (i32, [vp, vp, vp, vp, vp, i64, C.c_double, C.c_double, i64]),
    "hc_parse_doubles": (i32, [vp, vp, vp, i64, i32, vp, vp]),
    "hc_codes_csv_read": (i32, [vp, vp, i64, C.POINTER(i32), C.POINTER(i64), vp, vp, i64]),
    "hc_render": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "hc_render_latent_multipass": (i32, [vp, vp, vp, vp, vp, vp]),
    "hc_shade_latent_host": (i32, [vp, vp, i32, vp, i32, vp, vp, i64, vp, vp]),
    "hc_shade_latent_host_frames": (i32, [vp, vp, i32, vp, i32, i32, vp, vp, i64, vp, vp]),
    "hc_roundtrip_host": (i32, [vp, vp, i64, vp, vp, vp, vp]),
    "hc_stream_key": (u64, [u64, C.c_char_p]),
    "hc_synth_gm_spectra": (i32, [vp, u64, i64, i64, i32, f64, f64, vp]),
    "hc_synth_gbuffer": (i32, [vp, u64, u64, i64, i64, i32, i32, vp, vp]),
    "hc_synth_chain": (i32, [vp, u64, u64, u64, i64, i64, i32, i32, i32, vp, vp, vp]),
    "hc_synth_uniform": (i32, [vp, u64, i64, i64, vp]),
    "hc_flush_l2": (i32, [vp, vp, i64]),
    "hc_spin": (i32, [vp, i64]),
}

_lib = None


class HcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[hc {code}] {msg}")
        self.code = code


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2602_18741_b200.build` "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != HC_OK:
        msg = lib().hc_last_error().decode(errors="replace")
        if rc == HC_EINVAL:
            raise ValueError(msg)
        if rc == HC_EDOMAIN:
            raise ArithmeticError(msg)  # std::domain_error analogue
        raise HcError(rc, msg)
