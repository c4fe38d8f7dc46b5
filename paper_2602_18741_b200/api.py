"""Python host API over the C ABI, mirroring the reference ``hadacodec`` interface
for the per-pixel path (codec.hpp, colorimetry.hpp, renderer.hpp, upsampler.hpp,
evaluation.hpp) with batched torch CUDA tensors in place of single curves.

PyTorch provides device memory and streams only; every computation is a kernel
of ``libhadacodec_b200.so``.  Calls are enqueued on torch's current stream.

  reference (core/include/hadacodec)         here
  -------------------------------------      ---------------------------------------
  encode(EffectiveWeights, SpectralCurve)    Codec.encode(S[rows, n]) -> Z[rows, k]
  decode(EffectiveWeights, LatentCode)       Codec.decode(Z, check_negative=True)
  decode_image(ChannelImage, CodecWeights)   Codec.decode(Z) -> spectra / xyz / rgb
  image_to_linear_rgb(ChannelImage)          Codec.spectra_to_xyz_rgb(S)
  blockwise_hadamard(LatentCode, LatentCode) blockwise_hadamard(A, B)
  render(..., latent) / multipass            Codec.shade_latent / shade_latent_pass + reassemble
  render(..., spectral)                      Codec.shade_spectral
  multibounce chain (evaluation.cpp:50-76)   Codec.multibounce_latent / _spectral
  upsample(UpsamplerWeights, rgb)            Upsampler.forward(rgb[P, 3]) -> codes[P, k]
  loss residual (trainer.cpp:49-71)          Codec.hadamard_loss(A, B)
  exposure_for / tonemap_srgb8 / error_map   exposure_for / tonemap_srgb8 / error_map
  scene_color_report (evaluation.cpp)        scene_color_report; delta_e94_report (per pixel)
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .colorimetry import cmf_matrix, grid

_check = _lib.check


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _np_ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _cuda(t: torch.Tensor, dtype: torch.dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


class Context:
    """One hc_ctx per device; enqueues on torch's current stream at each call."""

    def __init__(self, device: int | torch.device | None = None):
        if device is None:
            index = torch.cuda.current_device()
        elif isinstance(device, int):
            index = device
        else:
            index = torch.device(device).index or 0
        dev = torch.device("cuda", index)
        self.device = dev
        L = _lib.lib()
        h = C.c_void_p()
        with torch.cuda.device(dev):
            _check(L.hc_ctx_create(dev.index, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream), C.byref(h)))
        self.h = h
        self._lib = L

    def bind_stream(self) -> None:
        self._lib.hc_ctx_set_stream(self.h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))

    def synchronize(self) -> None:
        """Stream sync + report latched device-side violations (HC_EDOMAIN / HC_EINVAL)."""
        self.bind_stream()
        _check(self._lib.hc_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(self._lib.hc_ctx_launch_count(self.h))

    def empty(self, *shape, dtype=torch.float32) -> torch.Tensor:
        return torch.empty(*shape, dtype=dtype, device=self.device)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._lib.hc_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Codec:
    """Effective encoder E (k x n) / decoder D (n x k) + CMF projection (codec.hpp:52-58)."""

    def __init__(self, ctx: Context, E: np.ndarray, D: np.ndarray, cmf: Optional[np.ndarray] = None,
                 dlambda: Optional[float] = None):
        E = np.ascontiguousarray(E, dtype=np.float32)
        D = np.ascontiguousarray(D, dtype=np.float32)
        k, n = E.shape
        if D.shape != (n, k):
            raise ValueError("codec weights: parameter array size mismatch")
        self.ctx, self.k, self.n = ctx, k, n
        self.E, self.D = E, D
        self.cmf = np.ascontiguousarray(cmf_matrix(n) if cmf is None else cmf, dtype=np.float64)
        self.dlambda = grid(n)[1] if dlambda is None else float(dlambda)
        h = C.c_void_p()
        _check(_lib.lib().hc_codec_create(ctx.h, k, n, _np_ptr(E), _np_ptr(D), _np_ptr(self.cmf), self.dlambda,
                                          C.byref(h)))
        self.h = h

    @classmethod
    def from_raw(cls, ctx: Context, raw_enc: np.ndarray, raw_dec: np.ndarray, beta: float = 10.0) -> "Codec":
        """CodecWeights path: effective = softplus_beta(raw) (codec.cpp:21-34), computed in the library."""
        re = np.ascontiguousarray(raw_enc, dtype=np.float64)
        rd = np.ascontiguousarray(raw_dec, dtype=np.float64)
        k, n = re.shape
        obj = cls.__new__(cls)
        obj.ctx, obj.k, obj.n = ctx, k, n
        obj.cmf = np.ascontiguousarray(cmf_matrix(n), dtype=np.float64)
        obj.dlambda = grid(n)[1]
        h = C.c_void_p()
        _check(_lib.lib().hc_codec_create_raw(ctx.h, k, n, beta, _np_ptr(re), _np_ptr(rd), _np_ptr(obj.cmf),
                                              obj.dlambda, C.byref(h)))
        obj.h = h
        sp = lambda r: np.where(beta * r > 30.0, r, np.log1p(np.exp(np.minimum(beta * r, 30.0))) / beta)  # noqa: E731
        obj.E, obj.D = sp(re).astype(np.float32), sp(rd).astype(np.float32)
        return obj

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().hc_codec_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def xyz_projection(self) -> np.ndarray:
        out = np.zeros((3, self.k), np.float32)
        _check(_lib.lib().hc_codec_xyz_projection(self.h, _np_ptr(out)))
        return out

    # ------------------------------------------------------------ codec
    def encode(self, S: torch.Tensor) -> torch.Tensor:
        S = _cuda(S, torch.float32, "S")
        rows = S.numel() // self.n
        Z = self.ctx.empty(rows, self.k)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_encode(self.h, _p(S), rows, _p(Z)))
        return Z

    def decode(self, Z: torch.Tensor, spectra: bool = True, xyz: bool = False, rgb: bool = False,
               check_negative: bool = False) -> dict:
        Z = _cuda(Z, torch.float32, "Z")
        rows = Z.numel() // self.k
        out = {"spectra": self.ctx.empty(rows, self.n) if spectra else None,
               "xyz": self.ctx.empty(rows, 3) if xyz else None,
               "rgb": self.ctx.empty(rows, 3) if rgb else None}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_decode(self.h, _p(Z), rows, _p(out["spectra"]), _p(out["xyz"]), _p(out["rgb"]),
                                    int(check_negative)))
        if check_negative:
            self.ctx.synchronize()
        return out

    def roundtrip(self, S: torch.Tensor, codes: bool = True, spectra: bool = True, xyz: bool = True,
                  rgb: bool = True, out: Optional[dict] = None) -> dict:
        S = _cuda(S, torch.float32, "S")
        rows = S.numel() // self.n
        if out is None:
            out = {"codes": self.ctx.empty(rows, self.k) if codes else None,
                   "spectra": self.ctx.empty(rows, self.n) if spectra else None,
                   "xyz": self.ctx.empty(rows, 3) if xyz else None,
                   "rgb": self.ctx.empty(rows, 3) if rgb else None}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_roundtrip(self.h, _p(S), rows, _p(out.get("codes")), _p(out.get("spectra")),
                                       _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def spectra_to_xyz_rgb(self, S: torch.Tensor) -> dict:
        S = _cuda(S, torch.float32, "S")
        rows = S.numel() // self.n
        out = {"xyz": self.ctx.empty(rows, 3), "rgb": self.ctx.empty(rows, 3)}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_spectra_to_xyz_rgb(self.h, _p(S), rows, _p(out["xyz"]), _p(out["rgb"])))
        return out

    # ------------------------------------------------------------ shading
    def shade_latent(self, pal_codes: torch.Tensor, light_codes: np.ndarray, idx: torch.Tensor,
                     cosv: torch.Tensor, latent: bool = False, spectra: bool = False, xyz: bool = True,
                     rgb: bool = True, out: Optional[dict] = None) -> dict:
        pal_codes = _cuda(pal_codes, torch.float32, "pal_codes")
        lc = np.ascontiguousarray(light_codes, dtype=np.float32)
        L = lc.shape[0]
        P = idx.numel()
        if out is None:
            out = {"latent": self.ctx.empty(P, self.k) if latent else None,
                   "spectra": self.ctx.empty(P, self.n) if spectra else None,
                   "xyz": self.ctx.empty(P, 3) if xyz else None,
                   "rgb": self.ctx.empty(P, 3) if rgb else None}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_latent(self.h, _p(pal_codes), pal_codes.shape[0], _np_ptr(lc), L, _p(idx),
                                          _p(cosv), P, _p(out.get("latent")), _p(out.get("spectra")),
                                          _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def shade_latent_pass(self, pass_index: int, pal_codes: torch.Tensor, light_codes: np.ndarray,
                          idx: torch.Tensor, cosv: torch.Tensor) -> torch.Tensor:
        lc = np.ascontiguousarray(light_codes, dtype=np.float32)
        P = idx.numel()
        img = self.ctx.empty(P, 3)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_latent_pass(self.h, pass_index, _p(pal_codes), pal_codes.shape[0],
                                               _np_ptr(lc), lc.shape[0], _p(idx), _p(cosv), P, _p(img)))
        return img

    def shade_spectral(self, pal_spectra: torch.Tensor, light_spectra: np.ndarray, idx: torch.Tensor,
                       cosv: torch.Tensor, spectra: bool = False, out: Optional[dict] = None) -> dict:
        pal_spectra = _cuda(pal_spectra, torch.float32, "pal_spectra")
        ls = np.ascontiguousarray(light_spectra, dtype=np.float32)
        P = idx.numel()
        if out is None:
            out = {"spectra": self.ctx.empty(P, self.n) if spectra else None,
                   "xyz": self.ctx.empty(P, 3), "rgb": self.ctx.empty(P, 3)}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_spectral(self.h, _p(pal_spectra), pal_spectra.shape[0], _np_ptr(ls),
                                            ls.shape[0], _p(idx), _p(cosv), P, _p(out.get("spectra")),
                                            _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def multibounce_latent(self, pal_codes, ill_codes, pidx, iidx, tw, latent: bool = False,
                           out: Optional[dict] = None) -> dict:
        P, spp = iidx.shape
        if out is None:
            out = {"latent": self.ctx.empty(P, self.k) if latent else None,
                   "xyz": self.ctx.empty(P, 3), "rgb": self.ctx.empty(P, 3)}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_multibounce_latent(self.h, _p(pal_codes), pal_codes.shape[0], _p(ill_codes),
                                                ill_codes.shape[0], _p(pidx), _p(iidx), _p(tw), P, spp,
                                                _p(out.get("latent")), _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def multibounce_spectral(self, pal_spectra, ill_spectra, pidx, iidx, tw, out: Optional[dict] = None) -> dict:
        P, spp = iidx.shape
        if out is None:
            out = {"xyz": self.ctx.empty(P, 3), "rgb": self.ctx.empty(P, 3)}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_multibounce_spectral(self.h, _p(pal_spectra), pal_spectra.shape[0], _p(ill_spectra),
                                                  ill_spectra.shape[0], _p(pidx), _p(iidx), _p(tw), P, spp,
                                                  _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def hadamard_loss(self, A: torch.Tensor, B: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        A = _cuda(A, torch.float32, "A")
        B = _cuda(B, torch.float32, "B")
        pairs = A.numel() // self.n
        if out is None:
            out = self.ctx.empty(1, dtype=torch.float64)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_hadamard_loss(self.h, _p(A), _p(B), pairs, _p(out)))
        return out

    # ------------------------------------------------------------ host-buffer (reference-facing) calls
    def shade_latent_host(self, pal_codes: np.ndarray, light_codes: np.ndarray, idx: np.ndarray,
                          cosv: np.ndarray, xyz: np.ndarray, rgb: np.ndarray) -> None:
        lc = np.ascontiguousarray(light_codes, dtype=np.float32)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_latent_host(self.h, _np_ptr(pal_codes), pal_codes.shape[0], _np_ptr(lc),
                                               lc.shape[0], _np_ptr(idx), _np_ptr(cosv), idx.size, _np_ptr(xyz),
                                               _np_ptr(rgb)))

    def roundtrip_host(self, S: np.ndarray, Z: Optional[np.ndarray] = None, S2: Optional[np.ndarray] = None,
                       xyz: Optional[np.ndarray] = None, rgb: Optional[np.ndarray] = None) -> None:
        """Host-buffer round trip (encode -> decode_image -> image_to_linear_rgb); outputs may be None."""
        S = np.ascontiguousarray(S, dtype=np.float32)
        rows = S.size // self.n
        self.ctx.bind_stream()
        _check(_lib.lib().hc_roundtrip_host(self.h, _np_ptr(S), rows, *[None if a is None else _np_ptr(a)
                                                                        for a in (Z, S2, xyz, rgb)]))


def blockwise_hadamard(ctx: Context, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """codec.cpp:77-85, batched over rows."""
    if A.shape != B.shape:
        raise ValueError("blockwise_hadamard: dimension mismatch")
    A = _cuda(A, torch.float32, "A")
    B = _cuda(B, torch.float32, "B")
    k = A.shape[-1]
    out = torch.empty_like(A)
    ctx.bind_stream()
    _check(_lib.lib().hc_blockwise_hadamard(ctx.h, _p(A), _p(B), A.numel() // k, k, _p(out)))
    return out


def reassemble(ctx: Context, passes: Sequence[torch.Tensor]) -> torch.Tensor:
    """render_latent_multipass reassembly (renderer.cpp:645-657)."""
    P = passes[0].shape[0]
    arr = (C.c_void_p * len(passes))(*[p.data_ptr() for p in passes])
    latent = ctx.empty(P, 3 * len(passes))
    ctx.bind_stream()
    _check(_lib.lib().hc_reassemble(ctx.h, C.cast(arr, C.c_void_p), len(passes), P, _p(latent)))
    return latent


# ------------------------------------------------------------ colour-metric tail
def _image(t: torch.Tensor, codec: "Codec", name: str) -> tuple[torch.Tensor, int, int]:
    t = _cuda(t, torch.float32, name)
    ch = t.shape[-1] if t.dim() > 1 else 1
    if ch not in (3, codec.n):
        raise ValueError(f"{name}: expected 3 or {codec.n} channels (decode latent images first)")
    return t, ch, t.numel() // ch


def exposure_for(codec: "Codec", img: torch.Tensor, percentile: float = 99.5) -> float:
    """renderer.cpp:721-752: 1 / nearest-rank luminance percentile (1 if <= 1e-12)."""
    img, ch, P = _image(img, codec, "img")
    out = C.c_double()
    codec.ctx.bind_stream()
    _check(_lib.lib().hc_exposure_for(codec.h, _p(img), P, ch, float(percentile), C.byref(out)))
    return out.value


def tonemap_srgb8(ctx: Context, rgb: torch.Tensor, exposure: float, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """renderer.cpp:754-773: uint8 [P, 3] sRGB of exposure-scaled linear RGB."""
    rgb = _cuda(rgb, torch.float32, "rgb")
    P = rgb.numel() // 3
    if out is None:
        out = torch.empty(P, 3, dtype=torch.uint8, device=rgb.device)
    ctx.bind_stream()
    _check(_lib.lib().hc_tonemap_srgb8(ctx.h, _p(rgb), P, float(exposure), _p(out)))
    return out


def error_map(codec: "Codec", a: torch.Tensor, b: torch.Tensor) -> tuple[torch.Tensor, float]:
    """renderer.cpp:775-802: (per-pixel linear-RGB MSE [P] f32, mean MSE)."""
    a, ca, P = _image(a, codec, "a")
    b, cb, Pb = _image(b, codec, "b")
    if P != Pb:
        raise ValueError("error_map: image sizes differ")
    mse = codec.ctx.empty(P)
    mean = C.c_double()
    codec.ctx.bind_stream()
    _check(_lib.lib().hc_error_map(codec.h, _p(a), ca, _p(b), cb, P, _p(mse), C.byref(mean)))
    return mse, mean.value


def scene_color_report(codec: "Codec", gt: torch.Tensor, test: torch.Tensor) -> dict:
    """evaluation.cpp:122-154: mean / p95 Delta E76, linear-RGB MSE, exposure of the ground truth."""
    gt, cg, P = _image(gt, codec, "gt")
    test, ct, Pt = _image(test, codec, "test")
    if P != Pt:
        raise ValueError("scene_color_report: image sizes differ")
    out = (C.c_double * 4)()
    codec.ctx.bind_stream()
    _check(_lib.lib().hc_scene_color_report(codec.h, _p(gt), cg, _p(test), ct, P, C.cast(out, C.c_void_p)))
    return {"mean_de76": out[0], "p95_de76": out[1], "mse": out[2], "exposure": out[3]}


def scene_color_report_dev(codec: "Codec", gt: torch.Tensor, test: torch.Tensor, out: Optional[torch.Tensor] = None,
                           preview: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Stream-ordered scene_color_report: f64 [4] device tensor {mean_de76, p95_de76, mse, exposure};
    `preview` (uint8 [P, 3], optional) receives tonemap_srgb8(test, exposure) from the same pass."""
    gt, cg, P = _image(gt, codec, "gt")
    test, ct, Pt = _image(test, codec, "test")
    if P != Pt:
        raise ValueError("scene_color_report: image sizes differ")
    if out is None:
        out = codec.ctx.empty(4, dtype=torch.float64)
    codec.ctx.bind_stream()
    _check(_lib.lib().hc_scene_color_report_dev(codec.h, _p(gt), cg, _p(test), ct, P, _p(out), _p(preview)))
    return out


def delta_e94_report(ctx: Context, xyz_gt: torch.Tensor, xyz_test: torch.Tensor, n: int = 81,
                     white: Optional[Sequence[float]] = None, per_pixel: bool = False) -> dict:
    """multibounce_eval's metric (evaluation.cpp:59-86) per pixel: mean / median / p95 Delta E94
    with the D65 white (CmfTable::white_xyz of grid n unless given) scaled to the truth's Y."""
    from .colorimetry import white_xyz

    xyz_gt = _cuda(xyz_gt, torch.float32, "xyz_gt")
    xyz_test = _cuda(xyz_test, torch.float32, "xyz_test")
    P = xyz_gt.numel() // 3
    if xyz_test.numel() != xyz_gt.numel():
        raise ValueError("delta_e94_report: image sizes differ")
    w = (C.c_double * 3)(*(white if white is not None else white_xyz(n)))
    out = (C.c_double * 3)()
    de = ctx.empty(P) if per_pixel else None
    ctx.bind_stream()
    _check(_lib.lib().hc_delta_e94_report(ctx.h, _p(xyz_gt), _p(xyz_test), P, C.cast(w, C.c_void_p), _p(de),
                                          C.cast(out, C.c_void_p)))
    res = {"mean_de94": out[0], "median_de94": out[1], "p95_de94": out[2]}
    if per_pixel:
        res["de94"] = de
    return res


def split_blocks(z: np.ndarray) -> list:
    """codec.cpp:87-98 (host-side; block i = channels 3i..3i+2)."""
    z = np.asarray(z)
    if z.shape[-1] % 3 != 0:
        raise ValueError("split_blocks: k must be a multiple of 3")
    return [z[..., 3 * i:3 * i + 3] for i in range(z.shape[-1] // 3)]


def join_blocks(blocks: Sequence[np.ndarray]) -> np.ndarray:
    """codec.cpp:100-109."""
    return np.concatenate([np.asarray(b) for b in blocks], axis=-1)


class Upsampler:
    """RGB -> code MLP (upsampler.cpp:42-72; ReLU / softplus head, bf16 tcgen05)."""

    def __init__(self, ctx: Context, w: dict):
        self.ctx = ctx
        self.hidden = w["w1"].shape[0]
        self.k = w["w3"].shape[0]
        arrs = [np.ascontiguousarray(w[key], dtype=np.float32) for key in ("w1", "b1", "w2", "b2", "w3", "b3")]
        self._keep = arrs
        h = C.c_void_p()
        _check(_lib.lib().hc_mlp_create(ctx.h, self.hidden, self.k, *[_np_ptr(a) for a in arrs], C.byref(h)))
        self.h = h

    def forward(self, rgb: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        rgb = _cuda(rgb, torch.float32, "rgb")
        P = rgb.numel() // 3
        if out is None:
            out = self.ctx.empty(P, self.k)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_mlp_forward(self.h, _p(rgb), P, _p(out)))
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().hc_mlp_destroy(self.h)
                self.h = None
        except Exception:
            pass


# ------------------------------------------------------------ device generators
def stream_key(seed: int, purpose: str) -> int:
    return int(_lib.lib().hc_stream_key(seed, purpose.encode()))


def synth_gm_spectra(ctx: Context, seed: int, purpose: str, first: int, count: int, n: int) -> torch.Tensor:
    lo, step = grid(n)
    out = ctx.empty(count, n)
    ctx.bind_stream()
    _check(_lib.lib().hc_synth_gm_spectra(ctx.h, stream_key(seed, purpose), first, count, n, lo, step, _p(out)))
    return out


def synth_gbuffer(ctx: Context, seed: int, first: int, P: int, L: int, n_pal: int):
    idx = ctx.empty(P, dtype=torch.int32)
    cosv = ctx.empty(P, L)
    ctx.bind_stream()
    _check(_lib.lib().hc_synth_gbuffer(ctx.h, stream_key(seed, "gbuffer.idx"), stream_key(seed, "gbuffer.cos"),
                                       first, P, L, n_pal, _p(idx), _p(cosv)))
    return idx, cosv


def synth_chain(ctx: Context, seed: int, first: int, P: int, spp: int, n_pal: int, n_ill: int):
    pidx = ctx.empty(P, spp, 4, dtype=torch.uint8)
    iidx = ctx.empty(P, spp, dtype=torch.uint8)
    tw = ctx.empty(P, spp, 4)
    ctx.bind_stream()
    _check(_lib.lib().hc_synth_chain(ctx.h, stream_key(seed, "chain.pidx"), stream_key(seed, "chain.iidx"),
                                     stream_key(seed, "chain.tw"), first, P, spp, n_pal, n_ill, _p(pidx),
                                     _p(iidx), _p(tw)))
    return pidx, iidx, tw


def synth_uniform(ctx: Context, seed: int, purpose: str, first: int, count: int) -> torch.Tensor:
    out = ctx.empty(count)
    ctx.bind_stream()
    _check(_lib.lib().hc_synth_uniform(ctx.h, stream_key(seed, purpose), first, count, _p(out)))
    return out


def flush_l2(ctx: Context, buf: torch.Tensor) -> None:
    ctx.bind_stream()
    _check(_lib.lib().hc_flush_l2(ctx.h, _p(buf), buf.numel() * buf.element_size()))
