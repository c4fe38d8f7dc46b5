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
  upsample / upsample_raw (fp64, SiLU)       Upsampler.forward(rgb[P, 3], clamp) -> codes[P, k], clamped
  BASELINE MLP (3-64-64-6, bf16 tcgen05)     CodeMLP.forward(rgb[P, 3]) -> codes[P, 6]
  loss residual (trainer.cpp:49-71)          Codec.hadamard_loss(A, B)
  compute_losses + gradients, adam_step      codec_train_grad, adam_step
  print_g17 / codes CSV / spectra CSV        format_g17, codes_csv, read_codes_csv, spectra_csv, read_spectra_csv
  run_encode / run_decode tools              encode_tool, decode_tool (encode_resampled, decode_f64)
  load_codec_weights, read/write_raw_image   load_codec_weights, read_raw_image, write_raw_image
  exposure_for / tonemap_srgb8 / error_map   exposure_for / tonemap_srgb8 / error_map
  scene_color_report (evaluation.cpp)        scene_color_report; delta_e94_report (per pixel)
  render / render_latent_multipass           render(codec, scene, mode, ..., multipass)
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .colorimetry import cmf_matrix, grid, wavelengths

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


_IDX_DTYPES = (torch.int32,) + ((torch.uint32,) if hasattr(torch, "uint32") else ())


def _shape_ok(shape, want) -> bool:
    return len(shape) == len(want) and all(w is None or s == w for s, w in zip(shape, want))


def _dev_in(t, dtypes, name: str, shape=None, numel=None) -> torch.Tensor:
    """A device input: CUDA tensor of one of `dtypes`, made contiguous, with the exact
    shape (None = any extent) or element count the C ABI will read."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    dtypes = dtypes if isinstance(dtypes, tuple) else (dtypes,)
    if t.dtype not in dtypes:
        raise TypeError(f"{name} must be {' or '.join(map(str, dtypes))}, got {t.dtype}")
    if shape is not None and not _shape_ok(tuple(t.shape), shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {shape}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name}: {t.numel()} elements, expected {numel}")
    return t.contiguous()


def _dev_out(t, name: str, shape, dtype=torch.float32) -> Optional[torch.Tensor]:
    """A caller-supplied device output: written in place, so it must already be contiguous."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype:
        raise TypeError(f"{name} must be a {dtype} CUDA tensor")
    if not t.is_contiguous() or t.numel() != int(np.prod(shape)):
        raise ValueError(f"{name}: must be contiguous with shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def _host_arr(a, dtypes, name: str, numel: int, writable: bool = False) -> Optional[np.ndarray]:
    """A host buffer the C ABI reads (or, writable, fills): exact dtype, C-contiguous, size."""
    if a is None:
        return None
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{name} must be a numpy array")
    dtypes = dtypes if isinstance(dtypes, tuple) else (dtypes,)
    if a.dtype not in [np.dtype(d) for d in dtypes]:
        raise TypeError(f"{name} must be {' or '.join(np.dtype(d).name for d in dtypes)}, got {a.dtype}")
    if not a.flags.c_contiguous or (writable and not a.flags.writeable):
        raise ValueError(f"{name} must be a C-contiguous{' writable' if writable else ''} array")
    if a.size != numel:
        raise ValueError(f"{name}: {a.size} elements, expected {numel}")
    return a


def _codes_table(a, k: int, name: str) -> np.ndarray:
    lc = np.ascontiguousarray(a, dtype=np.float32)
    if lc.ndim != 2 or lc.shape[1] != k:
        raise ValueError(f"{name}: shape {lc.shape}, expected (rows, {k})")
    return lc


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

    @classmethod
    def from_weights_file(cls, ctx: Context, path) -> "Codec":
        """A codec from the reference's weight file (load_codec_weights, io.cpp:370-393)."""
        w = load_codec_weights(path)
        return cls.from_raw(ctx, w["raw_enc"], w["raw_dec"], beta=w["beta"])

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().hc_codec_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def effective_f64(self) -> tuple[np.ndarray, np.ndarray]:
        """(E [k, n], D [n, k]) in fp64 as the library holds them (effective_weights)."""
        E = np.zeros((self.k, self.n), np.float64)
        D = np.zeros((self.n, self.k), np.float64)
        _check(_lib.lib().hc_codec_effective_f64(self.h, _np_ptr(E), _np_ptr(D)))
        return E, D

    @property
    def xyz_projection(self) -> np.ndarray:
        out = np.zeros((3, self.k), np.float32)
        _check(_lib.lib().hc_codec_xyz_projection(self.h, _np_ptr(out)))
        return out

    # ------------------------------------------------------------ codec
    def _rows(self, t: torch.Tensor, width: int, name: str) -> int:
        if t.numel() % width:
            raise ValueError(f"{name}: {t.numel()} elements is not a whole number of {width}-wide rows")
        return t.numel() // width

    def encode(self, S: torch.Tensor) -> torch.Tensor:
        S = _cuda(S, torch.float32, "S")
        rows = self._rows(S, self.n, "S")
        Z = self.ctx.empty(rows, self.k)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_encode(self.h, _p(S), rows, _p(Z)))
        return Z

    def decode(self, Z: torch.Tensor, spectra: bool = True, xyz: bool = False, rgb: bool = False,
               check_negative: bool = False) -> dict:
        Z = _cuda(Z, torch.float32, "Z")
        rows = self._rows(Z, self.k, "Z")
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
        rows = self._rows(S, self.n, "S")
        if out is None:
            out = {"codes": self.ctx.empty(rows, self.k) if codes else None,
                   "spectra": self.ctx.empty(rows, self.n) if spectra else None,
                   "xyz": self.ctx.empty(rows, 3) if xyz else None,
                   "rgb": self.ctx.empty(rows, 3) if rgb else None}
        for key, w in (("codes", self.k), ("spectra", self.n), ("xyz", 3), ("rgb", 3)):
            _dev_out(out.get(key), key, (rows, w))
        self.ctx.bind_stream()
        _check(_lib.lib().hc_roundtrip(self.h, _p(S), rows, _p(out.get("codes")), _p(out.get("spectra")),
                                       _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def spectra_to_xyz_rgb(self, S: torch.Tensor) -> dict:
        S = _cuda(S, torch.float32, "S")
        rows = self._rows(S, self.n, "S")
        out = {"xyz": self.ctx.empty(rows, 3), "rgb": self.ctx.empty(rows, 3)}
        self.ctx.bind_stream()
        _check(_lib.lib().hc_spectra_to_xyz_rgb(self.h, _p(S), rows, _p(out["xyz"]), _p(out["rgb"])))
        return out

    # ------------------------------------------------------------ shading
    def _gbuffer(self, idx, cosv, L: int):
        P = idx.numel() if isinstance(idx, torch.Tensor) else 0
        idx = _dev_in(idx, _IDX_DTYPES, "idx", numel=P)
        cosv = _dev_in(cosv, torch.float32, "cosv", numel=P * L)
        return idx, cosv, P

    def shade_latent(self, pal_codes: torch.Tensor, light_codes: np.ndarray, idx: torch.Tensor,
                     cosv: torch.Tensor, latent: bool = False, spectra: bool = False, xyz: bool = True,
                     rgb: bool = True, out: Optional[dict] = None) -> dict:
        pal_codes = _dev_in(pal_codes, torch.float32, "pal_codes", shape=(None, self.k))
        lc = _codes_table(light_codes, self.k, "light_codes")
        L = lc.shape[0]
        idx, cosv, P = self._gbuffer(idx, cosv, L)
        if out is None:
            out = {"latent": self.ctx.empty(P, self.k) if latent else None,
                   "spectra": self.ctx.empty(P, self.n) if spectra else None,
                   "xyz": self.ctx.empty(P, 3) if xyz else None,
                   "rgb": self.ctx.empty(P, 3) if rgb else None}
        for key, w in (("latent", self.k), ("spectra", self.n), ("xyz", 3), ("rgb", 3)):
            _dev_out(out.get(key), key, (P, w))
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_latent(self.h, _p(pal_codes), pal_codes.shape[0], _np_ptr(lc), L, _p(idx),
                                          _p(cosv), P, _p(out.get("latent")), _p(out.get("spectra")),
                                          _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def shade_latent_pass(self, pass_index: int, pal_codes: torch.Tensor, light_codes: np.ndarray,
                          idx: torch.Tensor, cosv: torch.Tensor) -> torch.Tensor:
        pal_codes = _dev_in(pal_codes, torch.float32, "pal_codes", shape=(None, self.k))
        lc = _codes_table(light_codes, self.k, "light_codes")
        idx, cosv, P = self._gbuffer(idx, cosv, lc.shape[0])
        img = self.ctx.empty(P, 3)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_latent_pass(self.h, pass_index, _p(pal_codes), pal_codes.shape[0],
                                               _np_ptr(lc), lc.shape[0], _p(idx), _p(cosv), P, _p(img)))
        return img

    def shade_spectral(self, pal_spectra: torch.Tensor, light_spectra: np.ndarray, idx: torch.Tensor,
                       cosv: torch.Tensor, spectra: bool = False, out: Optional[dict] = None) -> dict:
        pal_spectra = _dev_in(pal_spectra, torch.float32, "pal_spectra", shape=(None, self.n))
        ls = _codes_table(light_spectra, self.n, "light_spectra")
        idx, cosv, P = self._gbuffer(idx, cosv, ls.shape[0])
        if out is None:
            out = {"spectra": self.ctx.empty(P, self.n) if spectra else None,
                   "xyz": self.ctx.empty(P, 3), "rgb": self.ctx.empty(P, 3)}
        for key, w in (("spectra", self.n), ("xyz", 3), ("rgb", 3)):
            _dev_out(out.get(key), key, (P, w))
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_spectral(self.h, _p(pal_spectra), pal_spectra.shape[0], _np_ptr(ls),
                                            ls.shape[0], _p(idx), _p(cosv), P, _p(out.get("spectra")),
                                            _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def _chain(self, table, ill, pidx, iidx, tw, width: int):
        if not isinstance(iidx, torch.Tensor) or iidx.dim() != 2:
            raise ValueError("iidx must be a [P, spp] CUDA tensor")
        P, spp = iidx.shape
        table = _dev_in(table, torch.float32, "palette", shape=(None, width))
        ill = _dev_in(ill, torch.float32, "illuminants", shape=(None, width))
        pidx = _dev_in(pidx, torch.uint8, "pidx", numel=P * spp * 4)
        iidx = _dev_in(iidx, torch.uint8, "iidx", numel=P * spp)
        tw = _dev_in(tw, torch.float32, "tw", numel=P * spp * 4)
        return table, ill, pidx, iidx, tw, P, spp

    def multibounce_latent(self, pal_codes, ill_codes, pidx, iidx, tw, latent: bool = False,
                           out: Optional[dict] = None) -> dict:
        pal_codes, ill_codes, pidx, iidx, tw, P, spp = self._chain(pal_codes, ill_codes, pidx, iidx, tw, self.k)
        if out is None:
            out = {"latent": self.ctx.empty(P, self.k) if latent else None,
                   "xyz": self.ctx.empty(P, 3), "rgb": self.ctx.empty(P, 3)}
        for key, w in (("latent", self.k), ("xyz", 3), ("rgb", 3)):
            _dev_out(out.get(key), key, (P, w))
        self.ctx.bind_stream()
        _check(_lib.lib().hc_multibounce_latent(self.h, _p(pal_codes), pal_codes.shape[0], _p(ill_codes),
                                                ill_codes.shape[0], _p(pidx), _p(iidx), _p(tw), P, spp,
                                                _p(out.get("latent")), _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def multibounce_spectral(self, pal_spectra, ill_spectra, pidx, iidx, tw, out: Optional[dict] = None) -> dict:
        pal_spectra, ill_spectra, pidx, iidx, tw, P, spp = self._chain(pal_spectra, ill_spectra, pidx, iidx, tw,
                                                                       self.n)
        if out is None:
            out = {"xyz": self.ctx.empty(P, 3), "rgb": self.ctx.empty(P, 3)}
        for key in ("xyz", "rgb"):
            _dev_out(out.get(key), key, (P, 3))
        self.ctx.bind_stream()
        _check(_lib.lib().hc_multibounce_spectral(self.h, _p(pal_spectra), pal_spectra.shape[0], _p(ill_spectra),
                                                  ill_spectra.shape[0], _p(pidx), _p(iidx), _p(tw), P, spp,
                                                  _p(out.get("xyz")), _p(out.get("rgb"))))
        return out

    def hadamard_loss(self, A: torch.Tensor, B: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        A = _cuda(A, torch.float32, "A")
        B = _cuda(B, torch.float32, "B")
        pairs = self._rows(A, self.n, "A")
        if B.numel() != A.numel():
            raise ValueError("hadamard_loss: A and B must hold the same number of spectra")
        if out is None:
            out = self.ctx.empty(1, dtype=torch.float64)
        _dev_out(out, "out", (1,), torch.float64)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_hadamard_loss(self.h, _p(A), _p(B), pairs, _p(out)))
        return out

    # ------------------------------------------------------------ host-buffer (reference-facing) calls
    def shade_latent_host(self, pal_codes: np.ndarray, light_codes: np.ndarray, idx: np.ndarray,
                          cosv: np.ndarray, xyz: np.ndarray, rgb: np.ndarray) -> None:
        pal = _codes_table(pal_codes, self.k, "pal_codes")
        lc = _codes_table(light_codes, self.k, "light_codes")
        P = idx.size if isinstance(idx, np.ndarray) else 0
        _host_arr(idx, (np.uint32, np.int32), "idx", P)
        _host_arr(cosv, np.float32, "cosv", P * lc.shape[0])
        _host_arr(xyz, np.float32, "xyz", P * 3, writable=True)
        _host_arr(rgb, np.float32, "rgb", P * 3, writable=True)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_latent_host(self.h, _np_ptr(pal), pal.shape[0], _np_ptr(lc),
                                               lc.shape[0], _np_ptr(idx), _np_ptr(cosv), P,
                                               None if xyz is None else _np_ptr(xyz),
                                               None if rgb is None else _np_ptr(rgb)))

    def shade_latent_host_frames(self, pal_codes: np.ndarray, light_codes: np.ndarray, frames) -> None:
        """A frame stream through one host-buffer pipeline (hc_shade_latent_host_frames).

        frames: sequence of (idx, cosv, xyz, rgb) host arrays of P pixels each (xyz / rgb may be
        None); outputs are identical to one shade_latent_host call per frame.  Copies overlap
        the kernels only for page-locked (pinned) buffers."""
        import ctypes as C

        pal = _codes_table(pal_codes, self.k, "pal_codes")
        lc = _codes_table(light_codes, self.k, "light_codes")
        nf = len(frames)
        if nf == 0:
            return
        P = frames[0][0].size if isinstance(frames[0][0], np.ndarray) else 0
        for i, f in enumerate(frames):
            _host_arr(f[0], (np.uint32, np.int32), f"frames[{i}].idx", P)
            _host_arr(f[1], np.float32, f"frames[{i}].cosv", P * lc.shape[0])
            _host_arr(f[2], np.float32, f"frames[{i}].xyz", P * 3, writable=True)
            _host_arr(f[3], np.float32, f"frames[{i}].rgb", P * 3, writable=True)
        tab = [(C.c_void_p * nf)(*[(_np_ptr(f[j]) if f[j] is not None else None) for f in frames])
               for j in range(4)]
        self.ctx.bind_stream()
        _check(_lib.lib().hc_shade_latent_host_frames(self.h, _np_ptr(pal), pal.shape[0], _np_ptr(lc),
                                                      lc.shape[0], nf, C.addressof(tab[0]), C.addressof(tab[1]), P,
                                                      C.addressof(tab[2]), C.addressof(tab[3])))

    def roundtrip_host(self, S: np.ndarray, Z: Optional[np.ndarray] = None, S2: Optional[np.ndarray] = None,
                       xyz: Optional[np.ndarray] = None, rgb: Optional[np.ndarray] = None) -> None:
        """Host-buffer round trip (encode -> decode_image -> image_to_linear_rgb); outputs may be None."""
        S = np.ascontiguousarray(S, dtype=np.float32)
        if S.size % self.n:
            raise ValueError(f"S: {S.size} elements is not a whole number of {self.n}-sample spectra")
        rows = S.size // self.n
        for a, name, w in ((Z, "Z", self.k), (S2, "S2", self.n), (xyz, "xyz", 3), (rgb, "rgb", 3)):
            _host_arr(a, np.float32, name, rows * w, writable=True)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_roundtrip_host(self.h, _np_ptr(S), rows, *[None if a is None else _np_ptr(a)
                                                                        for a in (Z, S2, xyz, rgb)]))


GATHER_MODES = {"host": 0, "nccl": 1, "peer": 2, "fused": 3}


class Group:
    """Several GPUs driven from this process (hc_group_*: one host thread, context and stream
    per device, row bands, gather by host copies / NCCL / peer copies)."""

    def __init__(self, devices: Sequence[int], gather: str = "host"):
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(_lib.lib().hc_group_create(arr, len(devices), GATHER_MODES[gather], C.byref(h)))
        self.h, self.devices, self.gather = h, list(devices), gather
        self.k = self.n = None

    @staticmethod
    def nccl_version() -> int:
        return int(_lib.lib().hc_group_nccl_version())

    def set_codec(self, E: np.ndarray, D: np.ndarray) -> None:
        E = np.ascontiguousarray(E, dtype=np.float32)
        D = np.ascontiguousarray(D, dtype=np.float32)
        k, n = E.shape
        if D.shape != (n, k):
            raise ValueError("codec weights: parameter array size mismatch")
        cmf = np.ascontiguousarray(cmf_matrix(n), dtype=np.float64)
        _check(_lib.lib().hc_group_codec_create(self.h, k, n, _np_ptr(E), _np_ptr(D), _np_ptr(cmf), grid(n)[1]))
        self.k, self.n = k, n

    def shade_latent_host(self, pal_codes: np.ndarray, light_codes: np.ndarray, idx: np.ndarray, cosv: np.ndarray,
                          width: int, height: int, xyz: Optional[np.ndarray], rgb: Optional[np.ndarray]) -> None:
        if self.k is None:
            raise ValueError("group: set_codec first")
        pal = _codes_table(pal_codes, self.k, "pal_codes")
        lc = _codes_table(light_codes, self.k, "light_codes")
        P = width * height
        _host_arr(idx, (np.uint32, np.int32), "idx", P)
        _host_arr(cosv, np.float32, "cosv", P * lc.shape[0])
        _host_arr(xyz, np.float32, "xyz", P * 3, writable=True)
        _host_arr(rgb, np.float32, "rgb", P * 3, writable=True)
        _check(_lib.lib().hc_group_shade_latent_host(self.h, _np_ptr(pal), pal.shape[0], _np_ptr(lc), lc.shape[0],
                                                     _np_ptr(idx), _np_ptr(cosv), width, height,
                                                     None if xyz is None else _np_ptr(xyz),
                                                     None if rgb is None else _np_ptr(rgb)))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().hc_group_destroy(self.h)
                self.h = None
        except Exception:
            pass


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


# ------------------------------------------------------------ path tracer
class HcSceneObject(C.Structure):
    _fields_ = [("kind", C.c_int), ("center", C.c_double * 3), ("radius", C.c_double),
                ("box_min", C.c_double * 3), ("box_max", C.c_double * 3), ("material", C.c_int)]


class HcSceneLight(C.Structure):
    _fields_ = [("corner", C.c_double * 3), ("edge_u", C.c_double * 3), ("edge_v", C.c_double * 3),
                ("spd", C.POINTER(C.c_double)), ("scale", C.c_double)]


class HcScene(C.Structure):
    _fields_ = [("cam_position", C.c_double * 3), ("cam_look_at", C.c_double * 3), ("cam_up", C.c_double * 3),
                ("cam_vfov_degrees", C.c_double), ("box_min", C.c_double * 3), ("box_max", C.c_double * 3),
                ("wall_material", C.c_int * 6), ("n_materials", C.c_int), ("materials", C.POINTER(C.c_double)),
                ("n_objects", C.c_int), ("objects", C.POINTER(HcSceneObject)), ("n_lights", C.c_int),
                ("lights", C.POINTER(HcSceneLight))]


class HcRenderJob(C.Structure):
    _fields_ = [("mode", C.c_int), ("width", C.c_int), ("height", C.c_int), ("spp", C.c_int),
                ("max_depth", C.c_int), ("seed", C.c_uint64)]


RENDER_MODES = {"spectral": 0, "latent": 1, "rgb": 2}


def scene_struct(scene: dict, n: int):
    """(HcScene, keep-alive list) from a scene dict with the reference's field names
    (renderer.hpp:16-53): camera{position, look_at, up, vfov_degrees}, box_min, box_max,
    wall_material[6], materials [m][n], objects [{kind: 'sphere'|'block', center, radius,
    box_min, box_max, material}], lights [{corner, edge_u, edge_v, spd [n], scale}]."""
    keep = []
    cam = {"position": (0, 1, 3.25), "look_at": (0, 1, 0), "up": (0, 1, 0), "vfov_degrees": 40.0}
    cam.update(scene.get("camera", {}))
    mats = np.ascontiguousarray(np.asarray(scene.get("materials", []), dtype=np.float64).reshape(-1, n))
    keep.append(mats)
    objs = (HcSceneObject * max(1, len(scene.get("objects", []))))()
    for i, o in enumerate(scene.get("objects", [])):
        objs[i].kind = 0 if o.get("kind", "sphere") == "sphere" else 1
        objs[i].center[:] = o.get("center", (0, 0, 0))
        objs[i].radius = o.get("radius", 0.0)
        objs[i].box_min[:] = o.get("box_min", (0, 0, 0))
        objs[i].box_max[:] = o.get("box_max", (0, 0, 0))
        objs[i].material = o["material"]
    lts = (HcSceneLight * max(1, len(scene.get("lights", []))))()
    for i, l in enumerate(scene.get("lights", [])):
        spd = np.ascontiguousarray(np.asarray(l["spd"], dtype=np.float64))
        if spd.size != n:
            raise ValueError("scene light spd must have n samples")
        keep.append(spd)
        lts[i].corner[:] = l["corner"]
        lts[i].edge_u[:] = l["edge_u"]
        lts[i].edge_v[:] = l["edge_v"]
        lts[i].spd = spd.ctypes.data_as(C.POINTER(C.c_double))
        lts[i].scale = l.get("scale", 1.0)
    keep += [objs, lts]
    sc = HcScene()
    sc.cam_position[:] = cam["position"]
    sc.cam_look_at[:] = cam["look_at"]
    sc.cam_up[:] = cam["up"]
    sc.cam_vfov_degrees = cam["vfov_degrees"]
    sc.box_min[:] = scene.get("box_min", (-1, 0, -1))
    sc.box_max[:] = scene.get("box_max", (1, 2, 1))
    sc.wall_material[:] = scene.get("wall_material", (-1,) * 6)
    sc.n_materials = mats.shape[0]
    sc.materials = mats.ctypes.data_as(C.POINTER(C.c_double))
    sc.n_objects = len(scene.get("objects", []))
    sc.objects = C.cast(objs, C.POINTER(HcSceneObject))
    sc.n_lights = len(scene.get("lights", []))
    sc.lights = C.cast(lts, C.POINTER(HcSceneLight))
    return sc, keep


def render(codec: "Codec", scene: dict, mode: str = "spectral", width: int = 128, height: int = 128, spp: int = 64,
           max_depth: int = 3, seed: int = 0, path_hashes: bool = False, multipass: bool = False) -> dict:
    """render / render_latent_multipass (renderer.hpp:100-107): image [H, W, C] f32 on the device
    (C = n spectral, k latent, 3 rgb), shading_evals, optional per-pixel path hashes."""
    from .colorimetry import cmf_table

    sc, keep = scene_struct(scene, codec.n)
    job = HcRenderJob(RENDER_MODES["latent" if multipass else mode], width, height, spp, max_depth, seed)
    C_ = {"spectral": codec.n, "latent": codec.k, "rgb": 3}["latent" if multipass else mode]
    img = codec.ctx.empty(height, width, C_)
    hashes = torch.empty(height, width, dtype=torch.int64, device=img.device) if path_hashes else None
    evals = C.c_uint64()
    codec.ctx.bind_stream()
    if multipass:
        _check(_lib.lib().hc_render_latent_multipass(codec.h, C.addressof(sc), C.addressof(job), _p(img), _p(hashes),
                                                     C.addressof(evals)))
    else:
        d65 = np.ascontiguousarray(cmf_table(codec.n)["d65"])
        _check(_lib.lib().hc_render(codec.h, C.addressof(sc), C.addressof(job), _np_ptr(d65), _p(img), _p(hashes),
                                    C.addressof(evals)))
    del keep
    return {"image": img, "path_hashes": hashes, "shading_evals": evals.value}


# ------------------------------------------------------------ formats
def format_g17(ctx: Context, v: torch.Tensor) -> list:
    """print_g17 (io.cpp:108-112) of every value of a float64 CUDA tensor, on the device."""
    v = _cuda(v, torch.float64, "v").reshape(-1)
    n = v.numel()
    slots = torch.empty(n, 32, dtype=torch.uint8, device=v.device)
    lens = torch.empty(n, dtype=torch.uint8, device=v.device)
    ctx.bind_stream()
    _check(_lib.lib().hc_format_g17(ctx.h, _p(v), n, _p(slots), _p(lens)))
    s, ln = slots.cpu().numpy(), lens.cpu().numpy()
    return [bytes(s[i, :ln[i]]).decode() for i in range(n)]


def parse_doubles(ctx: Context, cells: Sequence[bytes]) -> tuple[np.ndarray, np.ndarray]:
    """parse_double (io.cpp:78-88) of trimmed cells on the device: (values, status 0/1/2)."""
    n = len(cells)
    stride = max([len(c) for c in cells] + [1])
    buf = np.zeros((n, stride), np.uint8)
    lens = np.zeros(n, np.uint8 if stride < 256 else np.int64)
    if stride >= 256:
        raise ValueError("parse_doubles: cells longer than 255 bytes")
    for i, c in enumerate(cells):
        buf[i, :len(c)] = np.frombuffer(c, np.uint8)
        lens[i] = len(c)
    d_buf, d_len = torch.from_numpy(buf).cuda(), torch.from_numpy(lens).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.int8, device="cuda")
    ctx.bind_stream()
    _check(_lib.lib().hc_parse_doubles(ctx.h, _p(d_buf), _p(d_len), n, stride, _p(out), _p(st)))
    return out.cpu().numpy(), st.cpu().numpy()


def _id_args(ids, rows: int):
    """(id_bytes, id_spans) device tensors for a list of id strings (None: no ids)."""
    if ids is None:
        return None, None
    if len(ids) != rows:
        raise ValueError("csv: one id per row")
    enc = [str(i).encode() for i in ids]
    lens = np.array([len(e) for e in enc], np.int64)
    spans = np.zeros((max(rows, 1), 2), np.int64)  # never an empty (NULL) tensor
    if rows:
        spans[1:, 0] = np.cumsum(lens)[:-1]
        spans[:, 1] = lens
    blob = b"".join(enc) + b"\0"
    return (torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda(), torch.from_numpy(spans).cuda())


def _values_dtype(t: torch.Tensor, name: str) -> tuple[torch.Tensor, int]:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype not in (torch.float32, torch.float64):
        t = t.float()
    return t.contiguous(), (1 if t.dtype == torch.float64 else 0)


def _sized_write(fn, device) -> bytes:
    length = C.c_int64()
    _check(fn(None, 0, C.byref(length)))
    out = torch.empty(length.value, dtype=torch.uint8, device=device)
    _check(fn(_p(out), length.value, C.byref(length)))
    return bytes(out.cpu().numpy())


def codes_csv(ctx: Context, codes: torch.Tensor, first_id: int = 0, ids: Optional[Sequence[str]] = None,
              id_prefix: Optional[str] = None) -> bytes:
    """write_codes_csv (io.cpp:312-330) of codes [rows, k] (float32 or float64, device); ids
    id_prefix + (first_id + row), or the given strings written verbatim (the reference's
    `ids` argument)."""
    codes, dtype = _values_dtype(codes, "codes")
    rows, k = codes.shape
    ib, isp = _id_args(ids, rows)
    ctx.bind_stream()
    lib = _lib.lib()
    pre = id_prefix.encode() if id_prefix else None
    return _sized_write(lambda out, cap, ln: lib.hc_codes_csv_write_ids(
        ctx.h, _p(codes), dtype, rows, k, _p(ib) if ib is not None else None, _p(isp) if isp is not None else None,
        pre, first_id, out, cap, ln), codes.device)


def spectra_csv(ctx: Context, values: torch.Tensor, wavelengths: np.ndarray, ids: Optional[Sequence[str]] = None
                ) -> bytes:
    """write_spectra_csv (io.cpp:165-186) of curves [rows, n] on the canonical grid (the n
    `wavelengths`), %.9g; ids = None writes no id column (the reference's empty ids)."""
    values, dtype = _values_dtype(values, "values")
    rows, n = values.shape
    wl = np.ascontiguousarray(wavelengths, dtype=np.float64)
    if wl.size != n:
        raise ValueError("spectra_csv: one wavelength per column")
    ib, isp = _id_args(ids, rows)
    ctx.bind_stream()
    lib = _lib.lib()
    return _sized_write(lambda out, cap, ln: lib.hc_spectra_csv_write(
        ctx.h, _p(values), dtype, rows, n, _np_ptr(wl), 1 if ids is not None else 0,
        _p(ib) if ib is not None else None, _p(isp) if isp is not None else None, None, 0, out, cap, ln),
        values.device)


def _device_text(data: Optional[bytes], text: Optional[torch.Tensor]) -> torch.Tensor:
    if text is not None:
        return text
    return torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda() if data else \
        torch.empty(0, dtype=torch.uint8, device="cuda")


def read_spectra_csv(ctx: Context, data: Optional[bytes], text: Optional[torch.Tensor] = None
                     ) -> tuple[np.ndarray, Optional[list], torch.Tensor, Optional[torch.Tensor]]:
    """read_spectra_csv (io.cpp:119-163) on the device: (wavelengths, ids or None, values
    [rows, m] float64 CUDA tensor, id spans [rows, 2] CUDA tensor or None)."""
    text = _device_text(data, text)
    lib = _lib.lib()
    has_id, m, rows = C.c_int(), C.c_int(), C.c_int64()
    ctx.bind_stream()
    n = text.numel()
    _check(lib.hc_spectra_csv_read(ctx.h, _p(text), n, C.byref(has_id), None, 0, C.byref(m), C.byref(rows), None,
                                   None, 0))
    wl = np.zeros(m.value, np.float64)
    vals = torch.empty(rows.value, m.value, dtype=torch.float64, device="cuda")
    spans = torch.empty(rows.value, 2, dtype=torch.int64, device="cuda")
    _check(lib.hc_spectra_csv_read(ctx.h, _p(text), n, C.byref(has_id), _np_ptr(wl), m.value, C.byref(m),
                                   C.byref(rows), _p(vals), _p(spans) if has_id.value else None, rows.value))
    ids = None
    if has_id.value:
        raw = data if data is not None else bytes(text.cpu().numpy())
        ids = [raw[a:a + ln].decode() for a, ln in spans.cpu().numpy().tolist()]
    return wl, ids, vals, (spans if has_id.value else None)


def encode_resampled(codec: "Codec", wavelengths: np.ndarray, values: torch.Tensor, zero_outside: bool = True
                     ) -> torch.Tensor:
    """resample (spectrum.cpp:60-98) of curves [rows, m] given on `wavelengths` onto the
    codec's canonical grid, then encode (codec.cpp:36-46), all in fp64 as the reference:
    codes [rows, k] float64, bit-identical to the reference's."""
    values = _cuda(values, torch.float64, "values")
    wl = np.ascontiguousarray(wavelengths, dtype=np.float64)
    rows, m = values.shape if values.dim() == 2 else (0, wl.size)
    if m != wl.size:
        raise ValueError("resample: grid/value size mismatch")
    lo, step = grid(codec.n)
    codes = torch.empty(rows, codec.k, dtype=torch.float64, device=values.device)
    codec.ctx.bind_stream()
    _check(_lib.lib().hc_encode_resampled_f64(codec.h, _np_ptr(wl), wl.size, _p(values), rows, lo, step,
                                              1 if zero_outside else 0, _p(codes)))
    return codes


def encode_f64(codec: "Codec", spectra: torch.Tensor) -> torch.Tensor:
    """encode (codec.cpp:36-46) of curves [rows, n] on the canonical grid in fp64 with the
    reference's summation order: codes [rows, k] float64, bit-identical to the reference."""
    spectra = _cuda(spectra, torch.float64, "spectra")
    rows, n = spectra.shape
    if n != codec.n:
        raise ValueError("encode: spectrum size does not match the grid")
    out = torch.empty(rows, codec.k, dtype=torch.float64, device=spectra.device)
    codec.ctx.bind_stream()
    _check(_lib.lib().hc_encode_f64(codec.h, _p(spectra), rows, _p(out)))
    return out


def decode_f64(codec: "Codec", codes: torch.Tensor) -> torch.Tensor:
    """decode (codec.cpp:52-71) in fp64 as the reference: spectra [rows, n] float64; a
    negative (or NaN) code entry raises ArithmeticError (the reference's std::domain_error)."""
    codes = _cuda(codes, torch.float64, "codes")
    rows, k = codes.shape
    if k != codec.k:
        raise ValueError("decode: code dimension mismatch")
    out = torch.empty(rows, codec.n, dtype=torch.float64, device=codes.device)
    codec.ctx.bind_stream()
    first = C.c_int64()
    _check(_lib.lib().hc_decode_f64(codec.h, _p(codes), rows, _p(out), C.byref(first)))
    return out


def load_codec_weights(path) -> dict:
    """load_codec_weights (io.cpp:370-393): the reference's codec weight file (JSON) as
    {k, n, beta, raw_enc [k, n], raw_dec [n, k], meta}; ValueError (the reference's
    FormatError) for a file that is not a valid codec weights file.  Python's float parsing
    is correctly rounded, as the reference's strtod is, so the doubles are identical."""
    import json as _json

    try:
        with open(path, "r") as f:
            j = _json.load(f)
    except OSError as e:
        raise ValueError(f"{path}: cannot open for reading") from e
    except _json.JSONDecodeError as e:
        raise ValueError(f"{path}: JSON parse error: {e}") from e
    try:
        if j["format"] != "codec-weights":
            raise ValueError(f"{path}: not a codec weights file")
        k, n, beta = int(j["k"]), int(j["n"]), float(j["beta"])
        re_ = np.asarray(j["raw_enc"], dtype=np.float64)
        rd = np.asarray(j["raw_dec"], dtype=np.float64)
        meta = j.get("meta")
    except (KeyError, TypeError) as e:
        raise ValueError(f"{path}: bad codec weights: {e}") from e
    # validate (codec.cpp:111-135)
    if k <= 0 or k % 3:
        raise ValueError(f"{path}: codec weights: k must be a positive multiple of 3")
    if n not in (47, 81):
        raise ValueError(f"{path}: codec weights: n must match the canonical grid")
    if not beta > 0.0:
        raise ValueError(f"{path}: codec weights: beta must be positive")
    if re_.size != k * n or rd.size != n * k:
        raise ValueError(f"{path}: codec weights: parameter array size mismatch")
    if not (np.isfinite(re_).all() and np.isfinite(rd).all()):
        raise ValueError(f"{path}: codec weights: non-finite entry")
    return {"k": k, "n": n, "beta": beta, "raw_enc": re_.reshape(k, n), "raw_dec": rd.reshape(n, k), "meta": meta}


def read_raw_image(path, device: str = "cuda") -> torch.Tensor:
    """read_raw_image (io.cpp:450-476): an HCF1 channel image as a float32 tensor [h, w, c]
    (row-major y, x, channel as ChannelImage), moved to `device` — the payload goes from the
    file to pinned memory and on to the GPU in one copy.  ValueError (FormatError) with the
    reference's causes for a bad magic, truncated header, implausible dimensions or
    truncated pixel data."""
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise ValueError(f"{path}: cannot open for reading") from e
    if len(raw) < 4 or raw[:4] != b"HCF1":
        raise ValueError(f"{path}: bad magic (expected HCF1)")
    if len(raw) < 16:
        raise ValueError(f"{path}: truncated header")
    w, h, c = (int(x) for x in np.frombuffer(raw, np.uint32, 3, 4).astype(np.int64))
    w, h, c = (x - (1 << 32) if x >= 1 << 31 else x for x in (w, h, c))  # static_cast<int>(uint32)
    if w <= 0 or h <= 0 or c <= 0 or w > 1 << 16 or h > 1 << 16 or c > 1024:
        raise ValueError(f"{path}: implausible image dimensions")
    count = w * h * c
    if len(raw) - 16 < 4 * count:
        raise ValueError(f"{path}: truncated pixel data")
    t = torch.frombuffer(bytearray(raw[16:16 + 4 * count]), dtype=torch.float32).reshape(h, w, c)
    if device == "cpu":
        return t
    return t.pin_memory().to(device, non_blocking=True)


def write_raw_image(path, image: torch.Tensor) -> None:
    """write_raw_image (io.cpp:478-492) of a float32 image [h, w, c] (any device)."""
    if image.dim() != 3 or image.numel() == 0:
        raise ValueError(f"{path}: image dimensions do not match data size")
    h, w, c = image.shape
    data = image.detach().to("cpu", torch.float32).contiguous().numpy().tobytes()
    with open(path, "wb") as f:
        f.write(b"HCF1" + np.array([w, h, c], np.uint32).tobytes() + data)


class Upsampler:
    """The reference's RGB -> code upsampler (upsampler.hpp:13-50): fp64, 3 -> hidden -> hidden
    -> k, SiLU, identity head; `forward` = upsample (clamp=True) / upsample_raw (clamp=False)
    on the GPU in the reference's summation order (~1e-15 relative: SiLU uses CUDA's exp).
    `w` holds w1 [hidden, 3], b1, w2 [hidden, hidden], b2, w3 [k, hidden], b3 (arrays)."""

    KEYS = ("w1", "b1", "w2", "b2", "w3", "b3")

    def __init__(self, ctx: Context, w: dict):
        arrs = [np.ascontiguousarray(w[n], dtype=np.float64).reshape(-1) for n in self.KEYS]
        hidden = arrs[1].size
        k = arrs[5].size
        self.ctx, self.k, self.hidden = ctx, k, hidden
        h = C.c_void_p()
        _check(_lib.lib().hc_upsampler_create(ctx.h, k, hidden, *[_np_ptr(a) for a in arrs], C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().hc_upsampler_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @classmethod
    def from_weights_file(cls, ctx: Context, path) -> "Upsampler":
        """An upsampler from the reference's weight file (load_upsampler_weights, io.cpp:405-431)."""
        return cls(ctx, load_upsampler_weights(path))

    def forward(self, rgb: torch.Tensor, clamp: bool = True) -> tuple[torch.Tensor, int]:
        """codes [P, k] float64 for linear-sRGB rows [P, 3] (float64 CUDA), and the number of
        clamped entries (the reference's telemetry)."""
        rgb = _cuda(rgb, torch.float64, "rgb")
        P = rgb.shape[0]
        codes = torch.empty(P, self.k, dtype=torch.float64, device=rgb.device)
        n = C.c_uint64(0)
        self.ctx.bind_stream()
        _check(_lib.lib().hc_upsample_f64(self.h, _p(rgb), P, 1 if clamp else 0, _p(codes), C.byref(n)))
        return codes, int(n.value)


LOSS_WEIGHTS = (0.5, 0.75, 1.0, 0.5, 0.0)  # LossWeights defaults {e2e, rec, code, col, alg} (trainer.hpp:13-19)
LOSS_NAMES = ("e2e", "rec", "code", "col", "alg", "total")


def codec_train_grad(ctx: Context, raw_enc: np.ndarray, raw_dec: np.ndarray, beta: float, refl: torch.Tensor,
                     illum: torch.Tensor, loss_weights=LOSS_WEIGHTS, grads: bool = True):
    """compute_losses + gradients (trainer.cpp:108-373) of raw codec weights over a batch of
    (reflectance, illumination) pairs [m, n] (float64 CUDA tensors), on the GPU, bit-identical
    to the reference: ({loss name: value}, g_raw_enc [k, n], g_raw_dec [n, k]) — the
    gradients are None with grads=False."""
    re_ = np.ascontiguousarray(raw_enc, dtype=np.float64)
    rd = np.ascontiguousarray(raw_dec, dtype=np.float64)
    k, n = re_.shape
    refl = _cuda(refl, torch.float64, "refl")
    illum = _cuda(illum, torch.float64, "illum")
    if refl.shape != illum.shape or refl.dim() != 2 or refl.shape[1] != n:
        raise ValueError("batch: reflectance/illumination size mismatch")
    lw = np.ascontiguousarray(loss_weights, dtype=np.float64)
    cmf = np.ascontiguousarray(cmf_matrix(n), dtype=np.float64)
    ge = np.zeros((k, n), np.float64) if grads else None
    gd = np.zeros((n, k), np.float64) if grads else None
    losses = np.zeros(6, np.float64)
    ctx.bind_stream()
    _check(_lib.lib().hc_codec_train_grad(ctx.h, k, n, float(beta), _np_ptr(re_), _np_ptr(rd), _np_ptr(cmf),
                                          grid(n)[1], _p(refl), _p(illum), refl.shape[0], _np_ptr(lw),
                                          _np_ptr(ge) if grads else None, _np_ptr(gd) if grads else None,
                                          _np_ptr(losses)))
    return dict(zip(LOSS_NAMES, losses.tolist())), ge, gd


def adam_step(ctx: Context, params: torch.Tensor, grad: torch.Tensor, m1: torch.Tensor, v1: torch.Tensor, lr: float,
              step: int) -> None:
    """adam_step (trainer.cpp:399-411) in place on float64 CUDA tensors, bit-identical."""
    for t, name in ((params, "params"), (grad, "grad"), (m1, "m"), (v1, "v")):
        _cuda(t, torch.float64, name)
        if not t.is_contiguous() or t.numel() != params.numel():
            raise ValueError("adam: parameter / state size mismatch")
    ctx.bind_stream()
    _check(_lib.lib().hc_adam_step(ctx.h, _p(params), _p(grad), _p(m1), _p(v1), params.numel(), float(lr), int(step)))


def upsample_train_grad(ctx: Context, w: dict, codec: "Codec", rgb: torch.Tensor, target: torch.Tensor,
                        lambda_maxabs: float = 0.3, lambda_color: float = 0.05, grads: bool = True):
    """upsample_loss + upsample_gradients (upsampler.cpp:207-369) on the GPU: the network `w`
    (Upsampler's dict layout), the frozen `codec` (its fp64 effective decoder), a batch of rgb
    [B, 3] and target codes [B, k] (float64 CUDA).  Returns ({latent_mse, latent_maxabs,
    color, total}, {w1: grad, ...} or None); within ~1e-12 of the reference (exp, cbrt)."""
    from .colorimetry import cmf_table, white_xyz

    arrs = [np.ascontiguousarray(w[n], dtype=np.float64).reshape(-1) for n in Upsampler.KEYS]
    hidden, k = arrs[1].size, arrs[5].size
    rgb = _cuda(rgb, torch.float64, "rgb")
    target = _cuda(target, torch.float64, "target")
    n = codec.n
    t = cmf_table(n)
    ys = [float(a) * float(b) for a, b in zip(t["ybar"], t["d65"])]
    norm = 0.0
    for v in ys:  # CmfTable (colorimetry.cpp:51-59), in the reference's order
        norm += v
    scale = 100.0 / norm
    wxyz = np.ascontiguousarray(np.stack([scale * t[c] * t["d65"] for c in ("xbar", "ybar", "zbar")]), np.float64)
    white = np.ascontiguousarray(white_xyz(n), dtype=np.float64)
    dec = np.ascontiguousarray(codec.effective_f64()[1], dtype=np.float64)
    ng = sum(a.size for a in arrs)
    g = np.zeros(ng) if grads else None
    losses = np.zeros(4)
    ctx.bind_stream()
    _check(_lib.lib().hc_upsample_train_grad(ctx.h, k, hidden, *[_np_ptr(a) for a in arrs], n, _np_ptr(dec),
                                             _np_ptr(wxyz), _np_ptr(white), _p(rgb), _p(target), rgb.shape[0],
                                             float(lambda_maxabs), float(lambda_color), _np_ptr(losses),
                                             _np_ptr(g) if grads else None))
    names = ("latent_mse", "latent_maxabs", "color", "total")
    out = None
    if grads:
        out, o = {}, 0
        for name, a in zip(Upsampler.KEYS, arrs):
            out[name] = g[o:o + a.size].reshape(np.asarray(w[name]).shape)
            o += a.size
    return dict(zip(names, losses.tolist())), out


def adamw_step(ctx: Context, params: torch.Tensor, grad: torch.Tensor, m1: torch.Tensor, v1: torch.Tensor, lr: float,
               weight_decay: float, step: int) -> None:
    """adamw_step (upsampler.cpp:378-391) in place on float64 CUDA tensors."""
    for t_, name in ((params, "params"), (grad, "grad"), (m1, "m"), (v1, "v")):
        _cuda(t_, torch.float64, name)
        if not t_.is_contiguous() or t_.numel() != params.numel():
            raise ValueError("adamw: parameter / state size mismatch")
    ctx.bind_stream()
    _check(_lib.lib().hc_adamw_step(ctx.h, _p(params), _p(grad), _p(m1), _p(v1), params.numel(), float(lr),
                                    float(weight_decay), int(step)))


def load_upsampler_weights(path) -> dict:
    """load_upsampler_weights (io.cpp:405-431): {k, hidden, w1 [h, 3], b1, w2 [h, h], b2, w3 [k, h],
    b3, meta}; ValueError (FormatError) for a file that is not valid upsampler weights."""
    import json as _json

    try:
        with open(path, "r") as f:
            j = _json.load(f)
    except OSError as e:
        raise ValueError(f"{path}: cannot open for reading") from e
    except _json.JSONDecodeError as e:
        raise ValueError(f"{path}: JSON parse error: {e}") from e
    try:
        if j["format"] != "upsampler-weights":
            raise ValueError(f"{path}: not an upsampler weights file")
        k, h = int(j["k"]), int(j["hidden"])
        arr = {n: np.asarray(j[n], dtype=np.float64) for n in ("w1", "b1", "w2", "b2", "w3", "b3")}
    except (KeyError, TypeError) as e:
        raise ValueError(f"{path}: bad upsampler weights: {e}") from e
    shapes = {"w1": h * 3, "b1": h, "w2": h * h, "b2": h, "w3": k * h, "b3": k}  # validate (upsampler.cpp:130-144)
    if k <= 0 or h <= 0 or any(arr[n].size != sz for n, sz in shapes.items()):
        raise ValueError(f"{path}: upsampler: weight shapes do not match k / hidden")
    if not all(np.isfinite(a).all() for a in arr.values()):
        raise ValueError(f"{path}: upsampler: weights must be finite")
    return {"k": k, "hidden": h, "w1": arr["w1"].reshape(h, 3), "b1": arr["b1"], "w2": arr["w2"].reshape(h, h),
            "b2": arr["b2"], "w3": arr["w3"].reshape(k, h), "b3": arr["b3"], "meta": j.get("meta")}


def encode_tool(codec: "Codec", spectra_csv_bytes: bytes) -> bytes:
    """The reference's `encode` tool (tools/main.cpp:285-308, without its manifest) on the
    device: spectra CSV -> resample + encode (fp64) -> codes CSV (%.17g).  Byte-identical
    to the reference; ids come from the input's id column, else "row" + r."""
    ctx = codec.ctx
    text = _device_text(spectra_csv_bytes, None)
    wl, _, vals, spans = read_spectra_csv(ctx, spectra_csv_bytes, text=text)
    codes = encode_resampled(codec, wl, vals, zero_outside=True)
    rows = codes.shape[0]
    lib = _lib.lib()
    ctx.bind_stream()
    if spans is not None:
        return _sized_write(lambda out, cap, ln: lib.hc_codes_csv_write_ids(
            ctx.h, _p(codes), 1, rows, codec.k, _p(text), _p(spans), None, 0, out, cap, ln), codes.device)
    return _sized_write(lambda out, cap, ln: lib.hc_codes_csv_write_ids(
        ctx.h, _p(codes), 1, rows, codec.k, None, None, b"row", 0, out, cap, ln), codes.device)


def decode_tool(codec: "Codec", codes_csv_bytes: bytes) -> bytes:
    """The reference's `decode` tool (tools/main.cpp:310-328, without its manifest) on the
    device: codes CSV -> decode (fp64) -> spectra CSV (%.9g), ids passed through."""
    ctx = codec.ctx
    text = _device_text(codes_csv_bytes, None)
    lib = _lib.lib()
    k, rows = C.c_int(), C.c_int64()
    ctx.bind_stream()
    _check(lib.hc_codes_csv_read(ctx.h, _p(text), text.numel(), C.byref(k), C.byref(rows), None, None, 0))
    codes = torch.empty(rows.value, k.value, dtype=torch.float64, device="cuda")
    spans = torch.empty(rows.value, 2, dtype=torch.int64, device="cuda")
    _check(lib.hc_codes_csv_read(ctx.h, _p(text), text.numel(), C.byref(k), C.byref(rows), _p(codes), _p(spans),
                                 rows.value))
    spectra = decode_f64(codec, codes)
    wl = wavelengths(codec.n)
    return _sized_write(lambda out, cap, ln: lib.hc_spectra_csv_write(
        ctx.h, _p(spectra), 1, rows.value, codec.n, _np_ptr(wl), 1, _p(text), _p(spans), None, 0, out, cap, ln),
        spectra.device)


def read_codes_csv(ctx: Context, data: bytes, text: Optional[torch.Tensor] = None) -> tuple[list, torch.Tensor]:
    """read_codes_csv (io.cpp:267-310) of a file image, parsed on the device: (ids, codes [rows, k]
    float64 CUDA tensor).  `text` may be the file already resident as a uint8 CUDA tensor."""
    if text is None:
        text = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda() if data else torch.empty(0, dtype=torch.uint8,
                                                                                                      device="cuda")
    k, rows = C.c_int(), C.c_int64()
    ctx.bind_stream()
    n = text.numel()
    _check(_lib.lib().hc_codes_csv_read(ctx.h, _p(text), n, C.byref(k), C.byref(rows), None, None, 0))
    codes = torch.empty(rows.value, k.value, dtype=torch.float64, device="cuda")
    spans = torch.empty(rows.value, 2, dtype=torch.int64, device="cuda")
    _check(_lib.lib().hc_codes_csv_read(ctx.h, _p(text), n, C.byref(k), C.byref(rows), _p(codes), _p(spans),
                                        rows.value))
    raw = data if data is not None else bytes(text.cpu().numpy())
    ids = [raw[a:a + ln].decode() for a, ln in spans.cpu().numpy().tolist()]
    return ids, codes


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


class CodeMLP:
    """The BASELINE.json RGB -> code MLP (3 -> 64 -> 64 -> 6, ReLU, softplus head) in bf16 on the
    tensor cores (tcgen05) — config 5a; the reference's own fp64 SiLU network is `Upsampler`."""

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


def spin(ctx: Context, cycles: int) -> None:
    """Keep the bound stream busy for `cycles` SM clocks (measurement helper, hc_spin)."""
    ctx.bind_stream()
    _check(_lib.lib().hc_spin(ctx.h, int(cycles)))


def flush_l2(ctx: Context, buf: torch.Tensor) -> None:
    ctx.bind_stream()
    _check(_lib.lib().hc_flush_l2(ctx.h, _p(buf), buf.numel() * buf.element_size()))
