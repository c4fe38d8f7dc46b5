"""Row-band sharding across GPUs (one process per GPU, torch.distributed).

The per-pixel path has no exchange step: every pixel (spectrum, pair, texel) is
independent.  An image is cut into contiguous row bands, one per
rank; each rank generates its own band of inputs from GLOBAL element indices
(counter streams, so values do not depend on the number of ranks), shades it on
its GPU, and — only when the caller wants the image on one rank — the linear-sRGB
(or XYZ) bands are gathered to rank 0 with one collective (NCCL over NVLink on
the B200 box, gloo in the CPU tests), or not gathered at all: with a `PeerFrame` every
rank's shade kernel stores its band straight into rank 0's frame through NVLink peer memory
(CUDA IPC mapping), so compute and gather are one kernel.  Nothing else crosses a GPU boundary.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Band:
    rank: int
    world: int
    row0: int
    row1: int
    width: int

    @property
    def rows(self) -> int:
        return self.row1 - self.row0

    @property
    def first_pixel(self) -> int:
        return self.row0 * self.width

    @property
    def pixels(self) -> int:
        return self.rows * self.width


def row_band(rank: int, world: int, height: int, width: int) -> Band:
    """Contiguous rows [row0, row1) of rank `rank`; sizes differ by at most one row.  The split
    is the library's (hc_row_band), so Python ranks and the C++ device group agree."""
    import ctypes as C

    from . import _lib

    if not (0 <= rank < world) or height < 0:
        raise ValueError("row_band: bad rank / size")
    r0, n = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().hc_row_band(rank, world, height, C.byref(r0), C.byref(n)))
    return Band(rank, world, r0.value, r0.value + n.value, width)


def gather_rows(local: torch.Tensor, band: Band, height: int, dst: int = 0) -> torch.Tensor | None:
    """Gather every rank's [band.pixels, C] rows into the [height * width, C] image on `dst`.

    Bands may differ by one row, so ranks pad to the largest band for the
    collective (torch.distributed.gather needs equal shapes) and `dst` trims.
    Returns the image on `dst`, None elsewhere."""
    world = band.world
    if world == 1:
        return local
    base, extra = divmod(height, world)
    max_rows = base + (1 if extra else 0)
    C = local.shape[1]
    padded = local.new_zeros((max_rows * band.width, C))
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)] if band.rank == dst else None
    dist.gather(padded, parts, dst=dst)
    if band.rank != dst:
        return None
    out = []
    for r in range(world):
        b = row_band(r, world, height, band.width)
        out.append(parts[r][: b.pixels])
    return torch.cat(out, dim=0)


def pair_range(rank: int, world: int, pairs: int) -> tuple[int, int]:
    """Contiguous index range [first, first + count) of rank `rank` over `pairs` items (spectra, pairs,
    texels): the row-band split with one item per row."""
    b = row_band(rank, world, pairs, 1)
    return b.first_pixel, b.pixels


def reduce_loss(partial: torch.Tensor) -> torch.Tensor:
    """The near-multiplicativity loss over sharded pairs: every rank's fp64 partial sum
    (`Codec.hadamard_loss` on its own pairs) is summed over the ranks by one all-reduce -- the only
    exchange step this path has.  Returns the total on every rank (in place)."""
    if partial.dtype != torch.float64:
        raise TypeError("reduce_loss: the partial sums are fp64")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM)
    return partial


class _DevicePointer:
    """A raw device pointer as a __cuda_array_interface__ object (float32, C-contiguous)."""

    def __init__(self, ptr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerFrame:
    """The [height * width, channels] float32 image on rank `dst`'s GPU, mapped into every rank.

    `dst` allocates the frame (hc_ipc_alloc) and broadcasts its CUDA IPC handle; the other ranks map
    it (hc_ipc_open enables peer access from their own device).  `local` is this rank's band of rows
    as a CUDA tensor — peer memory on every rank but `dst` — to be passed as the `out=` tensor of
    `Codec.shade_latent`, whose kernel then stores the band straight into `dst`'s frame over NVLink:
    no gather step, no staging copy.  After a `dist.barrier()` that follows every rank's stream
    synchronisation, `image` (on `dst`) holds the assembled frame.  Works with any backend that can
    broadcast a Python object (NCCL on the GPU box; gloo in the one-GPU two-process test)."""

    def __init__(self, band: Band, height: int, channels: int = 3, device: int | None = None, dst: int = 0):
        import ctypes as C

        from . import _lib

        self.band, self.height, self.channels, self.dst = band, height, channels, dst
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.owner = band.rank == dst
        nbytes = height * band.width * channels * 4
        ptr = C.c_void_p()
        handle = (C.c_ubyte * 64)()
        if self.owner:
            _lib.check(_lib.lib().hc_ipc_alloc(self.device, nbytes, C.byref(ptr), handle))
        box = [bytes(handle) if self.owner else None]
        if band.world > 1:
            dist.broadcast_object_list(box, src=dst)
        if not self.owner:
            handle = (C.c_ubyte * 64).from_buffer_copy(box[0])
            _lib.check(_lib.lib().hc_ipc_open(self.device, handle, C.byref(ptr)))
        self.ptr = ptr.value
        px = height * band.width
        # the pointer belongs to dst's device; torch only needs a CUDA tensor around it
        self.image = torch.as_tensor(_DevicePointer(self.ptr, (px, channels)), device="cuda")
        self.local = self.image[band.first_pixel:band.first_pixel + band.pixels]

    def close(self) -> None:
        from . import _lib

        if getattr(self, "ptr", None):
            self.image = self.local = None
            if self.owner:
                _lib.check(_lib.lib().hc_ipc_free(self.device, self.ptr))
            else:
                _lib.check(_lib.lib().hc_ipc_close(self.device, self.ptr))
            self.ptr = None
