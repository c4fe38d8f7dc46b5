"""Row-band sharding across GPUs (one process per GPU, torch.distributed).

The per-pixel path has no exchange step: every pixel (spectrum, pair, texel) is
independent.  An image is cut into contiguous row bands, one per
rank; each rank generates its own band of inputs from GLOBAL element indices
(counter streams, so values do not depend on the number of ranks), shades it on
its GPU, and — only when the caller wants the image on one rank — the linear-sRGB
(or XYZ) bands are gathered to rank 0 with one collective (NCCL over NVLink on
the B200 box, gloo in the CPU tests).  Nothing else crosses a GPU boundary.
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
