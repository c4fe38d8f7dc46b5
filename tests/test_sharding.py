"""Multi-rank path on CPU: world_size 2 over gloo.  Each rank generates its row
band of a G-buffer from global pixel indices, shades it with the oracle (the
checker stands in for the GPU kernel here), and the bands are gathered to rank 0;
the result must be bit-identical to one process shading the whole image."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_18741_b200 import synth
from paper_2602_18741_b200.colorimetry import cmf_matrix, grid
from paper_2602_18741_b200.sharding import gather_rows, pair_range, reduce_loss, row_band

W, H, L, K, SEED = 37, 23, 8, 6, 5


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shade_rows(orc, first: int, P: int) -> np.ndarray:
    E, D = synth.codec_weights(SEED, K, 81)
    pal = synth.palette(SEED, 16, 81)
    lts = synth.lights(SEED, L, 81)
    pc = np.zeros((16, K), np.float32)
    lc = np.zeros((L, K), np.float32)
    orc.orc_asset_codes(E, K, 81, pal, 16, pc)
    orc.orc_asset_codes(E, K, 81, lts, L, lc)
    idx, cosv = synth.gbuffer_np(SEED, first, P, L, 16)
    rgb = np.zeros((P, 3), np.float32)
    orc.orc_shade_latent(D, K, 81, cmf_matrix(81), grid(81)[1], pc, lc, L, idx, np.ascontiguousarray(cosv), P,
                         None, None, None, rgb)
    return rgb


def _worker(rank: int, world: int, port: int, out_path: str):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    orc = oracle.oracle()
    band = row_band(rank, world, H, W)
    local = torch.from_numpy(_shade_rows(orc, band.first_pixel, band.pixels))
    img = gather_rows(local, band, H)
    if rank == 0:
        np.save(out_path, img.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_row_bands_partition_the_image():
    for world in (1, 2, 3, 4, 8):
        bands = [row_band(r, world, H, W) for r in range(world)]
        assert bands[0].row0 == 0 and bands[-1].row1 == H
        assert all(a.row1 == b.row0 for a, b in zip(bands, bands[1:]))
        assert max(b.rows for b in bands) - min(b.rows for b in bands) <= 1
    with pytest.raises(ValueError):
        row_band(2, 2, H, W)


def test_inputs_do_not_depend_on_sharding():
    idx_all, cos_all = synth.gbuffer_np(SEED, 0, W * H, L, 16)
    b = row_band(1, 3, H, W)
    idx_b, cos_b = synth.gbuffer_np(SEED, b.first_pixel, b.pixels, L, 16)
    assert np.array_equal(idx_b, idx_all[b.first_pixel:b.first_pixel + b.pixels])
    assert np.array_equal(cos_b, cos_all[b.first_pixel:b.first_pixel + b.pixels])


def test_two_rank_gloo_gather_matches_single_process(tmp_path):
    import oracle

    out = str(tmp_path / "img.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    want = _shade_rows(oracle.oracle(), 0, W * H)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


# ---- config 5b across ranks: pairs split by index range, fp64 partial sums all-reduced
PAIRS = 1001


def _loss_pairs(first: int, count: int):
    a = synth.gm_spectra_ctr(SEED, "loss.a", first, count, 81)
    b = synth.gm_spectra_ctr(SEED, "loss.b", first, count, 81)
    return np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32)


def _loss_worker(rank: int, world: int, port: int, out_path: str):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    orc = oracle.oracle()
    E, D = synth.codec_weights(SEED, K, 81)
    first, count = pair_range(rank, world, PAIRS)
    a, b = _loss_pairs(first, count)
    partial = torch.tensor([orc.orc_hadamard_loss(E, D, K, 81, a, b, count)], dtype=torch.float64)
    total = reduce_loss(partial)
    np.save(out_path + f".{rank}.npy", total.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_pair_ranges_partition_the_pairs():
    for world in (1, 2, 3, 8):
        rs = [pair_range(r, world, PAIRS) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][0] + rs[-1][1] == PAIRS
        assert all(a[0] + a[1] == b[0] for a, b in zip(rs, rs[1:]))


def test_two_rank_gloo_loss_allreduce_matches_single_process(tmp_path):
    import oracle

    out = str(tmp_path / "loss")
    mp.spawn(_loss_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    E, D = synth.codec_weights(SEED, K, 81)
    a, b = _loss_pairs(0, PAIRS)
    want = oracle.oracle().orc_hadamard_loss(E, D, K, 81, a, b, PAIRS)
    got = [float(np.load(out + f".{rank}.npy")[0]) for rank in range(2)]
    assert got[0] == got[1]  # every rank holds the same total
    assert got[0] == pytest.approx(want, rel=1e-12)  # two fp64 partials vs one sequential sum
