"""Several GPUs from one process (hc_group_*) and the multi-process row-band path
on the GPU.  The box has one B200, so the multi-device code runs with the same device listed
twice (host and peer gathers; NCCL needs distinct devices and is exercised with one device),
and the two-rank test runs both ranks' kernels on cuda:0 with a gloo gather of the bands — the
ranks never wait on each other's kernels.  Results must be bit-identical to one process
shading the whole frame."""
import os
import socket

import numpy as np
import pytest

from paper_2602_18741_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED, K, L, W, H = 11, 6, 8, 256, 67


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


def _scene(api, ctx):
    E, D = synth.codec_weights(SEED, K, 81)
    codec = api.Codec(ctx, E, D)
    pal_codes = codec.encode(torch.from_numpy(synth.palette(SEED, 256, 81)).cuda()).cpu().numpy()
    light_codes = codec.encode(torch.from_numpy(synth.lights(SEED, L, 81)).cuda()).cpu().numpy()
    idx, cosv = synth.gbuffer_np(SEED, 0, W * H, L, 256)
    return E, D, codec, pal_codes, light_codes, np.ascontiguousarray(idx), np.ascontiguousarray(cosv)


@pytest.fixture(scope="module")
def reference_frame(api):
    ctx = api.Context(0)
    E, D, codec, pc, lc, idx, cosv = _scene(api, ctx)
    xyz, rgb = np.zeros((W * H, 3), np.float32), np.zeros((W * H, 3), np.float32)
    codec.shade_latent_host(pc, lc, idx, cosv, xyz, rgb)
    return E, D, pc, lc, idx, cosv, xyz, rgb


@pytest.mark.parametrize("devices,gather", [([0], "host"), ([0], "peer"), ([0], "nccl"), ([0, 0], "host"),
                                            ([0, 0], "peer"), ([0, 0, 0], "peer"), ([0], "fused"),
                                            ([0, 0], "fused"), ([0, 0, 0, 0, 0], "fused")])
def test_group_matches_single_context(api, reference_frame, devices, gather):
    E, D, pc, lc, idx, cosv, xyz_ref, rgb_ref = reference_frame
    g = api.Group(devices, gather)
    g.set_codec(E, D)
    xyz, rgb = np.zeros_like(xyz_ref), np.zeros_like(rgb_ref)
    g.shade_latent_host(pc, lc, idx, cosv, W, H, xyz, rgb)
    assert np.array_equal(xyz, xyz_ref) and np.array_equal(rgb, rgb_ref)
    rgb2 = np.zeros_like(rgb_ref)
    g.shade_latent_host(pc, lc, idx, cosv, W, H, None, rgb2)  # outputs may be skipped
    assert np.array_equal(rgb2, rgb_ref)


def test_group_nccl_needs_distinct_devices(api):
    from paper_2602_18741_b200 import _lib

    assert api.Group.nccl_version() > 0  # the NCCL PyTorch bundles, loaded at run time
    with pytest.raises(_lib.HcError):
        api.Group([0, 0], "nccl")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank: int, world: int, port: int, out_path: str):
    import torch.distributed as dist

    from paper_2602_18741_b200 import api as a
    from paper_2602_18741_b200.sharding import gather_rows, row_band

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = a.Context(0)
    E, D = synth.codec_weights(SEED, K, 81)
    codec = a.Codec(ctx, E, D)
    pal = codec.encode(torch.from_numpy(synth.palette(SEED, 256, 81)).cuda())
    lc = codec.encode(torch.from_numpy(synth.lights(SEED, L, 81)).cuda()).cpu().numpy()
    band = row_band(rank, world, H, W)
    idx, cosv = a.synth_gbuffer(ctx, SEED, band.first_pixel, band.pixels, L, 256)  # global pixel indices
    out = codec.shade_latent(pal, lc, idx, cosv)
    img = gather_rows(out["rgb"].cpu(), band, H)
    if rank == 0:
        np.save(out_path, img.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _rank_fused(rank: int, world: int, port: int, out_path: str):
    """The fused gather across processes: every rank's kernel stores its band into rank 0's frame
    (CUDA IPC mapping; on this one-GPU box both ranks use cuda:0, on a node each its own GPU)."""
    import torch.distributed as dist

    from paper_2602_18741_b200 import api as a
    from paper_2602_18741_b200.sharding import PeerFrame, row_band

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = a.Context(0)
    E, D = synth.codec_weights(SEED, K, 81)
    codec = a.Codec(ctx, E, D)
    pal = codec.encode(torch.from_numpy(synth.palette(SEED, 256, 81)).cuda())
    lc = codec.encode(torch.from_numpy(synth.lights(SEED, L, 81)).cuda()).cpu().numpy()
    band = row_band(rank, world, H, W)
    idx, cosv = a.synth_gbuffer(ctx, SEED, band.first_pixel, band.pixels, L, 256)
    rgb, xyz = PeerFrame(band, H, device=0), PeerFrame(band, H, device=0)
    if rank == 0:
        rgb.image.fill_(-1.0)
        xyz.image.fill_(-1.0)
        torch.cuda.synchronize()
    dist.barrier()
    for _ in range(3):  # repeated frames into the same mapping
        codec.shade_latent(pal, lc, idx, cosv, out={"latent": None, "spectra": None, "xyz": xyz.local,
                                                    "rgb": rgb.local})
    torch.cuda.synchronize()
    dist.barrier()  # every rank's stores are complete
    if rank == 0:
        np.save(out_path, np.concatenate([rgb.image.cpu().numpy(), xyz.image.cpu().numpy()], axis=1))
    dist.barrier()
    rgb.close()
    xyz.close()
    dist.destroy_process_group()


def test_two_ranks_fused_gather_through_peer_memory(api, tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "fused.npy")
    mp.spawn(_rank_fused, args=(2, _free_port(), out), nprocs=2, join=True)
    ctx = api.Context(0)
    E, D = synth.codec_weights(SEED, K, 81)
    codec = api.Codec(ctx, E, D)
    pal = codec.encode(torch.from_numpy(synth.palette(SEED, 256, 81)).cuda())
    lc = codec.encode(torch.from_numpy(synth.lights(SEED, L, 81)).cuda()).cpu().numpy()
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, W * H, L, 256)
    want = codec.shade_latent(pal, lc, idx, cosv)
    got = np.load(out)
    assert np.array_equal(got[:, :3], want["rgb"].cpu().numpy())
    assert np.array_equal(got[:, 3:], want["xyz"].cpu().numpy())


def test_two_ranks_on_the_gpu_match_one_process(api, tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "rgb.npy")
    mp.spawn(_rank, args=(2, _free_port(), out), nprocs=2, join=True)
    ctx = api.Context(0)
    E, D = synth.codec_weights(SEED, K, 81)
    codec = api.Codec(ctx, E, D)
    pal = codec.encode(torch.from_numpy(synth.palette(SEED, 256, 81)).cuda())
    lc = codec.encode(torch.from_numpy(synth.lights(SEED, L, 81)).cuda()).cpu().numpy()
    idx, cosv = api.synth_gbuffer(ctx, SEED, 0, W * H, L, 256)
    want = codec.shade_latent(pal, lc, idx, cosv)["rgb"].cpu().numpy()
    assert np.array_equal(np.load(out), want)
