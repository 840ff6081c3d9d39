"""Config 5: long decode sharded across ranks with halos + one all-gather of the PCM.

CPU (gloo, world 2 and 3): the host logic -- shard ranges, padding, byte all-gather and
trim -- reassembles the oracle's full decode exactly from the oracle's windowed shard
decodes (the reference's windowed identity, codec.py:136-164).
GPU: the sharded decode through the CUDA kernel equals the single-rank full decode bit
for bit, at world 1 and with 2 ranks sharing the device over gloo (the box has 1 GPU;
the NCCL path differs only in the collective call).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle.ringflow_np as O
import scenarios


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _cpu_worker(rank, world, port, frames, channels, hop, q):
    try:
        from paper_2605_28657_b200.sharded_decode import gather_shards, shard_ranges

        _init(rank, world, port)
        codec = O.Codec(channels=channels, hop=hop)
        lat = scenarios.keyed(5, "long-latent", (frames, channels))
        lo, hi = shard_ranges(frames, world)[rank]
        per = -(-frames // world) * hop
        local = torch.zeros(per, dtype=torch.int16)
        if hi > lo:
            local[: (hi - lo) * hop] = torch.from_numpy(codec.window(lat, lo, hi, codec.rf))
        pcm = gather_shards(local, frames * hop)
        q.put((rank, pcm.numpy().copy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))


def _run(worker, world, *args):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        assert not isinstance(v, str), f"rank {r}: {v}"
    return out


def test_shard_ranges():
    from paper_2605_28657_b200.sharded_decode import shard_ranges

    assert shard_ranges(6000, 8) == [(i * 750, (i + 1) * 750) for i in range(8)]
    assert shard_ranges(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert shard_ranges(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for frames in (1, 7, 96, 6000):
        for world in (1, 2, 3, 8):
            r = shard_ranges(frames, world)
            assert r[0][0] == 0 and r[-1][1] == frames
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    with pytest.raises(ValueError):
        shard_ranges(0, 2)


@pytest.mark.parametrize("world,frames", [(2, 96), (3, 97)])
def test_gloo_gather_reassembles_oracle_full_decode(world, frames):
    channels, hop = 8, 64
    out = _run(_cpu_worker, world, frames, channels, hop)
    codec = O.Codec(channels=channels, hop=hop)
    full = codec.full(scenarios.keyed(5, "long-latent", (frames, channels)))
    for r in range(world):
        assert out[r].dtype == np.int16 and out[r].shape == full.shape
        assert np.array_equal(out[r], full)


# ------------------------------------------------------------------------ GPU -----
def _gpu_worker(rank, world, port, frames, channels, hop, q):
    try:
        import paper_2605_28657_b200 as rf
        from paper_2605_28657_b200.sharded_decode import sharded_full_decode

        torch.cuda.set_device(0)
        _init(rank, world, port)
        codec = rf.ToyCodec(channels=channels, hop=hop)
        lat = scenarios.keyed(9, "long-latent", (frames, channels)) if rank == 0 else None
        chunk = sharded_full_decode(codec, lat, src=0, frames=frames)
        q.put((rank, chunk.samples.copy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e)))


@pytest.mark.gpu
def test_gpu_sharded_equals_full_world1():
    import paper_2605_28657_b200 as rf
    from paper_2605_28657_b200.sharded_decode import sharded_full_decode

    codec = rf.ToyCodec(channels=64, hop=1920)
    lat = scenarios.keyed(9, "long-latent", (400, 64))
    full = codec.full_decode(lat)
    sh = sharded_full_decode(codec, lat)
    assert sh.start_frame == 0 and sh.frame_count == 400
    assert np.array_equal(sh.samples, full.samples)
    ref = O.Codec(channels=64, hop=1920).full(lat)
    assert int(np.max(np.abs(sh.samples.astype(np.int32) - ref))) <= 1


@pytest.mark.gpu
@pytest.mark.parametrize("world,frames", [(2, 6000), (3, 301)])
def test_gpu_sharded_decode_two_ranks(world, frames):
    import paper_2605_28657_b200 as rf

    out = _run(_gpu_worker, world, frames, 64, 1920)
    full = rf.ToyCodec(channels=64, hop=1920).full_decode(scenarios.keyed(9, "long-latent", (frames, 64))).samples
    for r in range(world):
        assert np.array_equal(out[r], full), f"rank {r}"
