"""Long-audio decode sharded across ranks with halos, one NCCL all-gather of the PCM
(BASELINE config 5).

The reference decodes a whole latent in one ``ToyCodec.full_decode`` (codec.py:132-134)
and a playback window with ``windowed_decode`` (codec.py:136-164), whose overlap margins
make the window's samples independent of everything outside ``[start - ov, stop + ov)``.
That identity is what lets a long decode shard with no exchange but the result:

  1. the owner rank broadcasts the latent ``[T, C]`` (f64; 3 MB at 240 s);
  2. rank r decodes frames ``[lo_r, hi_r)`` with overlap ``ov >= receptive_field``
     (``rf_decode_window``: global-edge zero padding and the valid mask exactly as the
     full decode applies them), which on the GPU is bit-identical to the same frames of
     the full decode;
  3. one all-gather of the int16 shards (padded to equal length, carried as bytes since
     NCCL has no int16 type) assembles the full PCM on every rank.

Shards are equal ``ceil(T / G)`` frame ranges in rank order, so the gathered buffer is
already in frame order.  ``shard_ranges`` / ``gather_shards`` are backend-agnostic (the
CPU tests drive them over gloo); the decode itself runs only on the CUDA device.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _device
from .codec import PcmChunk, ToyCodec

__all__ = ["shard_ranges", "gather_shards", "sharded_decode_device", "sharded_full_decode"]


def shard_ranges(frames: int, world: int) -> list:
    """Equal contiguous frame ranges ``[(lo, hi)]`` in rank order (the last may be short or empty)."""
    if frames < 1 or world < 1:
        raise ValueError(f"need frames >= 1 and world >= 1 (got {frames}, {world})")
    per = -(-frames // world)
    return [(min(frames, r * per), min(frames, (r + 1) * per)) for r in range(world)]


def _world(group):
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def gather_shards(local: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather equal-length int16 shards (rank order) and trim to ``total`` samples.

    ``local`` is this rank's padded shard; every rank passes the same length.  The bytes
    travel as uint8 (NCCL has no 16-bit integer type; the gather does no arithmetic)."""
    world, _ = _world(group)
    if world == 1:
        return local[:total]
    flat = local.contiguous().view(torch.uint8)
    out = torch.empty(world * flat.numel(), dtype=torch.uint8, device=flat.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, flat, group=group)
    else:
        dist.all_gather(list(out.chunk(world)), flat, group=group)
    return out.view(torch.int16)[:total]


def sharded_decode_device(codec: ToyCodec, latent, group=None, src: int = 0, overlap: int = None,
                          frames: int = None) -> torch.Tensor:
    """Full-latent decode split across the ranks of ``group``; returns the int16 device PCM
    ``[T * hop]`` on every rank (bit-identical to ``codec.full_decode``).

    ``latent`` is needed on rank ``src`` only (others may pass None with ``frames``); it is
    broadcast over the group.  ``overlap`` defaults to the codec's receptive field, the
    smallest margin for which the shard equals the full decode."""
    world, rank = _world(group)
    dev = codec._dev
    ov = codec.receptive_field if overlap is None else int(overlap)
    if ov < codec.receptive_field:
        raise ValueError(f"overlap {ov} < receptive field {codec.receptive_field}: shards would not "
                         "reproduce the full decode")
    if latent is not None:
        lat = _device.to_device_f64(latent, dev)
        if lat.ndim != 2 or lat.shape[1] != codec.channels:
            raise ValueError(f"latent must be [T, {codec.channels}]")
        frames = lat.shape[0]
    elif frames is None:
        raise ValueError("frames is required on ranks that pass no latent")
    if world > 1:
        if rank == src and latent is None:
            raise ValueError("the src rank must pass the latent")
        if rank != src:
            lat = torch.empty(int(frames), codec.channels, dtype=torch.float64, device=dev)
        dist.broadcast(lat, src=dist.get_global_rank(group, src) if group is not None else src, group=group)
    elif latent is None:
        raise ValueError("a single-rank decode needs the latent")
    lo, hi = shard_ranges(int(frames), world)[rank]
    per = -(-int(frames) // world) * codec.hop
    local = torch.zeros(per, dtype=torch.int16, device=dev)
    if hi > lo:
        codec.decode_device(lat, lo, hi, ov, False, out=local[: (hi - lo) * codec.hop])
    return gather_shards(local, int(frames) * codec.hop, group)


def sharded_full_decode(codec: ToyCodec, latent, group=None, src: int = 0, frames: int = None) -> PcmChunk:
    """``ToyCodec.full_decode`` sharded over ``group`` (codec.py:132-134 semantics)."""
    pcm = sharded_decode_device(codec, latent, group=group, src=src, frames=frames)
    codec.frames_decoded_last = int(pcm.numel() // codec.hop)
    return PcmChunk(pcm.cpu().numpy().astype(np.int16, copy=False), start_frame=0, hop=codec.hop)
