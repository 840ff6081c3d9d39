"""Similarity-filter-gated playback decode.

The reference only *flags* a completion whose latent is within MSE 1e-3 of the previous
emitted one (``CompletionRecord.decode_skipped``, ``pipeline.py:473-476``) and decodes
the playback window on demand (``SessionManager.latest_pcm``, ``service.py:315-322``:
the last ``window_frames`` frames with ``overlap`` margins).  The paper's filter
(``PAPER.md:203``) acts on that flag: a flagged completion does not reach the VAE and
the previous audio chunk is reused.

``GatedDecoder`` does exactly that on the device.  ``feed(record)`` enqueues one
``rf_decode_window`` launch (the clustered windowed decode, ``csrc/rf_codec.cu``) on the
record's pipeline stream for every unflagged completion, writing the trimmed int16 chunk
into one of two HBM buffers, and does nothing for a flagged one (the last chunk stays
current).  Nothing synchronises until ``latest_pcm()`` reads the chunk to the host.
The audio of every completion therefore equals
``codec.windowed_decode(latent_of_last_unflagged_completion, window, overlap)``
bit for bit (tests/test_decode_gate.py).
"""
from __future__ import annotations

import contextlib

import torch

from .codec import PcmChunk, ToyCodec

__all__ = ["GatedDecoder"]


class GatedDecoder:
    """Decode the playback window of each completion unless the similarity filter flagged it."""

    def __init__(self, codec: ToyCodec, window_frames: int = 75, overlap: int = 15):
        if window_frames < 1:
            raise ValueError("window_frames must be >= 1")
        if overlap < 0:
            raise ValueError("overlap must be >= 0")
        self.codec = codec
        self.window_frames = window_frames
        self.overlap = overlap
        self.decodes = 0
        self.skips = 0
        self._bufs: list = []
        self._cur = -1              # index of the buffer holding the current chunk
        self._start_frame = 0
        self._frames = 0
        self._stream = None
        self._source_completion = None   # completion_index whose latent the chunk renders

    # ----------------------------------------------------------------- gating
    def window(self, frames: int) -> tuple:
        """The playback window service.py:318-321 picks: the last ``window_frames`` frames."""
        w = max(1, min(self.window_frames, frames))
        return frames - w, frames

    def feed(self, record) -> bool:
        """Handle one CompletionRecord; returns True when a decode was launched."""
        if record.decode_skipped and self._cur >= 0:
            self.skips += 1
            return False
        lat = record.latent_device
        frames = lat.shape[0]
        start, stop = self.window(frames)
        n = (stop - start) * self.codec.hop
        nxt = (self._cur + 1) % 2
        if len(self._bufs) < 2:
            self._bufs = [torch.empty(n, dtype=torch.int16, device=lat.device) for _ in range(2)]
        if self._bufs[nxt].numel() != n:
            self._bufs[nxt] = torch.empty(n, dtype=torch.int16, device=lat.device)
        stream = getattr(record, "_stream", None)
        if stream is None and lat.is_cuda:
            stream = torch.cuda.current_stream(lat.device)
        with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
            self.codec.decode_device(lat, start, stop, self.overlap, False, out=self._bufs[nxt])
        self._cur = nxt
        self._start_frame = start
        self._frames = frames
        self._stream = stream
        self._source_completion = record.completion_index
        self.decodes += 1
        self.codec.frames_decoded_last = (stop + self.overlap) - (start - self.overlap)
        return True

    # ----------------------------------------------------------------- output
    @property
    def skip_rate(self) -> float:
        total = self.decodes + self.skips
        return self.skips / total if total else 0.0

    @property
    def source_completion(self):
        """completion_index of the latent the current chunk was decoded from."""
        return self._source_completion

    def latest_device(self) -> torch.Tensor:
        """The current chunk's int16 samples in HBM (valid on the pipeline stream)."""
        if self._cur < 0:
            raise LookupError("no completion decoded yet")
        return self._bufs[self._cur]

    def latest_pcm(self) -> PcmChunk:
        """The current chunk on the host (service.py:315-322's return value)."""
        dev = self.latest_device()
        if self._stream is not None:
            self._stream.synchronize()
        return PcmChunk(dev.cpu().numpy(), start_frame=self._start_frame, hop=self.codec.hop)
