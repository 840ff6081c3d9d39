"""Similarity-filter-gated playback decode.

CPU: the gating bookkeeping with a stand-in codec (which completion is decoded, the
playback window of service.py:318-321, counts).  GPU: a real pipeline's completions,
every chunk bit-identical to codec.windowed_decode of the last unflagged completion,
and one decode launch per unflagged completion.
"""
import numpy as np
import pytest
import torch


class FakeCodec:
    hop = 4

    def __init__(self):
        self.calls = []
        self.frames_decoded_last = 0

    def decode_device(self, lat, start, stop, overlap, full, out=None):
        self.calls.append((start, stop, overlap, full))
        vals = lat[start:stop].sum(1).round().to(torch.int16)
        out.copy_(vals.repeat_interleave(self.hop))
        return out


class Rec:
    def __init__(self, idx, lat, skipped):
        self.completion_index = idx
        self.latent_device = lat
        self.decode_skipped = skipped
        self._stream = None


def test_gating_bookkeeping_cpu():
    from paper_2605_28657_b200.decode_gate import GatedDecoder

    codec = FakeCodec()
    g = GatedDecoder(codec, window_frames=5, overlap=3)
    with pytest.raises(LookupError):
        g.latest_pcm()
    lats = [torch.full((12, 2), float(i + 1), dtype=torch.float64) for i in range(6)]
    flags = [True, True, False, True, True, False]   # a first flagged record still decodes
    launched = [g.feed(Rec(i, l, f)) for i, (l, f) in enumerate(zip(lats, flags))]
    assert launched == [True, False, True, False, False, True]
    assert (g.decodes, g.skips) == (3, 3) and g.skip_rate == 0.5
    assert codec.calls == [(7, 12, 3, False)] * 3          # the last 5 frames, overlap 3
    pcm = g.latest_pcm()
    assert g.source_completion == 5 and pcm.start_frame == 7 and pcm.hop == 4
    assert np.array_equal(pcm.samples, np.full(20, 12, np.int16))
    assert g.window(3) == (0, 3)                              # window clamps to the latent
    with pytest.raises(ValueError):
        GatedDecoder(codec, window_frames=0)


@pytest.mark.gpu
def test_gated_decode_matches_windowed_decode():
    import paper_2605_28657_b200 as rf
    import scenarios

    conf = rf.PipelineConfig(depth=4, steps=4, frames=250, channels=8, seed=3)
    src = scenarios.keyed(3, "gate-source", (250, 8))
    req = rf.GenerationRequest(conditions=(rf.ConditionSet(prompt_hash=rf.content_hash("gate"), source=src),))
    pipe = rf.StreamPipeline(conf, request=req)
    codec = rf.ToyCodec(channels=8, hop=64)
    g = rf.GatedDecoder(codec, window_frames=75, overlap=15)
    n_flagged = n_records = 0
    last_unflagged = None
    for k in range(40):
        if k == 20:   # a control change: the next completions differ, then settle again
            pipe.set_shared_curve("sde_denoise_curve", np.linspace(0.2, 1.0, 250))
        for r in pipe.tick():
            n_records += 1
            launched = g.feed(r)
            assert launched == (not r.decode_skipped or last_unflagged is None)
            if launched:
                last_unflagged = r
            else:
                n_flagged += 1
            pcm = g.latest_pcm()
            ref = codec.windowed_decode(last_unflagged.latent, (175, 250), 15)
            assert pcm.start_frame == 175 and np.array_equal(pcm.samples, ref.samples)
    assert n_records > 20 and n_flagged > 0 and g.decodes + g.skips == n_records
    assert g.skips == n_flagged and 0.0 < g.skip_rate < 1.0
