"""Windowed / full decode on the GPU (reference codec.py) -- B2-B9.

Tolerance: int16 samples within 1 LSB of the reference's float64 numpy decode (the
GPU sums the conv and upsample contractions in a different fixed order; BLAS order is
not reproducible).  Bit-exact: window bookkeeping, and the GPU's windowed decode ==
its own full decode whenever overlap >= receptive field.
"""
import numpy as np
import pytest

import oracle.ringflow_np as O
import scenarios

pytestmark = pytest.mark.gpu
LSB_TOL = 1


@pytest.fixture(scope="module")
def rf():
    import paper_2605_28657_b200 as m

    return m


def lsb(a, b):
    return int(np.max(np.abs(a.astype(np.int32) - b.astype(np.int32)))) if a.size else 0


def test_full_and_windows_vs_reference(rf, goldens):
    codec = rf.ToyCodec(channels=8, hop=64)
    lat = goldens["codec8_latent"]
    full = codec.full_decode(lat)
    assert full.samples.dtype == np.int16 and full.start_frame == 0 and full.frame_count == 96
    assert lsb(full.samples, goldens["codec8_full"]) <= LSB_TOL
    for a, b, ov, fdl in goldens["codec8_windows"]:
        ch = codec.windowed_decode(lat, (int(a), int(b)), int(ov))
        assert ch.start_frame == a and ch.frame_count == b - a
        assert codec.frames_decoded_last == fdl
        assert lsb(ch.samples, goldens[f"codec8_win_{a}_{b}_{ov}"]) <= LSB_TOL
        if ov >= codec.receptive_field:   # windowed == full, bit for bit, on the GPU
            assert np.array_equal(ch.samples, full.samples[a * 64:b * 64])


def test_c64_hop1920_vs_reference(rf, goldens):
    codec = rf.ToyCodec(channels=64, hop=1920)
    lat = goldens["codec64_latent"]
    full = codec.full_decode(lat).samples
    assert lsb(full, goldens["codec64_full"]) <= LSB_TOL
    win = codec.windowed_decode(lat, (10, 25), 15).samples
    assert lsb(win, goldens["codec64_win"]) <= LSB_TOL
    assert np.array_equal(win, full[10 * 1920:25 * 1920])


def test_receptive_field_probe(rf, goldens):
    codec = rf.ToyCodec(channels=8, hop=64)
    assert codec.receptive_field == 15
    assert rf.measure_receptive_field(codec) == int(goldens["codec8_rf"]) == 15
    assert rf.measure_receptive_field(rf.ToyCodec(channels=8, hop=16, dilations=(1,))) == 1
    for dil in [(1,), (1, 2), (1, 2, 4)]:
        assert rf.measure_receptive_field(rf.ToyCodec(channels=8, hop=16, dilations=dil)) <= sum(dil)


def test_sixty_second_windows_identity(rf):
    """60-s latent (T=1500, C=64, hop=1920): the 3-s playback window + overlap 15 equals
    the full decode's slice bit for bit, and the full decode is within 1 LSB of the oracle."""
    codec = rf.ToyCodec(channels=64, hop=1920)
    lat = scenarios.keyed(7, "sixty", (1500, 64)) * 0.5
    full = codec.full_decode(lat).samples
    rng = np.random.default_rng(1)
    for _ in range(10):
        a = int(rng.integers(0, 1499))
        b = int(min(1500, a + rng.integers(1, 400)))
        assert np.array_equal(codec.windowed_decode(lat, (a, b), 15).samples, full[a * 1920:b * 1920])
    tail = codec.windowed_decode(lat, (1425, 1500), 15).samples
    assert np.array_equal(tail, full[1425 * 1920:])
    ref = O.Codec(64, 1920).window(lat, 1425, 1500, 15)
    assert lsb(tail, ref) <= LSB_TOL


def test_zero_overlap_differs_and_bounds(rf, goldens):
    codec = rf.ToyCodec(channels=8, hop=64)
    lat = goldens["codec8_latent"]
    full = codec.full_decode(lat).samples
    diffs = [lsb(codec.windowed_decode(lat, (a, b), 0).samples, full[a * 64:b * 64])
             for a, b in [(20, 40), (41, 60), (10, 30)]]
    assert max(diffs) > 0
    for bad in [(-1, 10), (0, 97), (5, 5)]:
        with pytest.raises(ValueError):
            codec.windowed_decode(lat, bad, 2)
    with pytest.raises(ValueError):
        codec.windowed_decode(lat, (0, 10), -1)
    assert np.all(codec.full_decode(np.zeros((96, 8))).samples == 0)


def test_pcm_chunk(rf, goldens):
    codec = rf.ToyCodec(channels=8, hop=64)
    ch = codec.windowed_decode(goldens["codec8_latent"], (4, 12), 15)
    assert np.array_equal(np.frombuffer(ch.to_bytes(), dtype="<i2"), ch.samples)
    assert ch.header() == {"hop": 64, "start_frame": 4, "frame_count": 8}
    assert rf.codec.quantize_pcm(np.array([0.0, 0.5 / 32767, -0.5 / 32767, 1.0, -1.0, 2.0, -2.0])).tolist() == \
        goldens["quantize_kat"].tolist()
    with pytest.raises(ValueError):
        rf.PcmChunk(np.zeros(10, dtype=np.int16), start_frame=0, hop=64)


def test_encode_vs_reference(rf):
    """ToyCodec.encode (codec.py:168-174) on the GPU (rf_encode_frames) vs the float64 numpy
    product of the same projection; tolerance 1e-12 relative (summation order differs)."""
    for C, hop in ((8, 64), (64, 1920)):
        codec = rf.ToyCodec(channels=C, hop=hop)
        x = scenarios.keyed(5, "encode-pcm", (37 * hop,))
        lat = codec.encode(x)
        ref = x.reshape(-1, hop) @ codec._encode_proj.T
        assert lat.shape == (37, C) and lat.dtype == np.float64
        assert np.max(np.abs(lat - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    with pytest.raises(ValueError):
        codec.encode(np.zeros(hop + 1))
