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


@pytest.mark.parametrize("C,hop,dil", [(8, 64, (1, 2, 4, 8)), (16, 48, (1, 2, 4, 8)), (32, 128, (3, 5)),
                                       (48, 256, (1, 2, 4, 8, 16)), (64, 1920, (1, 2, 4, 8)), (64, 16, (1,))])
def test_tensor_core_decode_shapes(rf, C, hop, dil):
    """rf_decode_window_tc (fp16 hi/lo operands on tcgen05) vs the float64 oracle: within
    1 LSB over full decodes and windows, windowed == full bit-exact at overlap >= RF, and
    within 1 LSB of the float64 CUDA-core kernel."""
    codec = rf.ToyCodec(channels=C, hop=hop, dilations=dil)
    assert codec.tensor_cores
    T = 300
    lat = scenarios.keyed(11, f"tc-{C}-{hop}", (T, C)) * 0.8
    full = codec.full_decode(lat).samples
    ref = O.Codec(C, hop, dil)
    assert lsb(full, ref.full(lat)) <= LSB_TOL
    rfield = sum(dil)
    for a, b in ((0, 7), (5, 150), (140, 300), (299, 300), (37, 38)):
        w = codec.windowed_decode(lat, (a, b), rfield).samples
        assert np.array_equal(w, full[a * hop:b * hop])
        assert lsb(w, ref.window(lat, a, b, rfield)) <= LSB_TOL
        w0 = codec.windowed_decode(lat, (a, b), 2).samples      # overlap < RF: reference semantics
        assert lsb(w0, ref.window(lat, a, b, 2)) <= LSB_TOL
    if C & (C - 1) == 0:                                       # shapes the float64 kernel takes
        packed = codec._packed
        codec._packed = None
        f64 = codec.full_decode(lat).samples
        codec._packed = packed
        assert lsb(full, f64) <= LSB_TOL


def test_non_tensor_core_shape_uses_float64_kernel(rf):
    codec = rf.ToyCodec(channels=8, hop=10)
    assert not codec.tensor_cores
    lat = scenarios.keyed(12, "f64-shape", (40, 8))
    full = codec.full_decode(lat).samples
    assert lsb(full, O.Codec(8, 10).full(lat)) <= LSB_TOL
    assert np.array_equal(codec.windowed_decode(lat, (10, 20), 15).samples, full[100:200])


def test_tensor_core_decode_large_latent_values(rf):
    """Latents 20x the pipeline's scale (|x| up to ~100): still within 1 LSB.  The fp32
    accumulator's rounding grows with the pre-activation magnitude; measured on B200:
    <= 1 LSB up to 1000x the pipeline's scale, 2 LSB at 5000x."""
    codec = rf.ToyCodec(channels=64, hop=1920)
    lat = scenarios.keyed(13, "big", (60, 64)) * 20.0
    full = codec.full_decode(lat).samples
    assert lsb(full, O.Codec(64, 1920).full(lat)) <= LSB_TOL
