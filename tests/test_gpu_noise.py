"""GPU keyed noise == numpy's Philox4x64-10 ziggurat, bit for bit."""
import hashlib

import numpy as np
import pytest
import torch

import oracle.ringflow_np as O

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def rf():
    import paper_2605_28657_b200 as m

    return m


def test_golden_draws(rf, goldens):
    for i in range(6):
        seed, stream, step, n = goldens[f"noise{i}_args"]
        tag = str(goldens[f"noise{i}_tag"])
        ns = rf.NoiseSource(seed=int(seed), stream=int(stream))
        assert sha(ns.normal(int(step), tag, (int(n),))) == str(goldens[f"noise{i}_normal_sha"]), i
        assert sha(ns.uniform(int(step), tag, (int(n),))) == str(goldens[f"noise{i}_uniform_sha"]), i
    ns = rf.NoiseSource(seed=123, stream=456)
    assert sha(ns.normal(9, "long", (1_000_000,))) == str(goldens["noise_long_sha"])


def test_survey_kat(rf):
    v = rf.NoiseSource(0, 0).normal(0, "sde", (4,))
    assert v.tolist() == [-0.8766545588837262, 1.8638264440516052, -0.3612334156474177, -1.833676777774578]


@pytest.mark.parametrize("n", [1, 2, 3, 15, 16, 17, 255, 4095, 4096, 4097, 96000, 384000])
def test_sizes_bit_exact(rf, n):
    for seed in range(3):
        ns = rf.NoiseSource(seed=seed, stream=n)
        got = ns.normal(seed, "sz", (n,))
        ref = O.normal(seed, n, seed, "sz", (n,))
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


def test_batched_draws_bit_exact(rf):
    """Many draws of mixed sizes in one rf_normal_fill batch (the tick's layout)."""
    from paper_2605_28657_b200.latents import fill_normals, philox_key

    dev = torch.device("cuda")
    specs = [(s, 1000 + s, s % 8, ("sde", "model", "init")[s % 3], [96000, 2000, 50, 130000][s % 4])
             for s in range(30)]
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for *_, n in specs]
    fill_normals([(philox_key(s, st, k, t), o) for (s, st, k, t, _), o in zip(specs, outs)])
    for (s, st, k, t, n), o in zip(specs, outs):
        assert np.array_equal(o.cpu().numpy(), O.normal(s, st, k, t, (n,)))


def test_ten_million_draws_bit_exact(rf):
    """~1e7 normals: ~120k wedge and ~2.6k tail events vs numpy (glibc exp/log1p vs CUDA)."""
    from paper_2605_28657_b200.latents import fill_normals, philox_key

    dev = torch.device("cuda")
    total_bad = 0
    for s in range(10):
        n = 1_000_000
        out = torch.empty(n, dtype=torch.float64, device=dev)
        fill_normals([(philox_key(77, s, 0, "big"), out)])
        ref = O.normal(77, s, 0, "big", (n,))
        total_bad += int(np.count_nonzero(out.cpu().numpy().view(np.uint64) != ref.view(np.uint64)))
    assert total_bad == 0


def test_uniform_and_errors(rf):
    ns = rf.NoiseSource(seed=9, stream=8)
    assert np.array_equal(ns.uniform(3, "u", (1000,)), O.uniform(9, 8, 3, "u", (1000,)))
    with pytest.raises(ValueError):
        ns.normal(-1, "x", (3,))
    a = ns.normal(1, "x", (2, 5))
    assert a.shape == (2, 5)
    assert np.array_equal(a, ns.normal(1, "x", (2, 5)))
    assert not np.array_equal(a, ns.normal(1, "y", (2, 5)))
