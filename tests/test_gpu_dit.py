"""DiT velocity model on sm_100a vs its plain-PyTorch fp32 oracle (oracle/dit_fp32.py).

The reference package has no DiT, so DiT parity is against the builder's
own fp32 forward of the same seeded bf16 weights.  Tolerances are relative RMS errors,
stated per test: both paths round GEMM operands to bf16 at the same points; differences
come from accumulation order and bf16 rounding flips, compounding over layers.
"""
import math

import numpy as np
import pytest
import torch

from oracle.dit_fp32 import reference_forward

pytestmark = pytest.mark.gpu


def rel_rms(a, b):
    return ((a.float() - b.float()).pow(2).mean().sqrt() / b.float().pow(2).mean().sqrt()).item()


@pytest.fixture(scope="module")
def dit_mod():
    from paper_2605_28657_b200 import dit

    return dit


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("B,Nq,Nk,H,Hk,grow", [(2, 750, 750, 16, 8, 0), (1, 100, 37, 4, 4, 0), (3, 750, 128, 16, 8, 0),
                                               (1, 128, 128, 2, 1, 0), (2, 300, 1000, 4, 2, 0),
                                               (2, 256, 900, 4, 2, 1), (1, 200, 640, 2, 2, 1),
                                               (2, 750, 750, 16, 8, 1), (1, 3000, 3000, 4, 2, 1)])
def test_tcgen05_attention_vs_sdpa(dit_mod, kernel, B, Nq, Nk, H, Hk, grow):
    """Every self-attention kernel (rf_attention_tc_bf16_kernel: 0 = the forward's default,
    1 = 64-key tiles, one head per CTA) against SDPA.
    grow: key norms rise along the sequence, so the running row max climbs tile after tile
    (exercises the lazy O / l rescaling)."""
    import ctypes

    from paper_2605_28657_b200 import _native

    lib = _native.load()
    lib.rf_attention_tc_bf16_kernel.restype = int
    g = torch.Generator(device="cuda").manual_seed(Nq * 11 + Nk)
    q = torch.randn(B * Nq, H * 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(B * Nk, Hk * 128, device="cuda", generator=g)
    if grow:
        k = k * torch.linspace(0.3, 4.0, Nk, device="cuda").repeat(B)[:, None]
    k = k.bfloat16()
    v = torch.randn(B * Nk, Hk * 128, device="cuda", generator=g).bfloat16()
    nk_pad = (Nk + 7) // 8 * 8
    vt = torch.zeros(B, Hk, 128, nk_pad, device="cuda", dtype=torch.bfloat16)
    vt[..., :Nk] = v.reshape(B, Nk, Hk, 128).permute(0, 2, 3, 1)
    out = torch.empty(B * Nq, H * 128, device="cuda", dtype=torch.bfloat16)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    _native.check(lib.rf_attention_tc_bf16_kernel(kernel, vp(q.data_ptr()), vp(k.data_ptr()), vp(vt.data_ptr()),
                                                  vp(out.data_ptr()), B, Nq, Nk, nk_pad, H, Hk, i64(H * 128),
                                                  i64(Hk * 128), i64(H * 128),
                                                  vp(torch.cuda.current_stream().cuda_stream)), "attention")
    qq = q.float().reshape(B, Nq, H, 128).transpose(1, 2)
    kk = k.float().reshape(B, Nk, Hk, 128).repeat_interleave(H // Hk, 2).transpose(1, 2)
    vv = v.float().reshape(B, Nk, Hk, 128).repeat_interleave(H // Hk, 2).transpose(1, 2)
    ref = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv).transpose(1, 2).reshape(B * Nq, H * 128)
    assert torch.isfinite(out).all()
    assert rel_rms(out, ref) < 1e-2


def _inputs(dit, rows, frames, C, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    xs = [torch.randn(frames, C, device="cuda", generator=g, dtype=torch.float64) for _ in range(rows)]
    ts = [1.0 - 0.13 * i for i in range(rows)]
    conds = [dit.cond_tokens(1000 + i) for i in range(rows)]
    return xs, ts, conds


def test_small_dit_vs_fp32_oracle(dit_mod):
    cfg = dit_mod.DiTConfig().small()
    dit = dit_mod.DiT(cfg, frames=96, max_rows=4)
    xs, ts, conds = _inputs(dit, 3, 96, 64)
    out = dit.forward(xs, ts, conds).clone()
    ref = reference_forward(dit, xs, ts, conds)
    assert out.shape == ref.shape and torch.isfinite(out).all()
    assert rel_rms(out, ref) < 1e-2   # 2 layers, d=256


def test_rows_are_independent(dit_mod):
    """A row's velocity does not depend on which other rows share the batch (bit-exact):
    this is what makes streaming == sequential render hold with the DiT."""
    cfg = dit_mod.DiTConfig().small()
    dit = dit_mod.DiT(cfg, frames=96, max_rows=4)
    xs, ts, conds = _inputs(dit, 4, 96, 64, seed=3)
    full = dit.forward(xs, ts, conds).clone()
    single = dit.forward(xs[2:3], ts[2:3], conds[2:3]).clone()
    assert torch.equal(full[2], single[0])


def test_full_size_dit_vs_fp32_oracle(dit_mod):
    """ACE-Step shape (24 layers, d=2048, T=1500 -> 750 tokens), 4 rows with distinct t."""
    dit = dit_mod.DiT(dit_mod.DiTConfig(), frames=1500, max_rows=4)
    xs, ts, conds = _inputs(dit, 4, 1500, 64, seed=1)
    out = dit.forward(xs, ts, conds).clone()
    ref = reference_forward(dit, xs, ts, conds)
    assert torch.isfinite(out).all()
    assert rel_rms(out, ref) < 3e-2   # 24 layers of bf16 operands


def test_full_size_dit_is_deterministic(dit_mod):
    """Repeated full-size forwards (replays of the captured graph, back to back) are
    bit-identical and finite -- a data race between warp-specialised roles (TMA, MMA,
    softmax, epilogue) shows up as run-to-run differences here; rows also bit-identical
    to the same rows forwarded in a different batch position."""
    dit = dit_mod.DiT(dit_mod.DiTConfig(), frames=1500, max_rows=4)
    xs, ts, conds = _inputs(dit, 4, 1500, 64, seed=7)
    ref = dit.forward(xs, ts, conds).clone()
    assert torch.isfinite(ref).all()
    outs = []
    for _ in range(6):
        outs.append(dit.forward(xs, ts, conds).clone())
    for o in outs:
        assert torch.equal(o, ref)
    swapped = dit.forward(xs[::-1], ts[::-1], conds[::-1]).clone()
    assert torch.equal(swapped.flip(0), ref)


def test_pipeline_with_dit(dit_mod):
    import scenarios

    import paper_2605_28657_b200 as rf

    cfg = dit_mod.DiTConfig().small()
    T, D = 96, 64
    src = scenarios.keyed(100, "source", (T, D))
    req = rf.GenerationRequest(conditions=(rf.ConditionSet(rf.prompt_id("p"), source=src),),
                               curves=rf.make_curves(T, sde_denoise_curve=np.linspace(0.2, 1.0, T)))
    conf = rf.PipelineConfig(depth=4, steps=8, frames=T, channels=D)
    dit = dit_mod.DiT(cfg, frames=T, max_rows=8)
    pipe = rf.StreamPipeline(conf, request=req, velocity_model=dit_mod.DiTVelocity(dit))
    toy = rf.StreamPipeline(conf, request=req)
    recs, trecs = [], []
    for _ in range(24):
        recs += pipe.tick()
        trecs += toy.tick()
    # bookkeeping is independent of the velocity model
    assert [(r.tick, r.submission_id, r.schedule_id) for r in recs] == \
        [(r.tick, r.submission_id, r.schedule_id) for r in trecs]
    assert all(np.isfinite(r.latent).all() for r in recs)
    # streaming == sequential render (bit-exact) with the DiT too
    assert np.array_equal(recs[-1].latent, pipe.render(req))


def test_full_size_pipeline_with_dit_is_reproducible(dit_mod):
    """Config 2 (ACE-Step-shape DiT, T=1500, depth 4, S=8) streamed twice with the same seed:
    every completion finite and bit-identical between the runs (the bench's workload; a
    softmax-warp race in the attention once surfaced only here, as non-finite latents)."""
    import scenarios

    import paper_2605_28657_b200 as rf

    T, D = 1500, 64
    src = scenarios.keyed(0, "bench-source", (T, D))
    req = rf.GenerationRequest(conditions=(rf.ConditionSet(prompt_hash=rf.content_hash("bench", "bench prompt"),
                                                           source=src),))
    conf = rf.PipelineConfig(depth=4, steps=8, frames=T, channels=D, seed=0)
    dit = dit_mod.DiT(dit_mod.DiTConfig(), frames=T, max_rows=4)
    runs = []
    for _ in range(2):
        # the two pipelines share the DiT (and its workspace): one finishes before the next starts
        torch.cuda.synchronize()
        pipe = rf.StreamPipeline(conf, request=req, velocity_model=dit_mod.DiTVelocity(dit))
        recs = []
        for _ in range(28):
            recs += pipe.tick()
        runs.append([r.latent for r in recs])   # host copies, ordered after the pipeline stream
        torch.cuda.synchronize()
    assert len(runs[0]) >= 8
    for a, b in zip(*runs):
        assert np.isfinite(a).all() and np.array_equal(a, b)


@pytest.mark.parametrize("full", [False, True])
def test_stream_group_batches_rows_bit_identically(dit_mod, full):
    """Two co-resident streams (different seeds, prompts, denoise schedules) ticked as a
    StreamGroup -- one batched DiT forward over both rings' rows per tick -- emit exactly
    the completions each stream emits when ticked alone (rows are independent)."""
    import scenarios

    import paper_2605_28657_b200 as rf

    cfg = dit_mod.DiTConfig() if full else dit_mod.DiTConfig().small()
    T, D = (1500, 64) if full else (96, 64)
    dit = dit_mod.DiT(cfg, frames=T, max_rows=8)

    def make(seed, vm):
        src = scenarios.keyed(seed, "bench-source", (T, D))
        req = rf.GenerationRequest(conditions=(rf.ConditionSet(rf.prompt_id(f"stream {seed}"), source=src),))
        return rf.StreamPipeline(rf.PipelineConfig(depth=4, steps=8, frames=T, channels=D, seed=seed,
                                                   denoise=1.0 if seed == 0 else 0.7),
                                 request=req, velocity_model=vm)

    ticks = 14
    alone = []
    for seed in (0, 1):
        p = make(seed, dit_mod.DiTVelocity(dit))
        recs = []
        for _ in range(ticks):
            recs += p.tick()
        alone.append([(r.tick, r.submission_id, r.latent) for r in recs])
        torch.cuda.synchronize()
    shared = dit_mod.DiTVelocity(dit)
    group = rf.StreamGroup([make(0, shared), make(1, shared)])
    together = [[], []]
    for _ in range(ticks):
        for i, recs in enumerate(group.tick()):
            together[i] += [(r.tick, r.submission_id, r.latent) for r in recs]
    for a, b in zip(alone, together):
        assert len(a) == len(b) >= 3
        for (ta, sa, la), (tb, sb, lb) in zip(a, b):
            assert ta == tb and sa == sb and np.array_equal(la, lb)


def test_attention_under_concurrent_load(dit_mod):
    """The self-attention kernel, launched back to back while another stream keeps the SMs
    busy (as the trajectory tests' oracle does): every launch completes and matches the
    first.  Its P-ready barriers alternate by key-tile parity -- with one barrier the softmax
    warps could finish two tiles before the MMA warp polled, leaving the waiter two phases
    behind (an intermittent hang, caught by the RF_HANG_TRAP diagnostic build)."""
    import ctypes

    from paper_2605_28657_b200 import _native

    lib = _native.load()
    B, N, H, Hk = 4, 750, 16, 8
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(B * N, H * 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(B * N, Hk * 128, device="cuda", generator=g).bfloat16()
    vt = torch.randn(B, Hk, 128, (N + 7) // 8 * 8, device="cuda", generator=g).bfloat16()
    vt[..., N:] = 0
    outs = [torch.empty(B * N, H * 128, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    side, main = torch.cuda.Stream(), torch.cuda.Stream()
    a = torch.randn(2048, 2048, device="cuda")
    for it in range(6):
        with torch.cuda.stream(side):
            for _ in range(20):
                a = torch.tanh(a @ a * 1e-3)
        with torch.cuda.stream(main):
            for r in range(50):
                _native.check(lib.rf_attention_tc_bf16_kernel(
                    0, vp(q.data_ptr()), vp(k.data_ptr()), vp(vt.data_ptr()), vp(outs[r % 2].data_ptr()), B, N, N,
                    vt.shape[-1], H, Hk, i64(H * 128), i64(Hk * 128), i64(H * 128), vp(main.cuda_stream)), "attention")
        main.synchronize()
        assert torch.equal(outs[0], outs[1])
    side.synchronize()


def test_persisting_l2_set_aside_is_returned(dit_mod):
    """A DiT raises the device's persisting-L2 limit for its residual stream; when the last
    DiT on the device is destroyed the previous limit is back (other work gets its L2)."""
    import gc

    before = _persisting_limit()
    a = dit_mod.DiT(dit_mod.DiTConfig().small(), frames=96, max_rows=2)
    b = dit_mod.DiT(dit_mod.DiTConfig().small(), frames=96, max_rows=2)
    assert _persisting_limit() >= before
    del a
    gc.collect()
    del b
    gc.collect()
    torch.cuda.synchronize()
    assert _persisting_limit() == before


def _persisting_limit() -> int:
    """cudaDeviceGetLimit(cudaLimitPersistingL2CacheSize) on the current device (cuda-python)."""
    try:
        from cuda.bindings import runtime as cudart
    except ImportError:
        try:
            from cuda import cudart
        except ImportError:
            pytest.skip("cuda-python runtime bindings not importable")
    err, v = cudart.cudaDeviceGetLimit(cudart.cudaLimit.cudaLimitPersistingL2CacheSize)
    assert int(err) == 0, err
    return int(v)


def test_residual_stream_larger_than_the_l2_window(dit_mod):
    """max_rows x tokens x d_model x 4 B above the device's maximum access-policy window
    (here 32 x 10 000 x 256 x 4 = 328 MB): the persisting window is clamped, the forward
    runs, and a row's velocity is bit-identical to the same row in a small-capacity DiT."""
    cfg = dit_mod.DiTConfig().small()
    w = dit_mod.DiTWeights(cfg)
    big = dit_mod.DiT(cfg, frames=20000, max_rows=32, weights=w)
    one = dit_mod.DiT(cfg, frames=20000, max_rows=1, weights=w)
    xs, ts, conds = _inputs(big, 2, 20000, 64, seed=9)
    a = big.forward(xs, ts, conds).clone()
    b = one.forward(xs[1:], ts[1:], conds[1:]).clone()
    assert torch.isfinite(a).all()
    assert torch.equal(a[1], b[0])


@pytest.mark.parametrize("rows", [2, 3, 4, 5, 8])
def test_row_bit_identical_across_projection_tile_widths(dit_mod, rows):
    """The O / cross-O / down projections take 256 x 256 or 256 x 128 tiles by the forward's
    row count (256 x 128 at 1 and 4 rows, 256 x 256 at 2, 3, 5 and 8): a row's velocity is
    the same bytes either way (same per-element MMA reduction; the fused norm's partial sums
    are per 128 columns whatever the tile width)."""
    dit = dit_mod.DiT(dit_mod.DiTConfig(), frames=1500, max_rows=8)
    xs, ts, conds = _inputs(dit, rows, 1500, 64, seed=11)
    full = dit.forward(xs, ts, conds).clone()
    for r in (0, rows - 1):
        one = dit.forward(xs[r:r + 1], ts[r:r + 1], conds[r:r + 1]).clone()
        assert torch.equal(full[r], one[0]), r
