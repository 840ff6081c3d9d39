"""CPU / fp32 oracle of the DiT velocity model (the ACE-Step-1.5-shape network that fills the
reference's model slot, ``model.py:91-152``, at BASELINE configs 2-5).

TEST INFRASTRUCTURE ONLY.  Only tests/, tools/ and bench.py's CPU baseline / reference arm
import this module; the product package (paper_2605_28657_b200/) never does.

* ``forward_fp32`` -- the network in plain PyTorch fp32 (bf16 weights upcast, no TF32), with
  the same bf16 rounding points as the sm_100a forward (csrc/rf_dit.cu).  The reference has
  no DiT, so DiT parity is unpinned by it; this is the oracle the GPU
  forward is tested against (tests/test_gpu_dit.py, rel-RMS tolerance stated there).
* ``reference_forward(dit, ...)`` -- the same on a GPU ``DiT``'s own weights.
* ``CpuDiTVelocity`` -- the network on the host CPU (fp32, or bf16 GEMM / attention operands
  for the timing arm), plugged into the oracle pipeline's model slot
  (``oracle/ringflow_np.py``: ``Pipeline.model.velocity``) so bench.py can time the
  reference's CPU path at config 2 on the same workload as the GPU arm (a DiT forward per
  ring row per tick), not the toy model.
"""
from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np
import torch


def _rmsnorm(x, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps)


def _rope(x, cos, sin):
    # interleaved pairs (2i, 2i+1) of each 128-dim head; x [B, N, H, 128]
    x0, x1 = x[..., 0::2], x[..., 1::2]
    y0 = x0 * cos - x1 * sin
    y1 = x0 * sin + x1 * cos
    return torch.stack([y0, y1], -1).flatten(-2)


def forward_fp32(cfg, W, frames, xs, ts, conds, layers=None, f=lambda w: w.float(), bf16_matmul=False, pure=False):
    """The DiT in fp32.  cfg: DiTConfig; W: weights with the DiTWeights attribute names
    (f maps a stored weight to the fp32 tensor used); xs: [frames, C] latents; ts: per-row
    timesteps; conds: [n_cond_tokens, d] conditioning tokens.  Returns [B, frames, C].
    bf16_matmul: GEMM and attention operands in bf16 (weights stored bf16; products
    accumulated in fp32 by the backend, outputs rounded to bf16) -- the CPU timing arm's
    fast path (AMX); the oracle itself is fp32.
    pure: no bf16 rounding points at all -- the latent, timestep features, every activation
    and GEMM operand stay fp32 (the weights and conditioning tokens are bf16-VALUED inputs
    of the model, upcast exactly); with TF32 off this is the true fp32 network, the
    reference the bf16-vs-fp32 drift of the GPU forward is measured against."""
    if bf16_matmul:
        matmul = lambda a, w: (a.bfloat16() @ w.T).float()  # noqa: E731
    else:
        matmul = lambda a, w: a @ f(w).T  # noqa: E731
    sdpa_dt = torch.bfloat16 if bf16_matmul else torch.float32
    B, T, C = len(xs), frames, cfg.latent_channels
    N, d = T // cfg.patch, cfg.d_model
    H, Hk, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    bfr = (lambda t: t) if pure else (lambda t: t.bfloat16().float())  # noqa: E731
    x = torch.stack([xx.float() for xx in xs]).reshape(B, N, cfg.in_dim)
    x = bfr(x)
    dev = x.device
    half = cfg.freq_dim // 2
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, device=dev, dtype=torch.float32) / half)
    args = 1000.0 * torch.tensor([float(t) for t in ts], device=dev)[:, None] * freqs[None]
    tf = bfr(torch.cat([torch.cos(args), torch.sin(args)], -1))
    silu = torch.nn.functional.silu
    temb = matmul(bfr(silu(matmul(tf, W.w_t1))), W.w_t2)
    st = bfr(silu(temb))
    mod = matmul(st, W.w_ada)                       # [B, 6d]
    fmod = matmul(st, W.w_final_ada)                # [B, 2d]
    h = matmul(x, W.w_in)                           # [B, N, d]
    pos = torch.arange(N, device=dev, dtype=torch.float64)
    inv = torch.pow(torch.tensor(cfg.rope_theta, dtype=torch.float64),
                    -2.0 * torch.arange(64, device=dev, dtype=torch.float64) / 128.0)
    ang = pos[:, None] * inv[None]
    cos, sin = torch.cos(ang).float()[None, :, None, :], torch.sin(ang).float()[None, :, None, :]
    cond = torch.stack([c.float() for c in conds])  # [B, Nc, d]
    L = cfg.n_layers if layers is None else layers
    for l in range(L):
        m = mod + W.ada_table[l][None]
        sh1, sc1, g1, sh2, sc2, g2 = [m[:, i * d:(i + 1) * d][:, None, :] for i in range(6)]
        a = bfr(_rmsnorm(h, cfg.norm_eps) * (1 + sc1) + sh1)
        qkv = bfr(matmul(a, W.w_qkv[l]))
        q = qkv[..., :H * hd].reshape(B, N, H, hd)
        k = qkv[..., H * hd:(H + Hk) * hd].reshape(B, N, Hk, hd)
        v = qkv[..., (H + Hk) * hd:].reshape(B, N, Hk, hd)
        q, k = bfr(_rope(q, cos, sin)), bfr(_rope(k, cos, sin))
        k = k.repeat_interleave(H // Hk, dim=2)
        v = v.repeat_interleave(H // Hk, dim=2)
        o = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2).to(sdpa_dt), k.transpose(1, 2).to(sdpa_dt),
                                                             v.transpose(1, 2).to(sdpa_dt)).float()
        o = bfr(o.transpose(1, 2).reshape(B, N, H * hd))
        h = h + g1 * (matmul(o, W.w_o[l]))
        c = bfr(_rmsnorm(h, cfg.norm_eps))
        qc = bfr(matmul(c, W.w_qc[l])).reshape(B, N, H, hd)
        kvc = bfr(matmul(cond, W.w_kvc[l]))
        kc = kvc[..., :Hk * hd].reshape(B, -1, Hk, hd).repeat_interleave(H // Hk, dim=2)
        vc = kvc[..., Hk * hd:].reshape(B, -1, Hk, hd).repeat_interleave(H // Hk, dim=2)
        oc = torch.nn.functional.scaled_dot_product_attention(qc.transpose(1, 2).to(sdpa_dt), kc.transpose(1, 2).to(sdpa_dt),
                                                              vc.transpose(1, 2).to(sdpa_dt)).float()
        oc = bfr(oc.transpose(1, 2).reshape(B, N, H * hd))
        h = h + matmul(oc, W.w_oc[l])
        mm = bfr(_rmsnorm(h, cfg.norm_eps) * (1 + sc2) + sh2)
        gu = matmul(mm, W.w_gu[l])
        gt, up = bfr(gu[..., 0::2]), bfr(gu[..., 1::2])
        hid = bfr(silu(gt) * up)
        h = h + g2 * (matmul(hid, W.w_down[l]))
    shf, scf = fmod[:, :d][:, None, :], fmod[:, d:][:, None, :]
    a = bfr(_rmsnorm(h, cfg.norm_eps) * (1 + scf) + shf)
    v = matmul(a, W.w_out)
    return v.reshape(B, T, C)


def reference_forward(dit, xs, ts, conds, layers: int = None, pure: bool = False) -> torch.Tensor:
    """forward_fp32 on a (GPU) ``paper_2605_28657_b200.dit.DiT``'s own bf16 weights, no TF32
    (pure=True: no bf16 rounding points anywhere -- the true fp32 network)."""
    prev = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    try:
        with torch.no_grad():
            return forward_fp32(dit.cfg, dit.weights, dit.frames, xs, ts, conds, layers, pure=pure)
    finally:
        torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = prev


class Fp32DiTVelocity:
    """The pure-fp32 DiT (``reference_forward(pure=True)`` on a GPU ``DiT``'s own weights and
    conditioning tokens) as the oracle pipeline's model (``oracle/ringflow_np.py``:
    ``Pipeline.model.velocity(x, t, cond, style, seed, stream, step)``): the trajectory
    reference for the bf16 GPU DiT.  The same conditioning as ``DiTVelocity`` (prompt tokens
    + 0.45 h hint + 0.45 tau timbre embeddings; the unconditional branch is prompt 0) and the
    same shared style offset in x0 space (v - style / t); no model jitter (the DiT path has
    none).  Runs on the GPU in fp32 for speed only -- it is the checker, never the product.
    ``log`` keeps (t, velocity) of every call when ``record`` is set."""

    def __init__(self, dit, record: bool = False):
        self.dit, self.record, self.log = dit, record, []

    def velocity(self, x, t, c, style, seed, stream, step):
        cond = self.dit.cond_tokens(c.prompt_hash, c.hint, c.timbre)
        xt = torch.from_numpy(np.ascontiguousarray(x)).to(self.dit.dev)
        v = reference_forward(self.dit, [xt], [t], [cond], pure=True)[0].double().cpu().numpy()
        if np.any(style != 0.0):
            v = v - style / t
        if self.record:
            self.log.append((float(t), v))
        return v


class CpuDiTVelocity:
    """The DiT as the oracle pipeline's model (``velocity(x, t, cond, style, seed, stream,
    step)`` like ``ringflow_np.Toy``): one CPU forward per ring row per step, seeded random-init
    weights of the config's shape (bf16-representable values).  bf16=True keeps the weights
    in bf16 and runs the GEMMs / attention with bf16 operands (the fastest CPU path: AMX on
    the GPU box's Xeon, 5x its fp32 GEMM rate); bf16=False is the fp32 oracle."""

    def __init__(self, cfg, frames: int, seed: int = 1234, bf16: bool = False):
        self.cfg, self.frames, self.bf16 = cfg, frames, bf16
        g = torch.Generator().manual_seed(seed)
        d, L, F = cfg.d_model, cfg.n_layers, cfg.mlp_hidden
        q, kv = cfg.n_heads * cfg.head_dim, cfg.n_kv_heads * cfg.head_dim

        def lin(*shape, std=None):
            s = std if std is not None else 1.0 / math.sqrt(shape[-1])
            w = (torch.randn(*shape, generator=g) * s).bfloat16()
            return w if bf16 else w.float()

        gate, up = lin(L, F, d), lin(L, F, d)
        self.W = SimpleNamespace(
            w_in=lin(d, cfg.in_dim), w_t1=lin(d, cfg.freq_dim), w_t2=lin(d, d), w_ada=lin(6 * d, d, std=0.02),
            ada_table=torch.randn(L, 6 * d, generator=g) * 0.1, w_qkv=lin(L, q + 2 * kv, d), w_o=lin(L, d, q),
            w_qc=lin(L, q, d), w_kvc=lin(L, 2 * kv, d), w_oc=lin(L, d, q),
            w_gu=torch.stack([gate, up], dim=2).reshape(L, 2 * F, d).contiguous(), w_down=lin(L, d, F),
            w_final_ada=lin(2 * d, d, std=0.02), w_out=lin(cfg.in_dim, d))
        self._cond = {}

    def cond_tokens(self, prompt_hash: int) -> torch.Tensor:
        t = self._cond.get(prompt_hash)
        if t is None:
            g = torch.Generator().manual_seed(int(prompt_hash) & ((1 << 62) - 1))
            t = torch.randn(self.cfg.n_cond_tokens, self.cfg.d_model, generator=g).bfloat16().float()
            self._cond[prompt_hash] = t
        return t

    def velocity(self, x, t, c, style, seed, stream, step):
        with torch.no_grad():
            v = forward_fp32(self.cfg, self.W, self.frames, [torch.from_numpy(np.ascontiguousarray(x))], [t],
                             [self.cond_tokens(c.prompt_hash)], f=lambda w: w, bf16_matmul=self.bf16)
        return v[0].double().numpy()
