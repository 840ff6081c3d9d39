"""Library baseline for the DiT forward: the same network (same weights, same bf16 rounding
points) written with stock PyTorch ops -- cuBLAS bf16 GEMMs, SDPA (flash / cuDNN backends,
GQA), elementwise RMSNorm / AdaLN / SwiGLU / RoPE in torch -- captured as one CUDA graph and
timed with CUDA events.  This is the "call the libraries" implementation the hand-written
tcgen05 forward (csrc/rf_dit.cu) is measured against; it is a measurement tool only.

usage: python tools/dit_torch_baseline.py [rows]
"""
import math
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import dit as D  # noqa: E402
from oracle.dit_fp32 import reference_forward  # noqa: E402


def build(dit, xs, ts, conds):
    cfg, W = dit.cfg, dit.weights
    B, T, C = len(xs), dit.frames, cfg.latent_channels
    N, d = T // cfg.patch, cfg.d_model
    H, Hk, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    dev = xs[0].device
    x_in = torch.stack(xs)
    cond = torch.stack(conds)                       # [B, Nc, d] bf16
    t_in = torch.tensor([float(t) for t in ts], device=dev)
    half = cfg.freq_dim // 2
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, device=dev, dtype=torch.float32) / half)
    pos = torch.arange(N, device=dev, dtype=torch.float64)
    inv = torch.pow(torch.tensor(cfg.rope_theta, dtype=torch.float64),
                    -2.0 * torch.arange(64, device=dev, dtype=torch.float64) / 128.0)
    ang = pos[:, None] * inv[None]
    cos = torch.cos(ang).float()[None, :, None, :]
    sin = torch.sin(ang).float()[None, :, None, :]
    # all layers' cross K/V in one GEMM, as the native forward does
    w_kvc_all = W.w_kvc.reshape(-1, d)

    def rms(x):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + cfg.norm_eps)

    def rope(x):
        xf = x.float()
        x0, x1 = xf[..., 0::2], xf[..., 1::2]
        return torch.stack([x0 * cos - x1 * sin, x0 * sin + x1 * cos], -1).flatten(-2).bfloat16()

    def fwd():
        x = x_in.float().reshape(B, N, cfg.in_dim).bfloat16()
        args = 1000.0 * t_in[:, None] * freqs[None]
        tf = torch.cat([torch.cos(args), torch.sin(args)], -1).bfloat16()
        temb = F.silu(tf @ W.w_t1.T) @ W.w_t2.T
        st = F.silu(temb)
        mod = (st @ W.w_ada.T).float()
        fmod = (st @ W.w_final_ada.T).float()
        h = (x @ W.w_in.T).float()
        kv_all = (cond @ w_kvc_all.T).reshape(B, -1, cfg.n_layers, 2 * Hk * hd)
        for l in range(cfg.n_layers):
            m = mod + W.ada_table[l][None]
            sh1, sc1, g1, sh2, sc2, g2 = [m[:, i * d:(i + 1) * d][:, None, :] for i in range(6)]
            a = (rms(h) * (1 + sc1) + sh1).bfloat16()
            qkv = a @ W.w_qkv[l].T
            q = rope(qkv[..., :H * hd].reshape(B, N, H, hd))
            k = rope(qkv[..., H * hd:(H + Hk) * hd].reshape(B, N, Hk, hd))
            v = qkv[..., (H + Hk) * hd:].reshape(B, N, Hk, hd)
            o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                               enable_gqa=True)
            o = o.transpose(1, 2).reshape(B, N, H * hd)
            h = h + g1 * (o @ W.w_o[l].T).float()
            c = rms(h).bfloat16()
            qc = (c @ W.w_qc[l].T).reshape(B, N, H, hd)
            kvc = kv_all[:, :, l]
            kc = kvc[..., :Hk * hd].reshape(B, -1, Hk, hd)
            vc = kvc[..., Hk * hd:].reshape(B, -1, Hk, hd)
            oc = F.scaled_dot_product_attention(qc.transpose(1, 2), kc.transpose(1, 2), vc.transpose(1, 2),
                                                enable_gqa=True)
            oc = oc.transpose(1, 2).reshape(B, N, H * hd)
            h = h + (oc @ W.w_oc[l].T).float()
            mm = (rms(h) * (1 + sc2) + sh2).bfloat16()
            gu = mm @ W.w_gu[l].T
            hid = F.silu(gu[..., 0::2]) * gu[..., 1::2]
            h = h + g2 * (hid @ W.w_down[l].T).float()
        shf, scf = fmod[:, :d][:, None, :], fmod[:, d:][:, None, :]
        a = (rms(h) * (1 + scf) + shf).bfloat16()
        return (a @ W.w_out.T).float().reshape(B, T, C)

    return fwd


def compare(rows=4, n=20, check=True):
    """Native forward vs the torch-library forward on the same weights and inputs: device
    ms per forward (CUDA graphs, CUDA events) and rel-RMS of each against the fp32 oracle."""
    with torch.cuda.stream(torch.cuda.Stream()):   # non-default stream: the native forward replays its graph
        return _compare(rows, n, check)


def _compare(rows, n, check):
    cfg = D.DiTConfig()
    dit = D.DiT(cfg, frames=1500, max_rows=max(rows, 4))
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(1500, 64, device="cuda", generator=g, dtype=torch.float64) for _ in range(rows)]
    ts = [1.0 - 0.1 * i for i in range(rows)]
    conds = [dit.cond_tokens(i) for i in range(rows)]
    fwd = build(dit, xs, ts, conds)
    out = {}
    with torch.no_grad():
        if check:
            ours = dit.forward(xs, ts, conds).clone()
            lib = fwd()
            ref = reference_forward(dit, xs, ts, conds)
            rr = lambda a: ((a - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()).item()  # noqa: E731
            out["rel_rms_vs_fp32"] = {"native": float(f"{rr(ours):.4g}"), "torch_library": float(f"{rr(lib):.4g}")}
            del ref, ours, lib
        s = torch.cuda.current_stream()
        for _ in range(3):
            fwd()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            fwd()
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
    fl = cfg.flops_per_forward(rows, 1500)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, call in (("torch_library_ms", graph.replay), ("native_ms", lambda: dit.forward(xs, ts, conds))):
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        a.record()
        for _ in range(n):
            call()
        b.record()
        torch.cuda.synchronize()
        out[name] = round(a.elapsed_time(b) / n, 4)
    out["torch_library_tflops"] = round(fl / out["torch_library_ms"] / 1e9, 1)
    out["native_tflops"] = round(fl / out["native_ms"] / 1e9, 1)
    out["speedup"] = round(out["torch_library_ms"] / out["native_ms"], 3)
    del graph, fwd, dit
    torch.cuda.empty_cache()
    return out


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    r = compare(rows)
    print(f"rows={rows} rel-RMS vs fp32 oracle: native {r['rel_rms_vs_fp32']['native']:.3e}  "
          f"torch-library {r['rel_rms_vs_fp32']['torch_library']:.3e}")
    print(f"rows={rows} torch-library (cuBLAS + SDPA, CUDA graph) {r['torch_library_ms']:8.3f} ms "
          f"{r['torch_library_tflops']:7.1f} TFLOP/s")
    print(f"rows={rows} native tcgen05 forward (CUDA graph)       {r['native_ms']:8.3f} ms "
          f"{r['native_tflops']:7.1f} TFLOP/s")
    print(f"speed-up native / torch-library: {r['speedup']:.3f}x")


if __name__ == "__main__":
    main()
