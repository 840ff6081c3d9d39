"""Self-attention kernels at BASELINE config-2 shape (4 rows x 750 tokens, 16 / 8 heads of 128):
device time (20 launches per CUDA graph replay, median of 10) and rel-RMS vs SDPA of the
self-attention kernel (rf_attention_tc_bf16_kernel).
python tools/attn_bench.py [B N]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
N = int(sys.argv[2]) if len(sys.argv) > 2 else 750
H, Hk = 16, 8
lib = _native.load()
lib.rf_attention_tc_bf16_kernel.restype = ctypes.c_int
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(B * N, H * 128, device="cuda", generator=g).bfloat16()
k = torch.randn(B * N, Hk * 128, device="cuda", generator=g).bfloat16()
v = torch.randn(B * N, Hk * 128, device="cuda", generator=g).bfloat16()
npad = (N + 7) // 8 * 8
vt = torch.zeros(B, Hk, 128, npad, device="cuda", dtype=torch.bfloat16)
vt[..., :N] = v.reshape(B, N, Hk, 128).permute(0, 2, 3, 1)
out = torch.empty(B * N, H * 128, device="cuda", dtype=torch.bfloat16)
qq = q.float().reshape(B, N, H, 128).transpose(1, 2)
kk = k.float().reshape(B, N, Hk, 128).repeat_interleave(H // Hk, 2).transpose(1, 2)
vv = v.float().reshape(B, N, Hk, 128).repeat_interleave(H // Hk, 2).transpose(1, 2)
ref = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv).transpose(1, 2).reshape(B * N, H * 128)
flops = 4.0 * B * H * N * N * 128
vp, i64 = ctypes.c_void_p, ctypes.c_int64
st = torch.cuda.current_stream().cuda_stream


def run(kern):
    _native.check(lib.rf_attention_tc_bf16_kernel(kern, vp(q.data_ptr()), vp(k.data_ptr()), vp(vt.data_ptr()),
                                                  vp(out.data_ptr()), B, N, N, npad, H, Hk, i64(H * 128),
                                                  i64(Hk * 128), i64(H * 128), vp(st)), "attn")


print(f"B={B} N={N}")
for kern, name in ((0, "fa64 (default)"),):
    for _ in range(3):
        run(kern)
    torch.cuda.synchronize()
    # device time: 20 launches captured in a CUDA graph (the per-call host planning -- tensor
    # maps, split rule -- is slower than the kernel, so eager launches would time the host)
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        st = gs.cuda_stream
        run(kern)
        with torch.cuda.graph(graph, stream=gs):
            for _ in range(20):
                run(kern)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    us = sorted(x.elapsed_time(y) for x, y in ts)[5] * 1e3 / 20
    err = ((out.float() - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()).item()
    print(f"{name:26s} {us:8.2f} us  {flops / us / 1e6:8.1f} TF/s  rel-rms {err:.2e}", flush=True)
