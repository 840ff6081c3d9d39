"""Per-tile timeline of one persistent GEMM launch (rf_gemm_set_trace: clock64 stamps per CTA
and tile): how long the MMA warp waits for a free accumulator (the epilogue is the bottleneck)
vs for operands (the TMA feed is), at the config-2 N = 2048 projection shape with the gated
residual epilogue (M = 3000, N = 2048, K = 2048; --K 6144 for the down projection).

    python tools/gemm_trace.py [--K 2048] [--bn -128] [--epi 2]"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28657_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=3000)
    ap.add_argument("--N", type=int, default=2048)
    ap.add_argument("--K", type=int, default=2048)
    ap.add_argument("--bn", type=int, default=-128)
    ap.add_argument("--epi", type=int, default=2)
    a = ap.parse_args()
    lib = _native.load()
    M, N, K = a.M, a.N, a.K
    A = (torch.randn(M, K, device="cuda") * 0.1).bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    h = torch.randn(M, N, device="cuda")
    gate = torch.ones(4, N, device="cuda")
    tr = torch.zeros(400 * 16 * 8, dtype=torch.int64, device="cuda")
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    st = vp(torch.cuda.current_stream().cuda_stream)

    def run():
        _native.check(lib.rf_gemm_bf16(vp(A.data_ptr()), vp(B.data_ptr()), vp(h.data_ptr()), i64(M), i64(N), i64(K),
                                       i64(K), i64(K), i64(N), a.epi, vp(gate.data_ptr()), i64(N), 750,
                                       ctypes.c_float(1.0), a.bn, st), "gemm")
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    print(f"M={M} N={N} K={K} bn={a.bn} epi={a.epi}: {e0.elapsed_time(e1) / 20 * 1e3:.2f} us per launch "
          f"({2.0 * M * N * K / (e0.elapsed_time(e1) / 20 * 1e-3) / 1e12:.0f} TF/s)")
    lib.rf_gemm_set_trace(vp(tr.data_ptr()))
    run()
    torch.cuda.synchronize()
    lib.rf_gemm_set_trace(vp(0))
    t = tr.view(400, 16, 8).cpu().numpy()
    ctas = [c for c in range(400) if t[c, 0, 0] > 0]
    # per tile (MMA warp of even CTAs): 0 start, 1 accumulator free, 2 first operands, 3 issued;
    # epilogue warp q = 2: 4 accumulator full, 5 done; producer: 6 tile start
    waits_acc, waits_op, issue, epi, gaps = [], [], [], [], []
    for c in ctas:
        for it in range(16):
            s = t[c, it]
            if s[0] == 0 or s[3] == 0:
                continue
            waits_acc.append(s[1] - s[0])
            waits_op.append(s[2] - s[1])
            issue.append(s[3] - s[2])
            if s[4] and s[5]:
                epi.append(s[5] - s[4])
    import statistics as S
    f = lambda v: f"mean {S.mean(v):8.0f}  max {max(v):8.0f}" if v else "-"  # noqa: E731
    print(f"tiles traced {len(issue)} over {len(ctas)} CTAs (clock cycles)")
    print(f"  MMA waits for a free accumulator : {f(waits_acc)}")
    print(f"  MMA waits for first operands      : {f(waits_op)}")
    print(f"  MMA issue span (all k blocks)     : {f(issue)}   ideal {K // 64} x 256 = {K // 64 * 256 if abs(a.bn) == 128 else K // 64 * 512}")
    print(f"  epilogue (acc full -> done, q=2)  : {f(epi)}")


if __name__ == "__main__":
    main()
