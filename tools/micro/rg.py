import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_28657_b200 import tensor_ops as ops
M, N, K = 3000, 2048, 2048
A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
x = torch.zeros(M, N, device="cuda"); gate = torch.randn(4, N, device="cuda")
for _ in range(2):
    ops.gemm(A, B, out=x, epilogue=ops.EPI_RESID_GATE, gate=gate, rows_per_batch=750, block_n=256)
torch.cuda.synchronize()
