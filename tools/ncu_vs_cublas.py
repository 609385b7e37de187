"""One cfg2 layer step plus cuBLAS products of the same FLOPs (torch.matmul /
bmm), for `ncu --set full` side-by-side captures of our grouped tcgen05 GEMM
and cuBLAS's kernel on this B200 (tools/gpu_ncu_cublas.sh)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_13262_b200 as fm  # noqa: E402

n, d, h, E, k = 65536, 1024, 4096, 64, 2
rows = n * k
torch.cuda.set_device(0)
layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, E, 1, 42), dtype=torch.bfloat16)
x = (torch.rand(n, d, device="cuda") * 2 - 1).bfloat16()
dy = (torch.rand(n, d, device="cuda") * 2 - 1).bfloat16()
for _ in range(2):
    layer.forward(x)
    layer.backward(dy)
A2 = torch.randn(rows, h, device="cuda").bfloat16()
B2 = torch.randn(h, d, device="cuda").bfloat16()
Xm = torch.randn(E, d, rows // E, device="cuda").bfloat16()
Dp = torch.randn(E, rows // E, h, device="cuda").bfloat16()
S = torch.randn(8192, 8192, device="cuda").bfloat16()
for _ in range(2):  # warm-up (cuBLAS heuristics, workspaces)
    torch.matmul(A2, B2)
    torch.bmm(Xm, Dp)
    torch.matmul(S, S)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("cublas")  # ncu --nvtx-include cublas/ captures these three
torch.matmul(A2, B2)          # fc2 shape
torch.bmm(Xm, Dp)             # wgrad_fc1 shape (K-major A)
torch.matmul(S, S)            # MEASURED_PEAKS' burst shape
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
