"""Per-kernel floor of a dependent chain in a CUDA graph: tiny tcgen05 GEMMs
(PDL launches) vs tiny torch elementwise kernels.
    python scripts/gemm_floor.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_09732_b200._lib import check, lib

res = {}
for (M, N, K) in [(128, 64, 64), (128, 64, 512), (3136, 64, 64), (784, 128, 1152)]:
    A = [torch.randn(M, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    n = 50
    with torch.cuda.stream(s):
        for _ in range(3):
            check(lib.trims_gemm_bf16(A[0].data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N, None, None, None,
                                      0, 0, 0, s.cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            check(lib.trims_gemm_bf16(A[i % 2].data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N, None, None,
                                      None, 0, 0, 0, torch.cuda.current_stream().cuda_stream))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res[f"gemm_{M}x{N}x{K}_us"] = round(e0.elapsed_time(e1) * 1e3 / (10 * n), 2)
x = torch.zeros(1024, device="cuda")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    x.add_(1)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    for _ in range(50):
        x.add_(1)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
res["torch_add_chain_us"] = round(e0.elapsed_time(e1) * 1e3 / 500, 2)
print(json.dumps(res))
