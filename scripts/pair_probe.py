import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1811_09732_b200._lib import lib, check
M, N, K, bn = 256, 128, 64, 128
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
D = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
check(lib.trims_gemm_bf16_ex(A.data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N, None, None, None, N, 0, bn, 1, -2, None))
torch.cuda.synchronize()
ref = (A.float() @ B.float().T)
print("max err", (D.float() - ref).abs().max().item(), "ref max", ref.abs().max().item())
print("row0-127 err", (D.float() - ref)[:128].abs().max().item(), "row128-255 err", (D.float() - ref)[128:].abs().max().item())
