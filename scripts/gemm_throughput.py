"""Large-GEMM throughput of the tcgen05 kernel (no epilogue extras) against
cuBLAS (torch.matmul) on the same bf16 operands, CUDA-graph replays timed
with events:  python scripts/gemm_throughput.py
One JSON line per (shape, variant): us per GEMM, TFLOP/s, fraction of the
cuBLAS number for that shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_09732_b200._lib import check, lib

SHAPES = [(8192, 8192, 8192), (4096, 4096, 4096), (100352, 64, 576), (25088, 128, 1152), (6272, 256, 2304),
          (1568, 512, 4608), (100352, 256, 64), (25088, 512, 256)]
VARIANTS = [(64, 1, 1), (128, 1, 1), (256, 1, 1), (128, 1, -2), (256, 1, -2), (64, 1, -3), (128, 1, -3), (256, 1, -3)]


def timed(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn(torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * n)


def main():
    torch.manual_seed(0)
    for (M, N, K) in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        flop = 2.0 * M * N * K
        ref = A @ B.t()
        us_cublas = timed(lambda s: torch.matmul(A, B.t(), out=D))
        base = {"M": M, "N": N, "K": K}
        print(json.dumps({**base, "impl": "cublas", "us": round(us_cublas, 2),
                          "tflops": round(flop / us_cublas / 1e6, 1)}), flush=True)
        for (bn, splits, mc) in VARIANTS + [(0, 0, 1)]:
            if bn and N % bn:
                continue

            def run(s, bn=bn, splits=splits, mc=mc):
                check(lib.trims_gemm_bf16_ex(A.data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N, None, None,
                                             None, 0, 0, bn, splits, mc, s.cuda_stream))
            try:
                us = timed(run)
            except Exception as e:  # a variant the shape does not admit
                print(json.dumps({**base, "bn": bn, "mc": mc, "error": str(e)[:120]}), flush=True)
                continue
            err = ((D.float() - ref.float()).norm() / ref.float().norm()).item()
            print(json.dumps({**base, "impl": "trims", "bn": bn or "auto", "splits": splits, "mc": mc,
                              "us": round(us, 2), "tflops": round(flop / us / 1e6, 1),
                              "of_cublas": round(us_cublas / us, 3), "rel_err": float(f"{err:.2e}")}), flush=True)
        del A, B, D, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
