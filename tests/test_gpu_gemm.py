"""K7 tcgen05 GEMM (bf16 in, fp32 TMEM accumulate, fused epilogue) vs a plain
PyTorch fp32 reference of the same op. Tolerance: the output is rounded to
bf16 once, so |out - ref| <= 2^-8 |ref| + 1e-3 * max|ref| (one bf16 ulp of
the value plus fp32 summation-order noise)."""
import pytest

from paper_1811_09732_b200._lib import check, lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K,bn", [
    (128, 64, 64, 64), (256, 128, 128, 128), (300, 200, 96, 64), (1000, 256, 576, 256),
    (49, 2048, 512, 64), (3136, 64, 576, 64), (17, 1000, 4096, 128), (777, 384, 2304, 128),
    (512, 512, 1024, 256),
    # 33 k-blocks over 8 splits of ceil(33/8) = 5: the last split owns none
    (49, 512, 2112, 64), (49, 512, 2112, 128),
])
@pytest.mark.parametrize("epi", ["plain", "full"])
def test_gemm_matches_fp32_reference(M, N, K, bn, epi):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    scale = bias = res = None
    ref = A.float() @ B.float().T
    if epi == "full":
        scale = torch.rand(N, device="cuda", generator=g) + 0.5
        bias = torch.randn(N, device="cuda", generator=g)
        res = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
        ref = torch.relu(ref * scale + bias + res.float())
    check(lib.trims_gemm_bf16(A.data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N,
                              scale.data_ptr() if scale is not None else None,
                              bias.data_ptr() if bias is not None else None,
                              res.data_ptr() if res is not None else None, N, int(epi == "full"), bn,
                              torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    out = D.float()
    assert torch.isfinite(out).all()
    err = (out - ref).abs()
    tol = ref.abs() * 2 ** -8 + 1e-3 * ref.abs().max()
    assert (err <= tol).all(), f"max err {err.max().item()} (ref max {ref.abs().max().item()})"


@pytest.mark.parametrize("M,N,K,bn,splits", [
    (49, 512, 4608, 64, 8), (49, 512, 2048, 128, 8), (196, 256, 2304, 64, 8), (196, 256, 1024, 128, 4),
    (784, 128, 1152, 128, 4), (3136, 64, 576, 64, 2), (300, 200, 1024, 64, 4), (17, 1000, 4096, 128, 2),
    # 33 k-blocks over 8 splits of ceil(33/8) = 5: the last split owns none
    (49, 512, 2112, 64, 8), (49, 512, 2112, 128, 8),
])
@pytest.mark.parametrize("epi", ["plain", "full"])
def test_gemm_split_k_matches_fp32_reference(M, N, K, bn, splits, epi):
    """Split-K through the C ABI (trims_gemm_bf16_split): the S splits of a
    tile reduce their fp32 partials in split order inside one cluster. Same
    tolerance as above; two launches are bit-identical (deterministic order)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 5 + N + K + splits)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    scale = bias = res = None
    ref = A.float() @ B.float().T
    if epi == "full":
        scale = torch.rand(N, device="cuda", generator=g) + 0.5
        bias = torch.randn(N, device="cuda", generator=g)
        res = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
        ref = torch.relu(ref * scale + bias + res.float())
    outs = []
    for _ in range(2):
        D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        check(lib.trims_gemm_bf16_split(A.data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N,
                                        scale.data_ptr() if scale is not None else None,
                                        bias.data_ptr() if bias is not None else None,
                                        res.data_ptr() if res is not None else None, N, int(epi == "full"), bn,
                                        splits, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        outs.append(D)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    out = outs[0].float()
    assert torch.isfinite(out).all()
    err = (out - ref).abs()
    tol = ref.abs() * 2 ** -8 + 1e-3 * ref.abs().max()
    assert (err <= tol).all(), f"max err {err.max().item()} (ref max {ref.abs().max().item()})"


def test_gemm_split_count_validated():
    import torch
    A = torch.zeros(128, 64, device="cuda", dtype=torch.bfloat16)
    D = torch.zeros(128, 64, device="cuda", dtype=torch.bfloat16)
    for bn, splits in ((64, 3), (64, 16), (256, 2)):
        rc = lib.trims_gemm_bf16_split(A.data_ptr(), 128, 64, 64, A.data_ptr(), 64, 64, D.data_ptr(), 64, None, None,
                                       None, 64, 0, bn, splits, None)
        assert rc != 0


@pytest.mark.parametrize("M,N,K,bn,splits,mc", [
    (3136, 256, 2304, 128, 2, 4), (784, 512, 4608, 128, 4, 2), (12544, 128, 1152, 128, 1, 4),
    (12544, 64, 576, 64, 1, 8), (3000, 200, 1024, 64, 2, 4), (700, 96, 640, 64, 1, 4),
    # tile rows not a multiple of the group: padding tiles (no rows) take part in the multicast
    (300, 256, 1024, 64, 2, 4), (1000, 128, 576, 128, 1, 8),
])
@pytest.mark.parametrize("epi", ["plain", "full"])
def test_gemm_weight_multicast_matches_fp32_reference(M, N, K, bn, splits, mc, epi):
    """Weight multicast (trims_gemm_bf16_ex): mc consecutive M-tiles share each
    B stage by TMA multicast; same tolerance, equal to the unshared launch."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + N * 3 + K + mc)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    scale = bias = res = None
    ref = A.float() @ B.float().T
    if epi == "full":
        scale = torch.rand(N, device="cuda", generator=g) + 0.5
        bias = torch.randn(N, device="cuda", generator=g)
        res = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
        ref = torch.relu(ref * scale + bias + res.float())
    outs = []
    for m in (mc, 1):
        D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        check(lib.trims_gemm_bf16_ex(A.data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N,
                                     scale.data_ptr() if scale is not None else None,
                                     bias.data_ptr() if bias is not None else None,
                                     res.data_ptr() if res is not None else None, N, int(epi == "full"), bn,
                                     splits, m, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        outs.append(D)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)), "multicast changed the result"
    out = outs[0].float()
    assert torch.isfinite(out).all()
    err = (out - ref).abs()
    tol = ref.abs() * 2 ** -8 + 1e-3 * ref.abs().max()
    assert (err <= tol).all(), f"max err {err.max().item()} (ref max {ref.abs().max().item()})"


@pytest.mark.parametrize("M,N,K,bn", [
    (256, 128, 64, 128), (512, 256, 576, 256), (3136, 128, 1152, 128), (1000, 256, 2304, 256),
    # an odd number of M-tiles: the last pair has a padding CTA with no rows
    (300, 128, 512, 128), (12544, 64 * 3, 576, 128),
])
@pytest.mark.parametrize("epi", ["plain", "full"])
def test_gemm_two_sm_pair_matches_fp32_reference(M, N, K, bn, epi):
    """2-SM pairs (trims_gemm_bf16_ex with mc = -2): tcgen05.mma.cta_group::2
    with M = 256 over two CTAs of one cluster, each loading its 128 rows of A
    and half of B; same tolerance, bit-identical to the single-CTA launch."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 11 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    scale = bias = res = None
    ref = A.float() @ B.float().T
    if epi == "full":
        scale = torch.rand(N, device="cuda", generator=g) + 0.5
        bias = torch.randn(N, device="cuda", generator=g)
        res = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
        ref = torch.relu(ref * scale + bias + res.float())
    outs = []
    for m in (-2, 1):
        D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        check(lib.trims_gemm_bf16_ex(A.data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N,
                                     scale.data_ptr() if scale is not None else None,
                                     bias.data_ptr() if bias is not None else None,
                                     res.data_ptr() if res is not None else None, N, int(epi == "full"), bn,
                                     1, m, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        outs.append(D)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)), "the pair changed the result"
    out = outs[0].float()
    err = (out - ref).abs()
    tol = ref.abs() * 2 ** -8 + 1e-3 * ref.abs().max()
    assert (err <= tol).all(), f"max err {err.max().item()} (ref max {ref.abs().max().item()})"


@pytest.mark.parametrize("M,N,K,bn", [
    (256, 128, 64, 128),            # fewer tiles than SMs: one tile per CTA
    (40000, 256, 64, 256),          # 313 tiles: 2-3 per CTA, both accumulators, K = one k-block
    (25088, 512, 256, 256),         # 392 tiles
    (100352, 64, 576, 64),          # 784 tiles, ring phases wrap across tiles
    (3000, 128, 1152, 128),         # ragged last M-tile
    (20000, 192, 128, 128),         # partial last N-tile
])
@pytest.mark.parametrize("epi", ["plain", "full"])
def test_gemm_persistent_matches_fp32_reference(M, N, K, bn, epi):
    """Persistent launch (trims_gemm_bf16_ex with mc = -3): one CTA per SM over
    all output tiles, two TMEM accumulators (tile i's epilogue overlaps tile
    i+1's k-loop); same tolerance, bit-identical to one CTA per tile."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    scale = bias = res = None
    ref = A.float() @ B.float().T
    if epi == "full":
        scale = torch.rand(N, device="cuda", generator=g) + 0.5
        bias = torch.randn(N, device="cuda", generator=g)
        res = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
        ref = torch.relu(ref * scale + bias + res.float())
    outs = []
    for m in (-3, 1):
        D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        check(lib.trims_gemm_bf16_ex(A.data_ptr(), M, K, K, B.data_ptr(), N, K, D.data_ptr(), N,
                                     scale.data_ptr() if scale is not None else None,
                                     bias.data_ptr() if bias is not None else None,
                                     res.data_ptr() if res is not None else None, N, int(epi == "full"), bn,
                                     1, m, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        outs.append(D)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)), "the persistent launch changed the result"
    out = outs[0].float()
    err = (out - ref).abs()
    tol = ref.abs() * 2 ** -8 + 1e-3 * ref.abs().max()
    assert (err <= tol).all(), f"max err {err.max().item()} (ref max {ref.abs().max().item()})"
