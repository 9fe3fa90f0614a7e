"""Kernel-level parity of the tcgen05 GEMMs (bf16 kind::f16 and the fp32 mode's split-TF32 (4 MMAs) kind::tf32) (§8(a) a7 forward update φ = W·CONCAT(z, h), PAPER.md:100 / Alg.1 l.10
PAPER.md:287; a9 its gradients, Alg.1 l.12 PAPER.md:290) through the C ABI entry bns_gemm, which launches the same
kernels as bns_epoch.  Expected values: a float64 product (torch, cuBLAS DGEMM) of the SAME bf16 operands -- the
definition, independent of the kernel.  No ReLU flips or epoch trajectories are involved, so the bar is the fp32
accumulation error alone:

* fp32 outputs (forward with fp32 epilogue, dW, and every output of the fp32 mode's split-TF32 (4 MMAs) kernels):
  normwise max|gpu - f64| / max|f64| <= 1e-5 -- for split-TF32 (4 MMAs) that is the fp32 mode's own bar (one-pass TF32 is ~1e-3);
* bf16 outputs (forward, dX): correctly rounded up to that accumulation error, i.e.
  max(|gpu - f64| - ulp_bf16(f64)/2) / max|f64| <= 1e-5.

Shapes are the bench's (Reddit-shaped, m = 1: M = 232,965 stacked rows, a ragged last 128-row tile; widths 608 /
512 / 256 / 48 padded) and the weight-gradient GEMMs run with the split-K factor the epoch uses (>= 32 slices on the
256-wide layers).  The bf16 GEMMs run both as single CTAs and as CTA pairs sharing the B operand by TMA multicast
(BNS_GEMM_MC=2; by default pairs are used from 256 K rows).
"""
import numpy as np
import pytest

from paper_2203_10983_b200 import bns

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

M_FULL = 232_965
TOL = 1e-5


def rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def rel_rounded(g, r):
    """bf16 output g vs float64 r: excess over half a bf16 ulp of r, normwise."""
    g = g.double()
    r = r.double()
    e = torch.floor(torch.log2(r.abs().clamp_min(1e-30)))
    half_ulp = torch.pow(2.0, e - 8)            # bf16: 8 significant bits -> ulp = 2^(e-7)
    excess = ((g - r).abs() - half_ulp).clamp_min(0)
    return float(excess.max() / r.abs().max().clamp_min(1e-30))


def act(M, K, g, zero_frac=0.5):
    """post-ReLU-like operand: non-negative, about half zeros"""
    x = torch.rand(M, K, generator=g, device="cpu", dtype=torch.float32)
    x[torch.rand(M, K, generator=g) < zero_frac] = 0
    return x.to("cuda").to(torch.bfloat16)


def sgn(M, K, g, scale=1.0):
    return (torch.randn(M, K, generator=g) * scale).to("cuda").to(torch.bfloat16)


def wt_pad(W, halves):
    """B = W^T stored [N][Kw], each concat half of W's K rows zero-padded to a multiple of 64 columns"""
    K2, N = W.shape
    K = K2 // halves
    Kp = (K + 63) // 64 * 64
    B = torch.zeros(N, halves * Kp, dtype=torch.bfloat16, device="cuda")
    for h in range(halves):
        B[:, h * Kp:h * Kp + K] = W[h * K:(h + 1) * K].t()
    return B.contiguous()


@pytest.mark.parametrize("K,N,concat,relu,out_f32", [
    (608, 512, False, False, True),    # layer 1 transform-first [Y | S] = H [W_top | W_bot]
    (608, 512, False, False, False),
    (256, 256, True, True, False),     # aggregate-first hidden layer: ReLU([Z | H] W), bf16 out
    (256, 256, True, False, True),
    (256, 96, False, False, False),    # layer 4 transform-first, 48-wide halves
])
@pytest.mark.parametrize("mc", ["1", "2"])
def test_forward(K, N, concat, relu, out_f32, mc, monkeypatch):
    monkeypatch.setenv("BNS_GEMM_MC", mc)   # 2: CTA pairs sharing B by TMA multicast
    g = torch.Generator().manual_seed(K * 7 + N)
    M = M_FULL
    A0 = act(M, K, g)
    A1 = act(M, K, g) if concat else None
    W = sgn(2 * K if concat else K, N, g, 0.05)
    C = torch.empty(M, N, dtype=torch.float32 if out_f32 else torch.bfloat16, device="cuda")
    B = wt_pad(W, 2 if concat else 1)
    bns.bns_gemm(bns.BNS_BF16, bns.BNS_GEMM_FWD, M, N, K, A0, A1, K, B, B.shape[1], C, N,
                 flags=(1 if relu else 0) | (2 if out_f32 else 0))
    torch.cuda.synchronize()
    X = torch.cat([A0, A1], 1) if concat else A0
    ref = X.double() @ W.double()
    if relu:
        ref = ref.clamp_min(0)
    e = rel(C, ref) if out_f32 else rel_rounded(C, ref)
    assert e <= TOL, e


@pytest.mark.parametrize("M,K,N,min_splits", [
    (M_FULL, 256, 256, 32),   # hidden-layer dW (Reddit 4 x 256)
    (M_FULL, 608, 256, 16),   # layer-1 dW_top = H^T dY (transform-first)
    (M_FULL, 256, 48, 32),    # last layer
    (29_121, 256, 256, 4),    # an m = 8 partition
    (1000, 64, 16, 1),        # tiny: a single split, ragged K block
])
@pytest.mark.parametrize("mc", ["1", "2"])
def test_wgrad(M, K, N, min_splits, mc, monkeypatch):
    monkeypatch.setenv("BNS_GEMM_MC", mc)   # 2: CTA pairs sharing B by TMA multicast
    g = torch.Generator().manual_seed(M + K + N)
    A = act(M, K, g)
    D = sgn(M, N, g, 1e-3)
    C = torch.full((K, N), float("nan"), dtype=torch.float32, device="cuda")
    S = bns.bns_gemm(bns.BNS_BF16, bns.BNS_GEMM_WGRAD, M, N, K, A, None, K, D, N, C, N)
    torch.cuda.synchronize()
    assert S >= min_splits, S
    e = rel(C, A.double().t() @ D.double())
    assert e <= TOL, (e, S)


@pytest.mark.parametrize("M,K,N", [(M_FULL, 256, 256), (M_FULL, 128, 48), (5000, 128, 128)])
@pytest.mark.parametrize("mc", ["1", "2"])
def test_wgrad_merged(M, K, N, mc, monkeypatch):
    monkeypatch.setenv("BNS_GEMM_MC", mc)   # 2: CTA pairs sharing B by TMA multicast
    """GraphSAGE [dW_z ; dW_h] = [Z | H]^T dPre in one launch + one split-K reduce"""
    g = torch.Generator().manual_seed(3 * M + K)
    Z = sgn(M, K, g)
    H = act(M, K, g)
    D = sgn(M, N, g, 1e-3)
    C = torch.full((2 * K, N), float("nan"), dtype=torch.float32, device="cuda")
    S = bns.bns_gemm(bns.BNS_BF16, bns.BNS_GEMM_WGRAD2, M, N, K, Z, H, K, D, N, C, N)
    torch.cuda.synchronize()
    if M == M_FULL and N == 256:
        assert S >= 32, S
    e = rel(C, torch.cat([Z, H], 1).double().t() @ D.double())
    assert e <= TOL, (e, S)


@pytest.mark.parametrize("M,K,N,scale_cols", [(M_FULL, 256, 512, 256), (M_FULL, 48, 512, 0), (M_FULL, 256, 256, 256),
                                              (777, 48, 96, 48)])
@pytest.mark.parametrize("mc", ["1", "2"])
def test_dx(M, K, N, scale_cols, mc, monkeypatch):
    monkeypatch.setenv("BNS_GEMM_MC", mc)   # 2: CTA pairs sharing B by TMA multicast
    """[dZ' | dX_self] = dPre W^T with the 1/deg_G row scale on the dZ' half (SAGE), or dY-side products"""
    g = torch.Generator().manual_seed(M * 5 + N)
    D = sgn(M, K, g, 1e-3)
    W = sgn(N, K, g, 0.05)                 # B = W stored [N][K] (the update's rows are this GEMM's columns)
    rs = (1.0 / torch.randint(1, 5000, (M,), generator=g).float()).to("cuda") if scale_cols else None
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    bns.bns_gemm(bns.BNS_BF16, bns.BNS_GEMM_DX, M, N, K, D, None, K, W, K, C, N, rowscale=rs, scale_cols=scale_cols)
    torch.cuda.synchronize()
    ref = D.double() @ W.double().t()
    if scale_cols:
        ref[:, :scale_cols] *= rs.double()[:, None]
    e = rel_rounded(C[:, :scale_cols] if scale_cols else C, ref[:, :scale_cols] if scale_cols else ref)
    assert e <= TOL, e
    if scale_cols and scale_cols < N:
        e = rel_rounded(C[:, scale_cols:], ref[:, scale_cols:])
        assert e <= TOL, e


def test_gemm_rejects_bad_arguments():
    x = torch.zeros(128, 128, dtype=torch.bfloat16, device="cuda")
    for args in [(7, bns.BNS_GEMM_FWD, 128, 128, 128), (bns.BNS_BF16, 9, 128, 128, 128),
                 (bns.BNS_BF16, bns.BNS_GEMM_WGRAD2, 128, 128, 64)]:
        with pytest.raises(bns.BnsError) as e:
            bns.bns_gemm(*args, x, x, 128, x, 128, x, 128)
        assert e.value.code == bns.BNS_ERR_INVALID


# ---------------- fp32 mode: split-TF32 (4 MMAs) (tcgen05 kind::tf32 on hi / lo operand splits) ----------------
def f32(t):
    return t.float().contiguous()


@pytest.mark.parametrize("K,N,concat,relu", [(608, 512, False, False), (256, 256, True, True), (256, 96, False, False),
                                             (40, 24, True, False)])   # an 8-padded narrow layer
def test_forward_fp32(K, N, concat, relu):
    g = torch.Generator().manual_seed(K * 11 + N)
    M = M_FULL if K >= 256 else 3001
    A0 = f32(torch.randn(M, K, generator=g).cuda())
    A1 = f32(torch.randn(M, K, generator=g).cuda()) if concat else None
    W = f32(torch.randn(2 * K if concat else K, N, generator=g).cuda() * 0.05)
    halves = 2 if concat else 1
    Kp = (K + 63) // 64 * 64
    B = torch.zeros(N, halves * Kp, dtype=torch.float32, device="cuda")
    for h in range(halves):
        B[:, h * Kp:h * Kp + K] = W[h * K:(h + 1) * K].t()
    C = torch.empty(M, N, dtype=torch.float32, device="cuda")
    bns.bns_gemm(bns.BNS_FP32, bns.BNS_GEMM_FWD, M, N, K, A0, A1, K, B, B.shape[1], C, N, flags=1 if relu else 0)
    torch.cuda.synchronize()
    X = torch.cat([A0, A1], 1) if concat else A0
    ref = X.double() @ W.double()
    if relu:
        ref = ref.clamp_min(0)
    e = rel(C, ref)
    assert e <= TOL, e


@pytest.mark.parametrize("M,K,N,merged", [(M_FULL, 256, 256, False), (M_FULL, 608, 256, False), (29_121, 256, 48, False),
                                          (M_FULL, 256, 256, True), (1000, 128, 16, True)])
def test_wgrad_fp32(M, K, N, merged):
    g = torch.Generator().manual_seed(M + 3 * K + N)
    A0 = f32(torch.randn(M, K, generator=g).cuda().clamp_min(0))
    A1 = f32(torch.randn(M, K, generator=g).cuda()) if merged else None
    D = f32(torch.randn(M, N, generator=g).cuda() * 1e-3)
    C = torch.full(((2 if merged else 1) * K, N), float("nan"), dtype=torch.float32, device="cuda")
    S = bns.bns_gemm(bns.BNS_FP32, bns.BNS_GEMM_WGRAD2 if merged else bns.BNS_GEMM_WGRAD, M, N, K, A0, A1, K, D, N, C, N)
    torch.cuda.synchronize()
    X = torch.cat([A0, A1], 1) if merged else A0
    e = rel(C, X.double().t() @ D.double())
    assert e <= TOL, (e, S)


@pytest.mark.parametrize("M,K,N,scale_cols", [(M_FULL, 256, 512, 256), (M_FULL, 48, 512, 0), (777, 48, 96, 48)])
def test_dx_fp32(M, K, N, scale_cols):
    g = torch.Generator().manual_seed(M * 7 + N)
    D = f32(torch.randn(M, K, generator=g).cuda() * 1e-3)
    W = f32(torch.randn(N, K, generator=g).cuda() * 0.05)
    rs = (1.0 / torch.randint(1, 5000, (M,), generator=g).float()).cuda() if scale_cols else None
    C = torch.empty(M, N, dtype=torch.float32, device="cuda")
    bns.bns_gemm(bns.BNS_FP32, bns.BNS_GEMM_DX, M, N, K, D, None, K, W, K, C, N, rowscale=rs, scale_cols=scale_cols)
    torch.cuda.synchronize()
    ref = D.double() @ W.double().t()
    if scale_cols:
        ref[:, :scale_cols] *= rs.double()[:, None]
    e = rel(C, ref)
    assert e <= TOL, e
