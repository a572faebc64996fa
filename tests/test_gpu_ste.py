"""GPU parity of the NEXT-4 STE backward (axq_ste_linear_backward) against the oracle.  fp32 FMA
sums in a different order than the oracle's fp64 products: each gradient must lie within the
fp32 dot-product bound gamma_n * sum|terms| (n = summed length, gamma_n = n u / (1 - n u),
u = 2^-24) plus the oracle's own final rounding."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda"
U = 2.0 ** -24


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _bound(n, absprod, ref):
    g = n * U / (1 - n * U)
    return g * absprod + U * np.abs(ref) + 1e-30


def _check(ax, M, N, K, seed, masked, split):
    x = datagen.normal(60 + seed, 1, (M, K))
    W = datagen.normal(60 + seed, 2, (N, K), 0.05)
    qa, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(W, 8)
    gy = datagen.normal(60 + seed, 3, (M, N))
    clip_a = np.float32(np.quantile(np.abs(x), 0.8)) if masked and x.size else np.float32(0)
    clip_w = np.float32(np.quantile(np.abs(W), 0.8)) if masked and W.size else np.float32(0)
    if masked:
        ref = oracle.ste_linear_backward(gy, qa, sa, qw, sw, x, clip_a, W, clip_w)
    else:
        ref = oracle.ste_linear_backward(gy, qa, sa, qw, sw)
    gx = torch.full((M, K), np.nan, device=DEV)
    gw = torch.full((N, K), np.nan, device=DEV)
    gb = torch.full((N,), np.nan, device=DEV)
    f = lambda v: _t(np.array([v], dtype=np.float32))
    kw = dict(x=_t(x), d_clip_a=f(clip_a), w=_t(W), d_clip_w=f(clip_w)) if masked else {}
    ws = torch.full((16 * max(M, N) * K,), np.nan, device=DEV) if split else None
    ax.axq_ste_linear_backward(_t(gy), _t(qa), f(sa), _t(qw), f(sw), gx=gx, gw=gw, gb=gb,
                               workspace=ws, **kw)
    torch.cuda.synchronize()
    wf, xf = np.abs(oracle.fake_quant(qw, sw)).astype(np.float64), np.abs(oracle.fake_quant(qa, sa)).astype(np.float64)
    ag = np.abs(gy).astype(np.float64)
    # outside the clip range the gradient is exactly 0 (the STE mask); inside, an fp32 sum may
    # still cancel to 0 -- that is covered by the error bound, not by the zero pattern
    out_a = ~(np.abs(x) <= clip_a) if masked else np.zeros((M, K), bool)
    out_w = ~(np.abs(W) <= clip_w) if masked else np.zeros((N, K), bool)
    for got, r, n, absprod, out in ((gx, ref[0], N, ag @ wf, out_a), (gw, ref[1], M, ag.T @ xf, out_w),
                                    (gb, ref[2], M, ag.sum(0), np.zeros(N, bool))):
        got = got.cpu().numpy()
        assert np.isfinite(got).all()
        err = np.abs(got.astype(np.float64) - r.astype(np.float64))
        assert (err <= _bound(n, absprod, r)).all(), float(err.max())
        assert (got[out] == 0).all() and (r[out] == 0).all()


@pytest.fixture(scope="module")
def ax():
    from paper_2203_04071_b200 import _lib
    _lib.load()
    return _lib


@pytest.mark.parametrize("M,N,K", [(256, 1024, 1024), (37, 50, 70), (1, 1, 1), (300, 129, 257),
                                   (130, 1000, 2048), (2000, 1000, 1000)])
@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("split", [False, True], ids=["one-pass", "split-k"])
def test_ste_backward(ax, M, N, K, masked, split):
    """split: a workspace -- the pre-converted operands, split-K in clusters (and, at
    (2000, 1000, 1000), 256-column tiles); else the in-kernel conversion."""
    _check(ax, M, N, K, M + N, masked, split)


def test_ste_backward_empty(ax):
    """M = 0: gw and gb are empty sums (zero)."""
    gy = torch.zeros(0, 8, device=DEV)
    qa = torch.zeros(0, 5, dtype=torch.int8, device=DEV)
    qw = torch.ones(8, 5, dtype=torch.int8, device=DEV)
    s = torch.ones(1, device=DEV)
    gw = torch.full((8, 5), 7.0, device=DEV)
    gb = torch.full((8,), 7.0, device=DEV)
    ax.axq_ste_linear_backward(gy, qa, s, qw, s, gw=gw, gb=gb)
    torch.cuda.synchronize()
    assert (gw == 0).all() and (gb == 0).all()


def test_ste_backward_invalid(ax):
    gy = torch.zeros(4, 8, device=DEV)
    qw = torch.ones(8, 5, dtype=torch.int8, device=DEV)
    gx = torch.empty(4, 5, device=DEV)
    with pytest.raises(ax.AxqError):   # gx requested without the weight scale
        ax.axq_ste_linear_backward(gy, torch.zeros(4, 5, dtype=torch.int8, device=DEV), None, qw,
                                   None, gx=gx)


CONV_SHAPES = [(2, 8, 9, 9, 16, 3, 3, 1, 1), (1, 16, 11, 10, 24, 3, 3, 2, 1), (3, 32, 6, 7, 20, 1, 1, 1, 0),
               (2, 64, 14, 14, 64, 3, 3, 1, 1), (1, 3, 20, 18, 8, 7, 7, 2, 3)]


@pytest.mark.parametrize("shape", CONV_SHAPES)
@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("prep", [False, True], ids=["in-kernel", "prep"])
def test_ste_conv_backward(ax, shape, masked, prep):
    """prep: a workspace large enough for the pre-converted operands (ste_pp_kernel), else the
    in-kernel conversion (ste_tc_kernel)."""
    N, C, H, W, K, R, S, st, pd = shape
    x = datagen.normal(90 + C, 1, (N, H, W, C))
    wt = datagen.normal(90 + C, 2, (K, R, S, C), 0.2)
    qx, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(wt, 8)
    Ho, Wo = (H + 2 * pd - R) // st + 1, (W + 2 * pd - S) // st + 1
    gy = datagen.normal(90 + C, 3, (N, Ho, Wo, K))
    clip_a = np.float32(np.quantile(np.abs(x), 0.8)) if masked else None
    clip_w = np.float32(np.quantile(np.abs(wt), 0.8)) if masked else None
    mk = dict(x=x, clip_a=clip_a, w=wt, clip_w=clip_w) if masked else {}
    ref = oracle.ste_conv2d_backward(gy, qx, sa, qw, sw, (st, st), (pd, pd), **mk)
    # sum of |terms| per output: the same products over absolute values
    absref = oracle.ste_conv2d_backward(np.abs(gy), np.abs(qx.astype(np.int64)).astype(np.int8), sa,
                                        np.abs(qw.astype(np.int64)).astype(np.int8), sw, (st, st), (pd, pd))
    f = lambda v: _t(np.array([v], dtype=np.float32))
    d = ax.conv_desc(N, H, W, C, K, R, S, (st, st), (pd, pd))
    gx = torch.full((N, H, W, C), np.nan, device=DEV)
    gw = torch.full((K, R, S, C), np.nan, device=DEV)
    gb = torch.full((K,), np.nan, device=DEV)
    kw = dict(x=_t(x), d_clip_a=f(clip_a), w=_t(wt), d_clip_w=f(clip_w)) if masked else {}
    ws = torch.full((16 << 20,), np.nan, device=DEV) if prep else None
    ax.axq_ste_conv2d_backward(d, _t(gy), _t(qx), f(sa), _t(qw), f(sw), gx=gx, gw=gw, gb=gb, workspace=ws, **kw)
    torch.cuda.synchronize()
    M = N * Ho * Wo
    for got, r, a_, n in ((gx, ref[0], absref[0], K * R * S), (gw, ref[1], absref[1], M), (gb, ref[2], absref[2], M)):
        got = got.cpu().numpy()
        assert np.isfinite(got).all()
        err = np.abs(got.astype(np.float64) - r.astype(np.float64))
        assert (err <= _bound(n, a_.astype(np.float64), r)).all(), float(err.max())


@pytest.mark.parametrize("M,N,K", [(96, 40, 70), (300, 129, 257), (520, 1000, 1500)])
@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("prep", [False, True], ids=["in-kernel", "prep"])
def test_ste_backward_per_channel(ax, M, N, K, masked, prep):
    """Per-output-channel weight scales and clips (axq_ste_linear_backward_pc), with the
    in-kernel conversion and with the pre-converted operands (workspace given)."""
    x = datagen.normal(65, M, (M, K))
    W = datagen.normal(65, N, (N, K), 0.05) * np.linspace(0.3, 2.5, N, dtype=np.float32)[:, None]
    qa, sa = oracle.quantize_tensor(x, 8)
    amax_ch = np.abs(W).max(axis=1).astype(np.float32)
    sw = (amax_ch / np.float32(127)).astype(np.float32)
    qw = np.clip(np.rint(W / sw[:, None]), -127, 127).astype(np.int8)
    gy = datagen.normal(65, 3, (M, N))
    clip_a = np.float32(np.quantile(np.abs(x), 0.8))
    clip_w = (amax_ch * np.float32(0.7)).astype(np.float32)
    if masked:
        ref = oracle.ste_linear_backward(gy, qa, sa, qw, sw, x, clip_a, W, clip_w)
    else:
        ref = oracle.ste_linear_backward(gy, qa, sa, qw, sw)
    gx = torch.full((M, K), np.nan, device=DEV)
    gw = torch.full((N, K), np.nan, device=DEV)
    f = lambda v: _t(np.atleast_1d(np.asarray(v, dtype=np.float32)))
    kw = dict(x=_t(x), d_clip_a=f(clip_a), w=_t(W), d_clip_w=f(clip_w)) if masked else {}
    ws = torch.full((16 << 20,), np.nan, device=DEV) if prep else None
    ax.axq_ste_linear_backward(_t(gy), _t(qa), f(sa), _t(qw), f(sw), gx=gx, gw=gw, workspace=ws, **kw)
    torch.cuda.synchronize()
    wf = np.abs(oracle.fake_quant(qw, sw)).astype(np.float64)
    xf = np.abs(oracle.fake_quant(qa, sa)).astype(np.float64)
    ag = np.abs(gy).astype(np.float64)
    out_a = ~(np.abs(x) <= clip_a)
    out_w = ~(np.abs(W) <= clip_w[:, None])
    for got, r, n, absprod, out in ((gx, ref[0], N, ag @ wf, out_a), (gw, ref[1], M, ag.T @ xf, out_w)):
        got = got.cpu().numpy()
        err = np.abs(got.astype(np.float64) - r.astype(np.float64))
        assert (err <= _bound(n, absprod, r)).all(), float(err.max())
        if masked:   # the STE mask zeroes exactly; cancellation inside the range is bounded above
            assert (got[out] == 0).all() and (r[out] == 0).all()


def test_ste_backward_large_m_workspace(ax):
    """M >= 4096 with a workspace: the two-pass deterministic column sums and the split-K
    products (the benchmarked paths)."""
    _check(ax, 5000, 96, 80, 77, True, True)


@pytest.mark.parametrize("masked", [False, True])
def test_ste_conv_backward_workspace_large_m(ax, masked):
    """A conv with N*Ho*Wo = 6272 positions and a workspace: gw split over up to 128 slices."""
    N, C, H, W, K, R, S, st, pd = 8, 32, 28, 28, 32, 3, 3, 1, 1
    x = datagen.normal(95, 1, (N, H, W, C))
    wt = datagen.normal(95, 2, (K, R, S, C), 0.2)
    qx, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(wt, 8)
    gy = datagen.normal(95, 3, (N, H, W, K))
    clip_a = np.float32(np.quantile(np.abs(x), 0.8)) if masked else None
    clip_w = np.float32(np.quantile(np.abs(wt), 0.8)) if masked else None
    mk = dict(x=x, clip_a=clip_a, w=wt, clip_w=clip_w) if masked else {}
    ref = oracle.ste_conv2d_backward(gy, qx, sa, qw, sw, (st, st), (pd, pd), **mk)
    absref = oracle.ste_conv2d_backward(np.abs(gy), np.abs(qx.astype(np.int64)).astype(np.int8), sa,
                                        np.abs(qw.astype(np.int64)).astype(np.int8), sw, (st, st), (pd, pd))
    f = lambda v: _t(np.array([v], dtype=np.float32))
    d = ax.conv_desc(N, H, W, C, K, R, S, (st, st), (pd, pd))
    gx = torch.full((N, H, W, C), np.nan, device=DEV)
    gw = torch.full((K, R, S, C), np.nan, device=DEV)
    gb = torch.full((K,), np.nan, device=DEV)
    ws = torch.full((64 * 1024 * 1024 // 4,), np.nan, device=DEV)
    kw = dict(x=_t(x), d_clip_a=f(clip_a), w=_t(wt), d_clip_w=f(clip_w)) if masked else {}
    ax.axq_ste_conv2d_backward(d, _t(gy), _t(qx), f(sa), _t(qw), f(sw), gx=gx, gw=gw, gb=gb, workspace=ws, **kw)
    torch.cuda.synchronize()
    M = N * H * W
    for got, r, a_, n in ((gx, ref[0], absref[0], K * R * S), (gw, ref[1], absref[1], M), (gb, ref[2], absref[2], M)):
        got = got.cpu().numpy()
        assert np.isfinite(got).all()
        err = np.abs(got.astype(np.float64) - r.astype(np.float64))
        assert (err <= _bound(n, a_.astype(np.float64), r)).all(), float(err.max())


@pytest.mark.parametrize("elems", [1, 70000, 190000, 400000])
def test_ste_backward_workspace_sizes(ax, elems):
    """Workspaces too small for the pre-converted operands fall back to the in-kernel
    conversion; in between, the pre-converted path runs with fewer (or no) split-K slices."""
    M, N, K = 200, 300, 260
    x = datagen.normal(67, 1, (M, K))
    W = datagen.normal(67, 2, (N, K), 0.05)
    qa, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(W, 8)
    gy = datagen.normal(67, 3, (M, N))
    ref = oracle.ste_linear_backward(gy, qa, sa, qw, sw)
    gx = torch.full((M, K), np.nan, device=DEV)
    gw = torch.full((N, K), np.nan, device=DEV)
    f = lambda v: _t(np.array([v], dtype=np.float32))
    ws = torch.full((elems,), np.nan, device=DEV)
    ax.axq_ste_linear_backward(_t(gy), _t(qa), f(sa), _t(qw), f(sw), gx=gx, gw=gw, workspace=ws)
    torch.cuda.synchronize()
    wf = np.abs(oracle.fake_quant(qw, sw)).astype(np.float64)
    xf = np.abs(oracle.fake_quant(qa, sa)).astype(np.float64)
    ag = np.abs(gy).astype(np.float64)
    for got, r, n, absprod in ((gx, ref[0], N, ag @ wf), (gw, ref[1], M, ag.T @ xf)):
        got = got.cpu().numpy()
        err = np.abs(got.astype(np.float64) - r.astype(np.float64))
        assert (err <= _bound(n, absprod, r)).all(), float(err.max())


def test_ste_binding_checks_and_strided_grad(ax):
    """The binding makes a strided / expanded gradient contiguous (autograd's stride-0 gy after
    y.sum()) and rejects mismatched shapes instead of letting the kernel write out of bounds."""
    M, N, K = 40, 24, 16
    x = datagen.normal(66, 1, (M, K))
    W = datagen.normal(66, 2, (N, K), 0.05)
    qa, sa = oracle.quantize_tensor(x, 8)
    qw, sw = oracle.quantize_tensor(W, 8)
    gy = torch.ones(1, 1, device=DEV).expand(M, N)              # stride 0
    ref = oracle.ste_linear_backward(np.ones((M, N), np.float32), qa, sa, qw, sw)
    gx = torch.empty(M, K, device=DEV)
    f = lambda v: _t(np.array([v], dtype=np.float32))
    ax.axq_ste_linear_backward(gy, _t(qa), f(sa), _t(qw), f(sw), gx=gx)
    torch.cuda.synchronize()
    np.testing.assert_allclose(gx.cpu().numpy(), ref[0], rtol=1e-5, atol=1e-6)
    with pytest.raises(ValueError):
        ax.axq_ste_linear_backward(gy, _t(qa), f(sa), _t(qw[:, :8]), f(sw), gx=gx)
    with pytest.raises(ValueError):
        ax.axq_ste_linear_backward(gy, _t(qa), f(sa), _t(qw), f(sw), gx=torch.empty(M, K + 1, device=DEV))
