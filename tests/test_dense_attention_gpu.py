"""Flash-style dense attention kernels (csrc/dense.cu) against the oracle's
dense_attention / dense_attention_backward (oracle/orc_graph_attn.c, pinned to
the compiled reference) and, for the Trainer's dense epochs with pad rows
(s_real < S, proj/src/model.cpp:395-405), against the oracle's sparse
attention over the explicit dense execution pattern.

Tolerances as tests/test_sparse_attention_gpu.py: f64 1e-12 (max-normalised),
f32 1e-5 (max-normalised and L2), bf16 2e-2 / 1e-2."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import CSR

from paper_2407_14106_b200 import attention as A
from paper_2407_14106_b200._lib import ConfigError, DataError

pytestmark = pytest.mark.gpu

TOL = {"f64": (1e-12, 1e-12), "f32": (1e-5, 1e-5), "bf16": (2e-2, 1e-2)}


def close(got, want, dtype, what):
    e = rel_err(got, want)
    assert e[0] <= TOL[dtype][0] and e[1] <= TOL[dtype][1], f"{what} [{dtype}] {e}"


@pytest.mark.parametrize("S,dk,dv", [(1, 4, 4), (7, 3, 5), (33, 8, 8), (100, 16, 12), (257, 24, 24), (64, 64, 64)])
def test_dense_f64_vs_oracle(cuda, orc, S, dk, dv):
    rng = np.random.default_rng(S * 100 + dk)
    q, k = rng.standard_normal((S, dk)), rng.standard_normal((S, dk))
    v, up = rng.standard_normal((S, dv)), rng.standard_normal((S, dv))
    bias = rng.normal(0, 0.3, (S, S))
    wm = (rng.random((S, S)) < 0.8) / 0.8
    for b, w in ((None, None), (bias, None), (bias, wm)):
        got = A.dense_attention(q, k, v, b, w)
        close(got.output, orc.dense_fwd(q, k, v, b, w), "f64", "out")
        assert got.macs.score_macs == S * S * dk and got.macs.weight_macs == S * S * dv
        g = A.dense_attention_backward(q, k, v, b, w, up)
        wq, wk, wv, wb = orc.dense_bwd(q, k, v, b, w, up)
        for x, y, nm in ((g.dq, wq, "dq"), (g.dk, wk, "dk"), (g.dv, wv, "dv"), (g.dbias, wb.reshape(-1), "dbias")):
            close(x, y, "f64", nm)


def test_dense_known_answers(cuda):
    # proj/tests/test_attention.cpp:23-40: S=1 -> O = V exactly; zero Q -> mean of V
    v = np.array([[1.5, -2.0, 3.0]])
    assert np.array_equal(A.dense_attention(np.ones((1, 3)), np.ones((1, 3)), v).output, v)
    v2 = np.array([[1.0, 2.0], [3.0, 6.0]])
    out = A.dense_attention(np.zeros((2, 2)), np.ones((2, 2)), v2).output
    assert np.allclose(out, [[2.0, 4.0], [2.0, 4.0]], atol=1e-15)
    with pytest.raises(DataError, match="non-finite K"):
        A.dense_attention(np.ones((2, 2)), np.array([[1.0, np.nan], [0, 0]]), v2)
    with pytest.raises(ConfigError, match="bias shape"):
        A.dense_attention(np.ones((2, 2)), np.ones((2, 2)), v2, np.zeros((2, 3)))


def test_complete_graph_sparse_equals_dense(cuda):
    # proj/tests/test_attention.cpp:75-87 with the flash kernel on the dense side
    rng = np.random.default_rng(5)
    s = 19
    q, k, v = (rng.standard_normal((s, 6)) for _ in range(3))
    ro = np.arange(s + 1, dtype=np.int64) * s
    co = np.tile(np.arange(s, dtype=np.int64), s)
    sp = A.edge_sparse_attention(q, k, v, A.Graph(s, ro, co)).output
    assert np.abs(sp - A.dense_attention(q, k, v).output).max() <= 1e-12


def _dev(x, dtype):
    import torch

    td = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    return torch.tensor(x, dtype=td, device="cuda")


def _exec_pattern(S, s_real):
    """dense_pattern_exec (model.cpp:395-405): real rows -> [0, s_real), pad rows -> self."""
    ro, co = [0], []
    for r in range(S):
        co.extend(range(s_real) if r < s_real else [r])
        ro.append(len(co))
    return CSR(S, np.array(ro, dtype=np.int64), np.array(co, dtype=np.int64))


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
@pytest.mark.parametrize("S,s_real,H,dh", [(300, 300, 8, 8), (300, 257, 8, 8), (130, 100, 4, 16)])
def test_multihead_and_pad_rows_vs_oracle(cuda, orc, dtype, S, s_real, H, dh):
    import torch

    rng = np.random.default_rng(S + s_real + H)
    q, k, v, up = (rng.standard_normal((S, H * dh)) for _ in range(4))
    acc = "f64" if dtype == "f64" else "f32"
    bias = rng.normal(0, 0.3, (S, S))
    wm = (rng.random((H, S, S)) < 0.8) / 0.8
    tq, tk, tv, tu = (_dev(x, dtype) for x in (q, k, v, up))
    tb, tw = _dev(bias, acc), _dev(wm, acc)
    att = A.DeviceDenseAttention(S, H, dh, dh, dtype, s_real=s_real)
    out, lse = att.forward(tq, tk, tv, tb, tw)
    dq, dk, dv, db = att.backward(tq, tk, tv, out, lse, tu, tb, tw, want_dbias=True)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    qn, kn, vn, un = f(tq), f(tk), f(tv), f(tu)
    g = _exec_pattern(S, s_real)
    rows = np.repeat(np.arange(S), np.diff(g.row_off))
    b_e = bias[rows, g.cols]
    want = {n: np.zeros((S, H * dh)) for n in ("out", "dq", "dk", "dv")}
    dbias = np.zeros(g.nnz)
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        w_e = wm[h][rows, g.cols]
        want["out"][:, sl] = orc.sparse_fwd(qn[:, sl], kn[:, sl], vn[:, sl], g, b_e, w_e)
        a, b, c, e = orc.sparse_bwd(qn[:, sl], kn[:, sl], vn[:, sl], g, b_e, w_e, un[:, sl])
        want["dq"][:, sl], want["dk"][:, sl], want["dv"][:, sl] = a, b, c
        dbias += e
    for nm, got in (("out", out), ("dq", dq), ("dk", dk), ("dv", dv)):
        close(f(got), want[nm], dtype, nm)
    db_dense = np.zeros((S, S))
    db_dense[rows, g.cols] = dbias
    db_dense[np.arange(s_real, S), np.arange(s_real, S)] = 0  # pad rows: no score gradient
    close(f(db)[:s_real], db_dense[:s_real], dtype, "dbias")
    # pad rows: out = m * v exactly
    pad = np.arange(s_real, S)
    if pad.size and dtype != "bf16":
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            assert np.array_equal(f(out)[pad, sl], (wm[h][pad, pad][:, None] * vn[pad, sl]).astype(
                np.float32 if dtype == "f32" else np.float64))


@pytest.mark.parametrize("S,s_real,H,dh,with_bias", [(300, 300, 8, 8, False), (300, 257, 8, 8, True),
                                                     (200, 200, 4, 16, True), (130, 130, 2, 24, False)])
def test_tcgen05_backward_vs_oracle(cuda, orc, S, s_real, H, dh, with_bias):
    """bf16 dense backward without weight_mult / dbias runs on tcgen05
    (dense_tc.cu: dq and dkdv kernels): gradients vs the oracle over the
    explicit dense execution pattern, bf16 tolerance."""
    import torch

    rng = np.random.default_rng(S + H + dh)
    q, k, v, up = (rng.standard_normal((S, H * dh)) for _ in range(4))
    bias = rng.normal(0, 0.3, (S, S)) if with_bias else None
    tq, tk, tv, tu = (_dev(x, "bf16") for x in (q, k, v, up))
    tb = _dev(bias, "f32") if with_bias else None
    att = A.DeviceDenseAttention(S, H, dh, dh, "bf16", s_real=s_real)
    out, lse = att.forward(tq, tk, tv, tb)
    dq, dk, dv, _ = att.backward(tq, tk, tv, out, lse, tu, tb)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    qn, kn, vn, un = f(tq), f(tk), f(tv), f(tu)
    g = _exec_pattern(S, s_real)
    rows = np.repeat(np.arange(S), np.diff(g.row_off))
    b_e = bias[rows, g.cols] if with_bias else None
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        a_, b_, c_, _ = orc.sparse_bwd(qn[:, sl], kn[:, sl], vn[:, sl], g, b_e, None, un[:, sl])
        close(f(dq)[:, sl], a_, "bf16", f"dq h{h}")
        close(f(dk)[:, sl], b_, "bf16", f"dk h{h}")
        close(f(dv)[:, sl], c_, "bf16", f"dv h{h}")


@pytest.mark.parametrize("S,s_real,H,dh", [(2048, 2048, 2, 8), (1536, 1500, 3, 16)])
def test_tcgen05_many_blocks_vs_torch_fp32(cuda, S, s_real, H, dh):
    """The tcgen05 kernels' mask-free full-block path (every 128-key block but
    the last, all rows / keys of a CTA real, no bias) over many blocks, forward
    and backward, against a torch fp32 restatement of the dense layer on the
    same bf16 inputs (real rows attend the real columns; pad rows only
    themselves). bf16 tolerance: max-normalised 2e-2, L2 1e-2."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(S + H)
    q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    att = A.DeviceDenseAttention(S, H, dh, dh, "bf16", s_real=s_real)
    out, lse = att.forward(q, k, v)
    dq, dk, dv, _ = att.backward(q, k, v, out, lse, up)
    torch.cuda.synchronize()
    qf, kf, vf = (t.float().view(S, H, dh).transpose(0, 1).requires_grad_() for t in (q, k, v))
    mask = torch.full((S, S), float("-inf"), device="cuda")
    mask[:s_real, :s_real] = 0.0
    idx = torch.arange(s_real, S, device="cuda")
    mask[idx, idx] = 0.0
    att_w = torch.softmax(qf @ kf.transpose(1, 2) / dh ** 0.5 + mask, dim=-1)
    ref = (att_w @ vf).transpose(0, 1).reshape(S, H * dh)
    ref.backward(up.float())
    f = lambda t: t.detach().double().cpu().numpy()  # noqa: E731
    rg = lambda t: f(t.grad.transpose(0, 1).reshape(S, H * dh))  # noqa: E731
    close(f(out), f(ref), "bf16", "out")
    close(f(dq)[:s_real], rg(qf)[:s_real], "bf16", "dq")
    close(f(dk)[:s_real], rg(kf)[:s_real], "bf16", "dk")
    close(f(dv), rg(vf), "bf16", "dv")


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_strided_fused_qkv_matches_contiguous(cuda, dtype):
    """q, k, v as column slices of one fused [S, 3 d] tensor (row stride 3 d):
    the C ABI takes one row stride per tensor family, so the outputs must be
    allocated with the inputs' strides — results equal the contiguous call's
    bit for bit. Mismatched dtypes / strides raise ConfigError."""
    import torch

    S, H, dh = 300, 2, 8
    d = H * dh
    t = {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]
    g = torch.Generator(device="cuda").manual_seed(7)
    qkv = torch.randn((S, 3 * d), generator=g, device="cuda").to(t)
    up = torch.randn((S, d), generator=g, device="cuda").to(t)
    q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
    att = A.DeviceDenseAttention(S, H, dh, dh, dtype)
    o1, l1 = att.forward(q, k, v)
    qc, kc, vc = q.contiguous(), k.contiguous(), v.contiguous()
    o2, l2 = att.forward(qc, kc, vc)
    torch.cuda.synchronize()
    assert o1.stride() == v.stride()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    # backward: dO and O with V's row stride, as the ABI requires
    do = torch.empty_strided(v.shape, v.stride(), dtype=t, device="cuda").copy_(up)
    dq1, dk1, dv1, _ = att.backward(q, k, v, o1, l1, do)
    dq2, dk2, dv2, _ = att.backward(qc, kc, vc, o2, l2, up)
    torch.cuda.synchronize()
    assert dq1.stride() == q.stride() and dv1.stride() == v.stride()
    for a_, b_ in ((dq1, dq2), (dk1, dk2), (dv1, dv2)):
        assert torch.equal(a_, b_)
    with pytest.raises(ConfigError):
        att.forward(q.float() if dtype == "bf16" else q.double(), k, v)
    with pytest.raises(ConfigError):
        att.backward(q, k, v, o1, l1, up)  # dO contiguous, O strided: two row strides


@pytest.mark.parametrize("boost_at", [384, 1000])
def test_tcgen05_forward_running_max_overrun(cuda, boost_at):
    """The forward's one-pass blocks score against the running max and redo a
    block exactly when a score outruns it by more than 8 (log2 units). Keys
    from `boost_at` on are scaled x 24, so later blocks overrun the max of the
    earlier ones by far more than 8: the redo path must give the same softmax
    as a torch fp32 restatement (bf16 tolerance 2e-2 / 1e-2)."""
    import torch

    S, H, dh = 1280, 2, 8
    g = torch.Generator(device="cuda").manual_seed(boost_at)
    q, k, v = (torch.randn((S, H * dh), generator=g, device="cuda") for _ in range(3))
    k[boost_at:] *= 24.0
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    att = A.DeviceDenseAttention(S, H, dh, dh, "bf16")
    out, lse = att.forward(q, k, v)
    torch.cuda.synchronize()
    qf, kf, vf = (t.float().view(S, H, dh).transpose(0, 1) for t in (q, k, v))
    logits = qf @ kf.transpose(1, 2) / dh ** 0.5
    ref = (torch.softmax(logits, dim=-1) @ vf).transpose(0, 1).reshape(S, H * dh)
    ref_lse = (torch.logsumexp(logits, dim=-1) / np.log(2.0)).transpose(0, 1)  # log2 units
    f = lambda t: t.detach().double().cpu().numpy()  # noqa: E731
    close(f(out), f(ref), "bf16", "out")
    assert np.abs(f(lse) - f(ref_lse)).max() <= 2e-2 * max(1.0, np.abs(f(ref_lse)).max())
