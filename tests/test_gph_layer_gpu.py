"""The transformer block around the attention: gte_gph_layer
forward + backward against a float64 numpy restatement of the reference
Trainer's layer (proj/src/model.cpp:533-595 forward, :669-744 backward;
LayerNorm proj/src/matrix.cpp:91-139; GELU model.cpp:20-32), whose attention
is the C oracle's per-head sparse attention (pinned to the compiled
reference). f64: 1e-9; f32: 1e-4; bf16: 5e-2 (max-normalised)."""
import numpy as np
import pytest

from oracle import CSR

from paper_2407_14106_b200 import attention as A
from paper_2407_14106_b200 import layer as LY
from paper_2407_14106_b200.datagen import community_graph

pytestmark = pytest.mark.gpu
TOL = {"f64": 1e-9, "f32": 1e-4, "bf16": 5e-2}


def ln(x, sc, sh):
    mu = x.mean(1, keepdims=True)
    var = ((x - mu) ** 2).mean(1, keepdims=True)
    inv = 1.0 / np.sqrt(var + 1e-6)
    nh = (x - mu) * inv
    return nh * sc + sh, (nh, inv)


def ln_bwd(dout, cache, sc):
    nh, inv = cache
    dn = dout * sc
    m1 = dn.mean(1, keepdims=True)
    m2 = (dn * nh).mean(1, keepdims=True)
    return inv * (dn - m1 - nh * m2), (dout * nh).sum(0), dout.sum(0)


C0, A0 = 0.7978845608028654, 0.044715


def gelu(x):
    return 0.5 * x * (1 + np.tanh(C0 * (x + A0 * x ** 3)))


def gelu_g(x):
    t = np.tanh(C0 * (x + A0 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * C0 * (1 + 3 * A0 * x * x)


def reference_layer(orc, g, H, p, h, bias, dh_up):
    d = h.shape[1]
    dh_ = d // H
    a, c1 = ln(h, p["ln1_scale"], p["ln1_shift"])
    q, k, v = a @ p["w_q"] + p["b_q"], a @ p["w_k"] + p["b_k"], a @ p["w_v"] + p["b_v"]
    attn = np.zeros_like(h)
    for hh in range(H):
        sl = slice(hh * dh_, (hh + 1) * dh_)
        attn[:, sl] = orc.sparse_fwd(q[:, sl], k[:, sl], v[:, sl], g, bias)
    h1 = h + attn @ p["w_o"] + p["b_o"]
    b, c2 = ln(h1, p["ln2_scale"], p["ln2_shift"])
    u = b @ p["w_ff1"] + p["b_ff1"]
    gu = gelu(u)
    out = h1 + gu @ p["w_ff2"] + p["b_ff2"]
    # backward (model.cpp:682-744)
    G = {}
    dh = dh_up.copy()
    G["w_ff2"] = gu.T @ dh
    G["b_ff2"] = dh.sum(0)
    du = (dh @ p["w_ff2"].T) * gelu_g(u)
    G["w_ff1"] = b.T @ du
    G["b_ff1"] = du.sum(0)
    dx, G["ln2_scale"], G["ln2_shift"] = ln_bwd(du @ p["w_ff1"].T, c2, p["ln2_scale"])
    dh = dh + dx
    G["w_o"] = attn.T @ dh
    G["b_o"] = dh.sum(0)
    dattn = dh @ p["w_o"].T
    dq, dk, dv = np.zeros_like(h), np.zeros_like(h), np.zeros_like(h)
    dbias = np.zeros(g.nnz)
    for hh in range(H):
        sl = slice(hh * dh_, (hh + 1) * dh_)
        a_, b_, c_, e_ = orc.sparse_bwd(q[:, sl], k[:, sl], v[:, sl], g, bias, None, dattn[:, sl])
        dq[:, sl], dk[:, sl], dv[:, sl] = a_, b_, c_
        dbias += e_
    for n, x in (("q", dq), ("k", dk), ("v", dv)):
        G["w_" + n] = a.T @ x
        G["b_" + n] = x.sum(0)
    da = dq @ p["w_q"].T + dk @ p["w_k"].T + dv @ p["w_v"].T
    dx, G["ln1_scale"], G["ln1_shift"] = ln_bwd(da, c1, p["ln1_scale"])
    return out, dh + dx, G, dbias, np.abs(dk).sum(0).max()


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_gph_layer_matches_reference_math(cuda, orc, dtype):
    import torch

    n, H, d, ffn = 600, 8, 64, 128
    ro, co = community_graph(n, 10.0, community=64, seed=3)
    ro, co = np.asarray(ro, np.int64), np.asarray(co, np.int64)
    g = CSR(n, ro, co)
    rng = np.random.default_rng(4)
    shapes = LY.param_shapes(d, ffn)
    p = {k: rng.normal(0, 0.15, s) for k, s in shapes.items()}
    p["ln1_scale"] += 1.0
    p["ln2_scale"] += 1.0
    td = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    acc = torch.float64 if dtype == "f64" else torch.float32
    tp = {k: torch.tensor(v, dtype=td if k in LY.WEIGHTS else acc, device="cuda") for k, v in p.items()}
    # the reference math on exactly the values the device sees
    pr = {k: t.double().cpu().numpy() for k, t in tp.items()}
    h = torch.tensor(rng.standard_normal((n, d)), dtype=td, device="cuda")
    up = torch.tensor(rng.standard_normal((n, d)), dtype=td, device="cuda")
    bias = torch.tensor(rng.normal(0, 0.3, g.nnz), dtype=acc, device="cuda")
    want_out, want_dh, want_g, want_db, dk_l1 = reference_layer(orc, g, H, pr, h.double().cpu().numpy(),
                                                         bias.double().cpu().numpy(), up.double().cpu().numpy())
    plan = A.DevicePlan.from_host(ro, co)
    layer = LY.GphLayer(plan, dtype, H, d, ffn, tp)
    out = layer.forward(h.clone(), bias)
    grads = {k: torch.zeros(s, dtype=acc, device="cuda") for k, s in shapes.items()}
    dh = up.clone()
    db = layer.backward(dh, bias, grads)
    torch.cuda.synchronize()

    def close(got, want, what, floor=1e-3):
        got = got.double().cpu().numpy() if hasattr(got, "cpu") else got
        e = np.abs(got - want).max() / max(np.abs(want).max(), floor)
        assert e <= TOL[dtype], f"{what} [{dtype}] {e:.3g}"

    close(out, want_out, "h_out")
    close(dh, want_dh, "dh_in")
    close(db, want_db, "dbias")
    for k in shapes:
        # grad b_k is zero in exact arithmetic (sum_j dK_j = sum_i q_i sum_j
        # ds_ij = 0): both sides hold the rounding noise of a 600-row sum,
        # compared on the sum's own scale (sum_r |dK_r|)
        close(grads[k], want_g[k], "grad " + k, floor=dk_l1 if k == "b_k" else 1e-3)
