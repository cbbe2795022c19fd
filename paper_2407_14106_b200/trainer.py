"""The Trainer's integration of the attention path on the device (SURVEY §8
f3; reference Trainer::build_plans / layout_for / train_epoch,
proj/src/model.cpp:339-468, 806-883) for one node-classification sequence:

  * build_plans: self loops, beta_G, interleave conditions, select_k, the
    cluster reorder, k x k grid and permuted graph (all through
    libgte_b200: GPU graph kernels + the exact reorder);
  * per epoch: the interleave mode (select_mode), the ECR threshold from the
    tuner (auto_tune) or 5 beta_G, the active pattern from a beta_thre-keyed
    layout cache (a new threshold builds a layout once: build_layout on the
    GPU, a device plan with its community schedule, SPD buckets of every
    attended pair on the GPU — no 20,000-node SPD guard), the bias gathered
    from the bucket table, L GPH blocks forward + backward on the device
    (csrc/gph_layer.cu), the bucket table's gradient reduced in fixed order,
    an SGD step, the tuner update with the epoch loss, and a metrics row.

Rows stay in execution (cluster-reordered) order for the whole epoch: every
row-wise operation commutes with the permutation, so the attention runs on
the layout's pattern with no per-layer gather/scatter (the reference
permutes rows inside each distributed layer, parallel.cpp:48-79).

The input encoder, final LayerNorm, classifier, cross-entropy and the SGD
update are small row-wise / GEMM operations outside the hot path; they run as
torch ops on the same device tensors (plumbing), like the reference's
model-side code is out of SURVEY §2's scope. Dropout is off.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import control, glue
from . import partition as P
from .attention import DevicePlan, Graph
from .layer import NAMES as LAYER_PARAMS
from .layer import WEIGHTS as LAYER_WEIGHTS
from .layer import GphLayer, param_shapes


@dataclass
class EpochStats:
    epoch: int
    mode: str
    reason: int
    beta_thre: float
    loss: float
    avg_loss: float
    epoch_time_s: float
    pattern_nnz: int
    dropped_edges: int
    layout_cached: bool

    CSV = "epoch,mode,reason,beta_thre,loss,avg_loss,epoch_time_s,pattern_nnz,dropped_edges,layout_cached"

    def csv(self) -> str:
        return (f"{self.epoch},{self.mode},{self.reason},{self.beta_thre:.10g},{self.loss:.10g},{self.avg_loss:.10g},"
                f"{self.epoch_time_s:.6f},{self.pattern_nnz},{self.dropped_edges},{int(self.layout_cached)}")


class _Active:
    def __init__(self, plan, buckets, dropped, layers):
        self.plan, self.buckets, self.dropped, self.layers = plan, buckets, dropped, layers


class DeviceTrainer:
    def __init__(self, row_offsets, cols, features, labels, *, layers: int = 2, heads: int = 8, hidden: int = 64,
                 ffn: int = 128, classes: int | None = None, cluster_k: int = 8, block_dim: int = 16,
                 spd_cap: int = 8, dense_period: int = 4, strategy: str = "elastic", auto_tune: bool = True,
                 delta: int = 1, lr: float = 0.05, seed: int = 0, dense_limit: int = 16384):
        import torch

        self.dev = torch.device("cuda", 0)
        ro, co = np.asarray(row_offsets, np.int64), np.asarray(cols, np.int64)
        self.n = n = ro.shape[0] - 1
        self.g = Graph(n, ro, co)
        self.L, self.H, self.d, self.ffn = layers, heads, hidden, ffn
        self.block_dim, self.spd_cap, self.dense_period = block_dim, spd_cap, dense_period
        self.strategy, self.auto_tune, self.lr, self.dense_limit = strategy, auto_tune, lr, dense_limit
        # ---- build_plans (model.cpp:339-392), node task: attention graph = graph + self loops
        self.attn = P.add_self_loops(self.g)
        self.beta_g = P.density(self.attn)
        self.flags, _ = control.check_conditions(self.attn.row_offsets, self.attn.col_indices, layers)
        k = cluster_k if cluster_k > 0 else control.select_k(50 * 2 ** 20, hidden, 1)
        self.perm = P.reorder(self.attn, k, seed)
        self.grid = P.build_cluster_grid(self.attn, self.perm, k)
        self.g_exec = P.permute_graph(self.attn, self.perm)
        self.inv = np.asarray(self.perm.inverse, np.int64)
        self.tuner = control.Tuner(self.beta_g, delta)
        self.cache: dict = {}
        self.epoch = 0
        self.history: list[EpochStats] = []
        # ---- parameters (f32), rows in execution order
        rng = np.random.default_rng(seed + 17)
        X = np.asarray(features, np.float32)[self.inv]
        y = np.asarray(labels, np.int64)[self.inv]
        self.classes = classes or int(y.max()) + 1
        t = lambda a: torch.tensor(a, dtype=torch.float32, device=self.dev)  # noqa: E731
        self.X, self.y = t(X), torch.tensor(y, device=self.dev)
        f_in = X.shape[1]
        self.w_in = t(rng.normal(0, 1 / np.sqrt(f_in), (f_in, hidden)))
        self.b_in = t(np.zeros(hidden))
        self.layer_params = []
        for _ in range(layers):
            p = {}
            for name, shape in param_shapes(hidden, ffn).items():
                fan = shape[0] if len(shape) == 2 else 1
                p[name] = t(rng.normal(0, 1 / np.sqrt(fan), shape) if name in LAYER_WEIGHTS else np.zeros(shape))
            p["ln1_scale"].fill_(1.0)
            p["ln2_scale"].fill_(1.0)
            self.layer_params.append(p)
        self.lnf_scale, self.lnf_shift = t(np.ones(hidden)), t(np.zeros(hidden))
        self.w_cls = t(rng.normal(0, 1 / np.sqrt(hidden), (hidden, self.classes)))
        self.b_cls = t(np.zeros(self.classes))
        self.spd_bias = t(rng.normal(0, 0.1, spd_cap + 2))

    # ------------------------------------------------------------ patterns
    def _pattern(self, kind: str, theta: float):
        if kind == "dense":  # dense_pattern_exec (model.cpp:395-405), node task: s_pad = s_real
            if self.n > self.dense_limit:
                raise ValueError(f"dense epoch over {self.n} rows exceeds dense_limit {self.dense_limit}")
            ro = np.arange(self.n + 1, dtype=np.int64) * self.n
            co = np.tile(np.arange(self.n, dtype=np.int64), self.n)
            return ro, co, 0
        if kind == "edge":
            return np.asarray(self.g_exec.row_offsets), np.asarray(self.g_exec.col_indices), 0
        lay = P.build_layout(self.grid, self.g_exec, P.ELASTIC, theta, self.beta_g, self.block_dim)
        return np.asarray(lay.pattern.row_offsets), np.asarray(lay.pattern.cols), int(lay.dropped_edges)

    def _active(self, kind: str, theta: float):
        key = (kind,) if kind != "cluster" else (kind, float(theta))
        if key in self.cache:
            return self.cache[key], True
        ro, co, dropped = self._pattern(kind, theta)
        plan = DevicePlan.from_host(ro, co)
        plan.schedule()
        buckets = glue.pattern_buckets_graph(ro, co, self.inv, -1, self.g.row_offsets, self.g.col_indices,
                                             self.spd_cap)
        layers = [GphLayer(plan, "f32", self.H, self.d, self.ffn, p) for p in self.layer_params]
        a = _Active(plan, buckets, dropped, layers)
        self.cache[key] = a
        return a, False

    # ------------------------------------------------------------ one epoch
    def train_epoch(self, force: str | None = None) -> EpochStats:
        """force: None (the reference policy), "dense", "cluster" or "edge"
        (Trainer::forward_backward's ForcedPattern, model.cpp:922-932)."""
        import torch
        import torch.nn.functional as F

        self.epoch += 1
        t0 = time.perf_counter()
        mode, reason = control.select_mode(self.flags, self.epoch, self.dense_period)
        if self.strategy == "indolent":
            theta = self.beta_g
        elif self.auto_tune:
            theta = self.tuner.beta_thre()
        else:
            theta = min(5.0 * self.beta_g, 1.0)
        kind = force or ("dense" if mode == 1 else ("edge" if self.strategy == "none" else "cluster"))
        act, cached = self._active(kind, theta)
        # forward
        w_in, b_in = self.w_in.requires_grad_(), self.b_in.requires_grad_()
        h0 = self.X @ w_in + b_in
        h = h0.detach().clone()
        bias_vals = glue.bias_from_table(act.buckets, self.spd_bias)
        for layer in act.layers:
            layer.forward(h, bias_vals)
        hf = h.clone().requires_grad_()
        lnf_s, lnf_b = self.lnf_scale.requires_grad_(), self.lnf_shift.requires_grad_()
        w_cls, b_cls = self.w_cls.requires_grad_(), self.b_cls.requires_grad_()
        logits = F.layer_norm(hf, (self.d,), lnf_s, lnf_b, eps=1e-6) @ w_cls + b_cls
        loss = F.cross_entropy(logits, self.y)
        loss.backward()
        # backward through the blocks on the device
        dh = hf.grad.detach().clone()
        dtable = torch.zeros_like(self.spd_bias)
        grads = []
        for layer, p in zip(reversed(act.layers), reversed(self.layer_params)):
            gr = {nm: torch.zeros_like(p[nm]) for nm in LAYER_PARAMS}
            db = layer.backward(dh, bias_vals, gr)
            dtable += glue.dbias_to_table(act.buckets, db, self.spd_bias.numel())
            grads.append((p, gr))
        h0.backward(dh)
        # SGD (model.cpp:sgd_step)
        with torch.no_grad():
            for t in (self.w_in, self.b_in, self.lnf_scale, self.lnf_shift, self.w_cls, self.b_cls):
                t -= self.lr * t.grad
                t.grad = None
            for p, gr in grads:
                for nm in LAYER_PARAMS:
                    p[nm] -= self.lr * gr[nm]
            self.spd_bias -= self.lr * dtable
        lv = float(loss.item())
        if not np.isfinite(lv):
            raise FloatingPointError(f"training diverged at epoch {self.epoch} (non-finite loss)")
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        self.tuner.update(lv, 1.0, self.epoch - 1)  # fixed 1 s epoch time unless tuner_clock=wall (model.cpp:871)
        st = EpochStats(self.epoch, kind, reason, float(theta), lv, self.tuner.state()[0], dt, act.plan.nnz,
                        act.dropped, cached)
        self.history.append(st)
        return st
