"""Visibility-MLP training.

The reference package ships no training code, so this follows the SPEC's
``nn.train``: the feature MLP (14 -> 32 -> 32 -> 6, per Gaussian) and the
visibility MLP (16 -> 32 -> 32 -> 1) are trained jointly on a
``VisibilityDataset`` (sampling.py) with a weighted binary cross-entropy on
the logits (pos_weight biases toward "visible": over-predicting is preferred,
PAPER §4.4), Adam, a cosine warm-up to lr_init over the first 20 % of the
iterations and an exponential decay to lr_final at the last one.  Every
iteration samples a batch of (view, Gaussian) pairs uniformly across views and
Gaussians and builds the 16 inputs exactly as the renderer does for the
training camera (identity instance, focal = the training focal, so
d_t = d_r): [mean / r, unit direction camera -> Gaussian, normalised
distance, camera forward, feature].  Torch autograd on the GPU (or CPU);
this is offline work, off the render path.  The trained weights feed stage (b)
through ``ComposedScene.add_asset(asset, model)``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .asset import Asset
from .asset import asset_hash
from .nn import Mlp, VisibilityModel, feature_inputs, make_model


@dataclass
class TrainConfig:
    """SPEC.md TrainConfig: paper values 2e-3 -> 2e-4, 20 % warm-up, batch 2^19, 30K iterations."""

    lr_init: float = 2e-3
    lr_final: float = 2e-4
    warmup_frac: float = 0.2
    batch_size: int = 1 << 15
    iterations: int = 5000
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-8
    pos_weight: float = 2.0
    seed: int = 0

    def __post_init__(self):
        if not (0.0 < self.lr_final <= self.lr_init):
            raise ValueError("need 0 < lr_final <= lr_init")
        if not (0.0 < self.warmup_frac < 1.0):
            raise ValueError("warmup_frac must be in (0, 1)")
        if self.batch_size < 1 or self.iterations < 1:
            raise ValueError("batch_size and iterations must be >= 1")


def lr_at(t: int, cfg: TrainConfig) -> float:
    """Learning rate of iteration t = 1..N: cosine ramp 0 -> lr_init over the first
    warmup_frac N iterations, then lr_init (lr_final / lr_init)^((t - t_w) / (N - t_w))."""
    n = cfg.iterations
    tw = cfg.warmup_frac * n
    if t <= tw:
        return cfg.lr_init * 0.5 * (1.0 - math.cos(math.pi * t / tw))
    return cfg.lr_init * (cfg.lr_final / cfg.lr_init) ** ((t - tw) / (n - tw))


class _Net:
    """The two MLPs as torch parameters (float32 or float64)."""

    def __init__(self, model: VisibilityModel, device, dtype):
        import torch

        def params(mlp: Mlp):
            return ([torch.tensor(w, dtype=dtype, device=device, requires_grad=True) for w in mlp.weights],
                    [torch.tensor(b, dtype=dtype, device=device, requires_grad=True) for b in mlp.biases])

        self.fw, self.fb = params(model.feature_mlp)
        self.vw, self.vb = params(model.vis_mlp)

    def parameters(self):
        return self.fw + self.fb + self.vw + self.vb

    @staticmethod
    def _mlp(x, ws, bs):
        import torch

        for li, (w, b) in enumerate(zip(ws, bs)):
            x = x @ w.T + b
            if li < len(ws) - 1:
                x = torch.relu(x)
        return x

    def logits(self, geo, feat_in):
        """geo (B, 10) = [mean / r, dir, dist, forward]; feat_in (B, 14) -> (B,) logits."""
        import torch

        feat = self._mlp(feat_in, self.fw, self.fb)
        return self._mlp(torch.cat([geo, feat], dim=1), self.vw, self.vb)[:, 0]

    def to_mlps(self):
        def mlp(ws, bs):
            return Mlp([w.detach().float().cpu().numpy() for w in ws], [b.detach().float().cpu().numpy() for b in bs])

        return mlp(self.fw, self.fb), mlp(self.vw, self.vb)


class _Sampler:
    """Builds the 16-input batches of (view, Gaussian) pairs on the device."""

    def __init__(self, dataset, asset: Asset, model: VisibilityModel, device, dtype):
        import torch

        self.torch = torch
        self.n, self.v = len(asset), dataset.n_views
        t = lambda a: torch.as_tensor(np.asarray(a), dtype=dtype, device=device)   # noqa: E731
        self.means = t(asset.means.astype(np.float64))
        self.feat_in = t(feature_inputs(asset, model.mean_scale).astype(np.float64))
        # camera forward = third row of the world->camera rotation, as the renderer feeds it
        self.pos, self.fwd = t(dataset.positions), t(np.asarray(dataset.rotations)[:, 2, :])
        self.labels = torch.as_tensor(dataset.labels(), device=device)
        self.r, self.dn, self.df = model.mean_scale, model.d_near, model.d_far

    def batch(self, size, gen):
        torch = self.torch
        vi = torch.randint(0, self.v, (size,), generator=gen, device=self.pos.device)
        gi = torch.randint(0, self.n, (size,), generator=gen, device=self.pos.device)
        return self.inputs(vi, gi) + (self.labels[vi, gi].to(self.means.dtype),)

    def inputs(self, vi, gi):
        torch = self.torch
        m = self.means[gi]
        d = m - self.pos[vi]
        d_r = torch.linalg.norm(d, dim=1, keepdim=True)
        dist = torch.clamp(2.0 * (d_r - self.dn) / (self.df - self.dn) - 1.0, -1.0, 1.0)
        geo = torch.cat([m / self.r, d / d_r, dist, self.fwd[vi]], dim=1)
        return geo, self.feat_in[gi]


def train(dataset, asset: Asset, cfg: TrainConfig | None = None, device=None, init: VisibilityModel | None = None,
          log_every: int = 0) -> VisibilityModel:
    """Train a VisibilityModel on ``dataset`` (views of ``asset``); see the module docstring."""
    import torch

    cfg = cfg or TrainConfig()
    if dataset.n_views < 1 or dataset.n_gaussians < 1:
        raise ValueError("dataset is empty")
    if dataset.n_gaussians != len(asset):
        raise ValueError("dataset and asset disagree on the number of Gaussians")
    if dataset.asset_hash != asset_hash(asset):
        raise ValueError("dataset was extracted from a different asset")
    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    # f_train = the extraction cameras' focal, so d_t = d_r on every training view
    model = init or make_model(asset, seed=cfg.seed, f_train=dataset.config.train_focal)
    net = _Net(model, dev, torch.float32)
    smp = _Sampler(dataset, asset, model, dev, torch.float32)
    opt = torch.optim.Adam(net.parameters(), lr=cfg.lr_init, betas=tuple(cfg.betas), eps=cfg.eps)
    pw = torch.tensor(cfg.pos_weight, device=dev)
    gen = torch.Generator(device=dev).manual_seed(cfg.seed)
    loss_v = float("nan")
    for it in range(1, cfg.iterations + 1):
        lr = lr_at(it, cfg)
        for g in opt.param_groups:
            g["lr"] = lr
        geo, fin, y = smp.batch(cfg.batch_size, gen)
        loss = torch.nn.functional.binary_cross_entropy_with_logits(net.logits(geo, fin), y, pos_weight=pw)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        if it == cfg.iterations or (log_every and it % log_every == 0):
            loss_v = float(loss.detach())
            if not math.isfinite(loss_v):
                raise FloatingPointError(f"non-finite loss at iteration {it} (lr {lr:.3g})")
            if log_every:
                print(f"  iter {it}: loss {loss_v:.5f} lr {lr:.2e}", flush=True)
    feat, vis = net.to_mlps()
    meta = dict(model.meta)
    meta.update({"final_loss": loss_v, "iterations": cfg.iterations, "batch_size": cfg.batch_size,
                 "pos_weight": cfg.pos_weight})
    return VisibilityModel(feat, vis, model.mean_scale, model.d_near, model.d_far, model.f_train,
                           threshold=model.threshold, asset_hash=model.asset_hash, meta=meta)


def evaluate(model: VisibilityModel, dataset, asset: Asset, views=None, device=None) -> dict:
    """Accuracy / recall / keep-rate of ``model`` on the dataset's labels (all Gaussians of the given views)."""
    import torch

    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    net = _Net(model, dev, torch.float32)
    smp = _Sampler(dataset, asset, model, dev, torch.float32)
    views = range(dataset.n_views) if views is None else views
    tp = fp = fn = tn = 0
    thr = model.logit_threshold
    with torch.no_grad():
        for v in views:
            gi = torch.arange(smp.n, device=dev)
            vi = torch.full_like(gi, int(v))
            geo, fin = smp.inputs(vi, gi)
            pred = net.logits(geo, fin) >= thr
            y = smp.labels[int(v)]
            tp += int((pred & y).sum())
            fp += int((pred & ~y).sum())
            fn += int((~pred & y).sum())
            tn += int((~pred & ~y).sum())
    tot = tp + fp + fn + tn
    return {"accuracy": (tp + tn) / tot, "recall": tp / max(1, tp + fn), "keep_rate": (tp + fp) / tot,
            "visible_rate": (tp + fn) / tot}


def grad_check(model: VisibilityModel, geo: np.ndarray, feat_in: np.ndarray, labels: np.ndarray,
               pos_weight: float = 2.0, h: float = 1e-5) -> float:
    """Max relative error between autograd and central-difference gradients of the
    weighted BCE w.r.t. every weight, in float64 (SPEC nn.grad_check)."""
    import torch

    net = _Net(model, torch.device("cpu"), torch.float64)
    g = torch.as_tensor(geo, dtype=torch.float64)
    f = torch.as_tensor(feat_in, dtype=torch.float64)
    y = torch.as_tensor(labels, dtype=torch.float64)
    pw = torch.tensor(pos_weight, dtype=torch.float64)

    def loss_fn():
        return torch.nn.functional.binary_cross_entropy_with_logits(net.logits(g, f), y, pos_weight=pw)

    loss = loss_fn()
    grads = torch.autograd.grad(loss, net.parameters())
    worst = 0.0
    with torch.no_grad():
        for p, gp in zip(net.parameters(), grads):
            flat, gflat = p.view(-1), gp.reshape(-1)
            for i in range(flat.numel()):
                old = float(flat[i])
                flat[i] = old + h
                lp = float(loss_fn())
                flat[i] = old - h
                lm = float(loss_fn())
                flat[i] = old
                num = (lp - lm) / (2.0 * h)
                ana = float(gflat[i])
                worst = max(worst, abs(num - ana) / max(abs(num), abs(ana), 1e-6))
    return worst
