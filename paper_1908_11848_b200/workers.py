"""PyTorch workers on the engine.

Replaces the reference's numpy worker side (engine.py:251-286: a worker
computes a mini-batch gradient on its local weights, pushes it, and pulls
fresh weights) with real forward/backward passes. Every parameter and every
gradient of the model is a VIEW into one flat fp32 CUDA buffer, so

  * push reads the gradient in place: ``server.handle_push(GradientVector(
    flat_grad, w, it), now)`` hands the engine a device pointer, no copy;
  * pull writes the parameters in place: ``server.handle_pull(w,
    out=flat_param)`` materializes the server's weights straight into them.

The server applies ``lr * grad`` (the reference's update rule, server.py:37);
the worker never steps an optimizer of its own.
"""

from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F

from .server import GradientVector


class _Basic(nn.Module):
    def __init__(self, cin, cout, stride):
        super().__init__()
        self.c1 = nn.Conv2d(cin, cout, 3, stride, 1, bias=False)
        self.b1 = nn.BatchNorm2d(cout)
        self.c2 = nn.Conv2d(cout, cout, 3, 1, 1, bias=False)
        self.b2 = nn.BatchNorm2d(cout)
        self.short = None
        if stride != 1 or cin != cout:
            self.short = nn.Sequential(nn.Conv2d(cin, cout, 1, stride, bias=False), nn.BatchNorm2d(cout))

    def forward(self, x):
        y = F.relu(self.b1(self.c1(x)))
        y = self.b2(self.c2(y))
        return F.relu(y + (x if self.short is None else self.short(x)))


class CifarResNet(nn.Module):
    """He et al. CIFAR ResNet-(6n+2): 16/32/64 channels, basic blocks.
    depth 20 -> 272,474 parameters (configs[1]); 110 -> 1,730,714 (configs[3])."""

    def __init__(self, depth=20, num_classes=10):
        super().__init__()
        assert (depth - 2) % 6 == 0
        n = (depth - 2) // 6
        self.conv = nn.Conv2d(3, 16, 3, 1, 1, bias=False)
        self.bn = nn.BatchNorm2d(16)
        layers, cin = [], 16
        for cout, stride in ((16, 1), (32, 2), (64, 2)):
            for i in range(n):
                layers.append(_Basic(cin, cout, stride if i == 0 else 1))
                cin = cout
        self.layers = nn.Sequential(*layers)
        self.fc = nn.Linear(64, num_classes)

    def forward(self, x):
        y = F.relu(self.bn(self.conv(x)))
        y = self.layers(y)
        return self.fc(F.adaptive_avg_pool2d(y, 1).flatten(1))


def resnet50_cifar(num_classes=10):
    """ResNet-50 with a 10-class head: 23,528,522 parameters (configs[2])."""
    import torchvision
    return torchvision.models.resnet50(num_classes=num_classes)


def flatten_(model: nn.Module, device="cuda", into=None, copy_params=True):
    """Re-home every parameter and its gradient as views of two flat fp32
    buffers (padded to a multiple of 4 floats). ``into=(params, grads)``
    uses caller-owned buffers instead -- e.g. a sharded server's replica and
    update buffer, so pulls land in the parameters and pushes read the
    gradients with no copy at all. Returns (params, grads, n)."""
    params = [p for p in model.parameters()]
    n = sum(p.numel() for p in params)
    pad = (n + 3) // 4 * 4
    if into is None:
        flat_p = torch.zeros(pad, dtype=torch.float32, device=device)
        flat_g = torch.zeros(pad, dtype=torch.float32, device=device)
    else:
        flat_p, flat_g = into
        if flat_p.numel() < n or flat_g.numel() < n:
            raise ValueError(f"buffers hold {flat_p.numel()} / {flat_g.numel()} floats, model has {n}")
    off = 0
    for p in params:
        k = p.numel()
        if copy_params:
            flat_p[off:off + k].copy_(p.data.reshape(-1))
        p.data = flat_p[off:off + k].view_as(p)
        p.grad = flat_g[off:off + k].view_as(p)
        off += k
    return flat_p, flat_g, n


class TorchWorker:
    """One data-parallel worker: local replica, a data shard, fwd/bwd."""

    def __init__(self, worker_id, model, batches, device="cuda"):
        self.worker = worker_id
        self.model = model.to(device)
        self.params, self.grads, self.dimension = flatten_(self.model, device)
        self.batches = batches          # list of (x, y) CUDA tensors
        self.cursor = 0
        self.iterations = 0
        self.last_loss = float("nan")

    def adopt_from(self, server):
        """handle_pull straight into the parameters (server.py:84-91)."""
        server.handle_pull(self.worker, out=self.params[:self.dimension])

    def step(self):
        """Forward + backward on the current stream into the flat gradient
        buffer (one static batch: the body of a captured iteration graph,
        freerun.FreeRunningCluster)."""
        x, y = self.batches[0]
        self.grads.zero_()
        loss = F.cross_entropy(self.model(x), y)
        loss.backward()
        self.iterations += 1

    def begin_iteration(self):
        """engine.py:263-272: next batch, loss and gradient at the local weights."""
        x, y = self.batches[self.cursor]
        self.cursor = (self.cursor + 1) % len(self.batches)
        self.grads.zero_()
        loss = F.cross_entropy(self.model(x), y)
        loss.backward()
        self.iterations += 1
        self.last_loss = loss.detach()
        return GradientVector(self.grads[:self.dimension], self.worker, self.iterations)


class SyntheticWorker:
    """A worker whose "backward" writes the next of K resident updates into its
    gradient buffer (device-side index, so the step is graph-capturable):
    push k carries ring[k % K]. For parity runs of the free-running path."""

    def __init__(self, ring, device="cuda"):
        self.ring = ring                                   # [K, dpad] fp32
        self.K, self.dpad = ring.shape
        self.params = torch.zeros(self.dpad, dtype=torch.float32, device=device)
        self.grads = torch.zeros(self.dpad, dtype=torch.float32, device=device)
        self.idx = torch.zeros(1, dtype=torch.long, device=device)

    def step(self):
        self.grads.copy_(self.ring.index_select(0, self.idx).squeeze(0))
        self.idx.add_(1).remainder_(self.K)


def synthetic_cifar(n_batches, batch, seed, device="cuda"):
    """32x32x3, 10-class synthetic data (no dataset download on the box)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    out = []
    for _ in range(n_batches):
        x = torch.randn(batch, 3, 32, 32, generator=g).to(device)
        y = torch.randint(0, 10, (batch,), generator=g).to(device)
        out.append((x, y))
    return out
