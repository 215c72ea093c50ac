"""The real Transformer-big producer (producer/transformer.py) at toy width on CPU: its parameter layout is
synth/models.py's ready-ordered list, every tensor's gradient is announced exactly once, the packed buffer holds the
gradient of the SCALED token-sum loss, and the announcement order is close to ready order with the tied embedding
last."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "producer"))

from synth import models  # noqa: E402
from transformer import Producer, TransformerBig  # noqa: E402


def test_producer_gradients_hooks_and_order():
    torch.manual_seed(0)
    d, ffn, V, L = 32, 64, 101, 2
    tensors = models.transformer_tensors(d, ffn, V, layers=L)
    n = sum(t[1] for t in tensors)
    w = (torch.randn(n) * 0.05).to(torch.float32)
    m = TransformerBig(tensors, w, d=d, heads=4, ffn=ffn, layers=L, dropout=0.0, max_len=64)
    grad = torch.zeros(n, dtype=torch.float32)
    scale = torch.tensor([8.0])
    prod = Producer(m, grad, scale, seed=1)
    src, ti, to, nt = prod.batch(tokens=60, length=6)
    assert nt == 60 and src.shape == (10, 6)
    seen = []
    loss = prod.micro(src, ti, to, on_tensor=seen.append)
    assert sorted(seen) == list(range(len(tensors)))          # each tensor announced exactly once
    assert seen[-1] == len(tensors) - 1                       # the tied embedding is complete last
    # packed gradient == autograd of 8 x the summed loss, computed independently
    P = {k: v.detach().clone().requires_grad_(True) for k, v in m.leaves().items()}
    (m.loss(P, src, ti, to) * 8.0).backward()
    ref = torch.cat([P[t[0]].grad.reshape(-1) for t in tensors])
    assert torch.allclose(grad, ref, rtol=1e-5, atol=1e-6)
    assert float(loss) > 0 and m.vocab == V
    # announcement order follows the backward: mostly the reverse of forward order (Spearman rank correlation)
    r = np.corrcoef(np.argsort(seen), np.arange(len(seen)))[0, 1]
    assert r > 0.9, r
