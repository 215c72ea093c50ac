#!/usr/bin/env python
"""A real fp16 training loop with libsmpu as its update step (the fairseq-style usage of the paper's method).

The model is a tiny tied-embedding language model (embedding -> 2 ReLU layers -> output projection shared with
the embedding, P:93-102's weight tying at toy scale) on a learnable synthetic task.  Everything the paper puts on
the update path is the library's:
  * the model's fp16 weights ARE the library's w16 buffer (zero-copy views, "forward-backward ... in FP16");
  * the loss is scaled by the library's device loss scale -- no host round trip;
  * each micro-batch's token-SUM gradients are packed in ready order (reverse forward order) and handed
    to smpu_accumulate with the micro-batch's token count; update_freq of them make one update;
  * smpu_step does the overflow test, scaler, LR, Adam, fp16 re-cast.
    python examples/train_tiny.py            (one B200)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1806_00187_b200 as P  # noqa: E402


class _View:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def run(updates=150, update_freq=4, V=64, d=64, tokens=512, seed=0, peak_lr=3e-3, warmup=20, verbose=True):
    torch.manual_seed(seed)
    dev = torch.device("cuda")
    # forward-order parameter shapes; ready order is the reverse, tied embedding last
    fwd = [("emb", (V, d)), ("w1", (d, d)), ("b1", (d,)), ("w2", (d, d)), ("b2", (d,))]
    ready = list(reversed(fwd[1:])) + [fwd[0]]
    numel = [int(np.prod(s)) for _, s in ready]
    init = torch.cat([(torch.randn(int(np.prod(s))) * (0.1 if len(s) == 2 else 0.0)) for _, s in ready]).float()
    cfg = P.config_default(update_freq=update_freq, peak_lr=peak_lr, warmup_updates=warmup)
    step = P.UpdateStep(numel, init.numpy(), cfg)
    w16 = torch.as_tensor(_View(step.weights_fp16_ptr(), step.n, "<f2"), device=dev)
    scale = torch.as_tensor(_View(step.loss_scale_ptr(), 1, "<f4"), device=dev)
    offs = np.concatenate([[0], np.cumsum(numel)])
    W = {name: w16[offs[j]:offs[j + 1]].view(*shape) for j, (name, shape) in enumerate(ready)}
    grad_buf = torch.empty(step.n, dtype=torch.float16, device=dev)
    # synthetic task: next token = (3 * token + 1) mod V, with 10% label noise
    losses, scales = [], []
    for u in range(updates):
        tot = 0.0
        for k in range(update_freq):
            x = torch.randint(0, V, (tokens,), device=dev)
            y = (3 * x + 1) % V
            noise = torch.rand(tokens, device=dev) < 0.1
            y = torch.where(noise, torch.randint(0, V, (tokens,), device=dev), y)
            params = {n: t.detach().requires_grad_(True) for n, t in W.items()}
            h = params["emb"][x]
            h = torch.relu(h @ params["w1"].t() + params["b1"])
            h = torch.relu(h @ params["w2"].t() + params["b2"])
            logits = h @ params["emb"].t()                              # tied output projection
            loss_sum = torch.nn.functional.cross_entropy(logits.float(), y, reduction="sum")
            (loss_sum * scale[0]).backward()                           # scaled token-SUM loss
            for j, (name, _) in enumerate(ready):
                grad_buf[offs[j]:offs[j + 1]].copy_(params[name].grad.reshape(-1))
            step.accumulate(grad_buf.view(torch.int16), tokens)
            tot += loss_sum.item()
        res = step.step()
        losses.append(tot / (tokens * update_freq))
        scales.append(res["scale_log2_next"])
        if verbose and (u % 25 == 0 or u == updates - 1):
            print(f"update {u:4d}  loss/token {losses[-1]:.4f}  scale 2^{res['scale_log2_used']}  "
                  f"lr {res['lr']:.2e}  applied {res['applied']}")
    step.close()
    return losses, scales


if __name__ == "__main__":
    run()
