"""A real Transformer-big producer for the update step: the micro-gradients of row a1 computed by an
actual forward + backward of the paper's model, not emulated.

The model is PAPER.md 3.2: the "big" Transformer, 6 encoder + 6 decoder blocks, word representations of
1024, feed-forward inner dimension 4,096, 16 attention heads, residual connections followed by layer normalisation
(post-LN), ReLU, dropout 0.3 (En-De) / 0.1 (En-Fr), label smoothing 0.1, source / target / output embeddings shared
(210M parameters En-De, 222M En-Fr), sinusoidal positions (no parameters).  The parameter tensors are
exactly synth/models.py's list, in the same packed ready order.

What it does per micro-batch:
  * forward in FP16 straight on the library's fp16 weights (smpu_weights_fp16: zero-copy views);
  * the loss is the label-smoothed cross-entropy SUMMED over the non-pad target tokens (reading R11), multiplied by
    the library's device loss scale 2^e right after the forward pass -- no host round trip;
  * backward in FP16 (torch autograd, cuBLAS GEMMs, flash attention); as each parameter's gradient is complete
    (a post-accumulate-grad hook) it is copied into a packed fp16 gradient buffer in ready order and announced
    (`on_tensor(j)`), so the harness can hand a bucket to the library the moment its last tensor is in (P:211:
    "when the gradient computation for a layer finishes, we add the result to a synchronization buffer").

Synthetic data (no datasets here): token ids uniform over the shared vocabulary (the special ids 0..3 excluded),
sentences of one length per micro-batch (fairseq batches by length), B x L <= the token budget (3.5k).
This module is a producer (harness), not the product: nothing in paper_1806_00187_b200/ imports it.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F


class _View:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def device_view(ptr: int, n: int, dtype: str, device) -> torch.Tensor:
    """A torch tensor over library-owned device memory (typestr <f2 / <f4)."""
    return torch.as_tensor(_View(ptr, n, dtype), device=device)


class TransformerBig:
    """Functional Transformer-big over a packed fp16 weight vector (ready order, synth/models.py names)."""

    def __init__(self, tensors, w16: torch.Tensor, d=1024, heads=16, ffn=4096, layers=6, dropout=0.3,
                 label_smoothing=0.1, max_len=1024):
        self.d, self.h, self.ffn, self.L = d, heads, ffn, layers
        self.dropout, self.eps_ls = dropout, label_smoothing
        self.names = [t[0] for t in tensors]
        self.numel = [int(t[1]) for t in tensors]
        self.offsets = np.concatenate([[0], np.cumsum(self.numel)]).astype(np.int64)
        self.index = {nm: j for j, nm in enumerate(self.names)}
        self.w16 = w16
        self.vocab = self.numel[self.index["embed_tokens.weight"]] // d
        self.device = w16.device
        # sinusoidal positions (Vaswani et al.), no parameters
        pos = torch.arange(max_len, dtype=torch.float32)[:, None]
        i = torch.arange(d // 2, dtype=torch.float32)[None, :]
        ang = pos / torch.pow(10000.0, 2 * i / d)
        self.pos = torch.cat([torch.sin(ang), torch.cos(ang)], 1).to(self.device, torch.float16)

    def _shape(self, name):
        n = self.numel[self.index[name]]
        d = self.d
        if name == "embed_tokens.weight":
            return (self.vocab, d)
        if name.endswith("in_proj.weight"):
            return (3 * d, d)
        if name.endswith("fc1.weight"):
            return (self.ffn, d)
        if name.endswith("fc2.weight"):
            return (d, self.ffn)
        if name.endswith("out_proj.weight"):
            return (d, d)
        return (n,)

    def leaves(self):
        """Fresh autograd leaves sharing the library's weight storage (one set per micro-batch)."""
        P = {}
        for j, nm in enumerate(self.names):
            a, b = int(self.offsets[j]), int(self.offsets[j + 1])
            P[nm] = self.w16[a:b].view(self._shape(nm)).detach().requires_grad_(True)
        return P

    # ------------------------------------------------------------------------------------------ layers
    def _drop(self, x):
        return F.dropout(x, self.dropout, True) if self.dropout > 0 else x

    def _attn(self, P, pre, x, mem=None, causal=False):
        """Multi-head attention with fused in_proj (fairseq layout: rows [q; k; v])."""
        B, T, d = x.shape
        W, bias = P[pre + ".in_proj.weight"], P[pre + ".in_proj.bias"]
        if mem is None:
            q, k, v = F.linear(x, W, bias).chunk(3, dim=-1)
        else:
            q = F.linear(x, W[:d], bias[:d])
            k, v = F.linear(mem, W[d:], bias[d:]).chunk(2, dim=-1)
        S = k.shape[1]
        q = q.view(B, T, self.h, d // self.h).transpose(1, 2)
        k = k.view(B, S, self.h, d // self.h).transpose(1, 2)
        v = v.view(B, S, self.h, d // self.h).transpose(1, 2)
        o = F.scaled_dot_product_attention(q, k, v, is_causal=causal)
        o = o.transpose(1, 2).reshape(B, T, d)
        return F.linear(o, P[pre + ".out_proj.weight"], P[pre + ".out_proj.bias"])

    def _ln(self, P, pre, x):
        return F.layer_norm(x, (self.d,), P[pre + ".weight"], P[pre + ".bias"])

    def _ffn(self, P, pre, x):
        h = F.relu(F.linear(x, P[pre + ".fc1.weight"], P[pre + ".fc1.bias"]))
        return F.linear(h, P[pre + ".fc2.weight"], P[pre + ".fc2.bias"])

    def _embed(self, P, tok):
        E = P["embed_tokens.weight"]
        x = F.embedding(tok, E) * math.sqrt(self.d) + self.pos[: tok.shape[1]]
        return self._drop(x)

    def loss(self, P, src, tgt_in, tgt_out):
        """Label-smoothed cross-entropy summed over the target tokens (fp32 accumulation of an fp16 network)."""
        x = self._embed(P, src)
        for l in range(self.L):
            p = f"encoder.layers.{l}"
            x = self._ln(P, p + ".ln1", x + self._drop(self._attn(P, p + ".self_attn", x)))
            x = self._ln(P, p + ".ln2", x + self._drop(self._ffn(P, p, x)))
        mem = x
        y = self._embed(P, tgt_in)
        for l in range(self.L):
            p = f"decoder.layers.{l}"
            y = self._ln(P, p + ".ln1", y + self._drop(self._attn(P, p + ".self_attn", y, causal=True)))
            y = self._ln(P, p + ".ln2", y + self._drop(self._attn(P, p + ".encoder_attn", y, mem=mem)))
            y = self._ln(P, p + ".ln3", y + self._drop(self._ffn(P, p, y)))
        logits = F.linear(y, P["embed_tokens.weight"])                 # tied output projection
        return F.cross_entropy(logits.float().view(-1, self.vocab), tgt_out.reshape(-1), reduction="sum",
                               label_smoothing=self.eps_ls)


class Producer:
    """Runs micro-batches of the model and writes their fp16 gradients, packed in ready order, into `grad`
    (fp16[n]); `on_tensor(j)` fires once tensor j's gradient is in place (stream-ordered on the current stream)."""

    def __init__(self, model: TransformerBig, grad: torch.Tensor, loss_scale: torch.Tensor, seed=0):
        self.m, self.grad, self.scale = model, grad, loss_scale
        self.gen = torch.Generator(device=model.device)
        self.gen.manual_seed(seed)

    def batch(self, tokens=3500, length=28):
        """B sentences of `length` source and target tokens, B * length <= tokens (P:317's 3.5k budget)."""
        B = max(1, tokens // length)
        V = self.m.vocab
        src = torch.randint(4, V, (B, length), device=self.m.device, generator=self.gen)
        tgt = torch.randint(4, V, (B, length + 1), device=self.m.device, generator=self.gen)
        return src, tgt[:, :-1], tgt[:, 1:], B * length

    def micro(self, src, tgt_in, tgt_out, on_tensor=None):
        """One forward + backward; returns the (unscaled) loss sum as a device scalar."""
        m = self.m
        P = m.leaves()
        handles = []
        for nm, p in P.items():
            j = m.index[nm]
            a, b = int(m.offsets[j]), int(m.offsets[j + 1])

            def hook(t, a=a, b=b, j=j):
                self.grad[a:b].copy_(t.grad.reshape(-1))
                t.grad = None
                if on_tensor is not None:
                    on_tensor(j)
            handles.append(p.register_post_accumulate_grad_hook(hook))
        loss = m.loss(P, src, tgt_in, tgt_out)
        (loss * self.scale[0]).backward()                  # the scaled token-SUM loss (R11)
        for h in handles:
            h.remove()
        return loss.detach()

    def flops_per_token(self):
        """Dense GEMM flops of forward + backward per target token (6 x the non-embedding weights touched per token
        + the tied output projection), attention score flops excluded -- a Table 1-style load figure."""
        m = self.m
        w = sum(nm_n for nm, nm_n in zip(m.names, m.numel) if nm.endswith(".weight") and "ln" not in nm
                and nm != "embed_tokens.weight")
        return 6 * (w + m.vocab * m.d)


class GraphedProducer:
    """Producer.micro captured once per batch shape as a CUDA graph -- forward, backward and the per-tensor gradient
    copies into the packed buffer -- and replayed, so the producer runs at GPU speed instead of Python / launch
    speed (CUDA graphs instead of a tracing compiler).  Inside the graph, the completion of bucket b's last tensor
    gradient records the external event `bucket_done[b]`: a consumer stream can wait on it and hand bucket b to
    the library while the rest of the backward still runs."""

    def __init__(self, prod: Producer, tensor_bucket, n_buckets):
        self.p = prod
        self.tb = list(tensor_bucket)
        self.nb = n_buckets
        self.graphs = {}

    def _capture(self, shape):
        m, p = self.p.m, self.p
        S, Ls, Lt = shape
        dev = m.device
        st = {"src": torch.randint(4, m.vocab, (S, Ls), device=dev, generator=p.gen),
              "ti": torch.randint(4, m.vocab, (S, Lt), device=dev, generator=p.gen),
              "to": torch.randint(4, m.vocab, (S, Lt), device=dev, generator=p.gen)}
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):               # warm-up outside the graph (allocator, kernel selection)
            for _ in range(3):
                p.micro(st["src"], st["ti"], st["to"])
        torch.cuda.current_stream(dev).wait_stream(side)
        events = [torch.cuda.Event(external=True) for _ in range(self.nb)]
        left = np.bincount(self.tb, minlength=self.nb)

        def on_tensor(j):
            b = self.tb[j]
            left[b] -= 1
            if left[b] == 0:
                events[b].record()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            loss = p.micro(st["src"], st["ti"], st["to"], on_tensor=on_tensor)
        assert (left == 0).all(), "every bucket must complete inside the graph"
        self.graphs[shape] = (g, st, events, loss)
        return self.graphs[shape]

    def forget(self):
        """Drop every captured graph (and its private memory pool)."""
        self.graphs.clear()
        torch.cuda.empty_cache()

    def micro(self, src, tgt_in, tgt_out):
        """Replay the graph of this batch shape on the current stream; returns the bucket events (recorded by the
        replay) and the static loss tensor."""
        shape = (src.shape[0], src.shape[1], tgt_in.shape[1])
        g, st, events, loss = self.graphs.get(shape) or self._capture(shape)
        st["src"].copy_(src)
        st["ti"].copy_(tgt_in)
        st["to"].copy_(tgt_out)
        g.replay()
        return events, loss
