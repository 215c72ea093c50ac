"""Parameter-tensor lists and workload configurations (input STRUCTURE only).

The method never sees a model: it sees a packed fp16 gradient vector whose
segments are the model's parameter tensors in gradient-ready order.  These
lists reproduce the shapes of the paper's models so that the bucket plan and
the element counts are those of the real workload.

* Transformer "big": 6+6 blocks, d=1024, FFN 4096, 16 heads, post-LN residual
  blocks, shared embedding (PAPER.md 3.2 "Models and Hyperparameters", P:92-102;
  210M params En-De, 222M En-Fr).  Counts: SURVEY.md Appendix A.1.
* Transformer "base" (d=512, FFN 2048): BASELINE.json configs[1]; not in the
  paper (reading R21).
* Ready order = reverse of forward order, tied embedding last: "back-propagation
  proceeds sequentially from the top of the network down to the inputs"
  (PAPER.md 4.3).
"""
from __future__ import annotations

from dataclasses import dataclass, field

WEIGHT, BIAS, EMBED = 0, 1, 2  # tensor classes (sigma / q_t selection in synth.c)


def _attn(prefix, d):
    return [(f"{prefix}.in_proj.weight", 3 * d * d, WEIGHT), (f"{prefix}.in_proj.bias", 3 * d, BIAS),
            (f"{prefix}.out_proj.weight", d * d, WEIGHT), (f"{prefix}.out_proj.bias", d, BIAS)]


def _ln(prefix, d):
    return [(f"{prefix}.weight", d, BIAS), (f"{prefix}.bias", d, BIAS)]


def _ffn(prefix, d, f):
    return [(f"{prefix}.fc1.weight", f * d, WEIGHT), (f"{prefix}.fc1.bias", f, BIAS),
            (f"{prefix}.fc2.weight", d * f, WEIGHT), (f"{prefix}.fc2.bias", d, BIAS)]


def transformer_tensors(d: int, ffn: int, vocab: int, layers: int = 6):
    """(name, numel, class) in gradient-READY order (reverse forward order)."""
    fwd = [("embed_tokens.weight", vocab * d, EMBED)]
    for l in range(layers):
        p = f"encoder.layers.{l}"
        fwd += _attn(p + ".self_attn", d) + _ln(p + ".ln1", d) + _ffn(p, d, ffn) + _ln(p + ".ln2", d)
    for l in range(layers):
        p = f"decoder.layers.{l}"
        fwd += (_attn(p + ".self_attn", d) + _ln(p + ".ln1", d) + _attn(p + ".encoder_attn", d)
                + _ln(p + ".ln2", d) + _ffn(p, d, ffn) + _ln(p + ".ln3", d))
    # backward finishes the top first; the tied embedding (input lookup AND output
    # projection) is finished last.  Reverse everything after the embedding, append it.
    return list(reversed(fwd[1:])) + [fwd[0]]


@dataclass
class Workload:
    name: str
    tensors: list            # [(name, numel, cls)] in ready order
    world: int = 1
    update_freq: int = 1
    config_id: int = 0
    injections: list = field(default_factory=list)
    family: str = "real"     # real | exact | zero
    updates: int = 10
    embed_row: int = 0       # > 0: row-sparse embedding gradient with rows of this many elements;
                             # 0: dense (reading R27: the tied output projection touches every row)

    @property
    def numel(self):
        return [t[1] for t in self.tensors]

    @property
    def classes(self):
        return [t[2] for t in self.tensors]

    @property
    def n(self):
        return sum(self.numel)

    @property
    def seed(self):
        return 1234567 ^ self.config_id


def tiny(updates=10, injections=None):
    """BASELINE.json configs[0]: 1M-param fp16 vector, world=1, update_freq=2, 10 steps, one injected inf."""
    inj = [dict(u=5, kind="INF", r=0, k=2, i=123457)] if injections is None else injections
    return Workload("tiny", [("flat.weight", 1_000_000, WEIGHT)], 1, 2, 0, inj, "real", updates)


def base_ende(world=1, update_freq=1):
    """BASELINE.json configs[1]: Transformer-base En-De (~61M params, 32k joint BPE)."""
    return Workload("transformer_base_ende", transformer_tensors(512, 2048, 32768), world, update_freq, 1)


def big_ende(world=1, update_freq=16):
    """BASELINE.json configs[2]: Transformer-big En-De (~210M params), update_freq=16."""
    return Workload("transformer_big_ende", transformer_tensors(1024, 4096, 32768), world, update_freq, 2)


def big_enfr(world=8, update_freq=16, vocab=44512):
    """BASELINE.json configs[3]: Transformer-big En-Fr (40k vocab; V=44,512 gives the paper's 222M, reading R20)
    with a burst of four injected overflows every 2,500 updates."""
    inj = []
    for base in (2500, 5000):
        inj += [dict(u=base, kind="INF", r=0, k=1, i=777),
                dict(u=base + 1, kind="NAN", r=world - 1, k=update_freq, i=4242),
                dict(u=base + 2, kind="ACC_OVF", r=0, i=31337),
                dict(u=base + 3, kind="RED_OVF" if world >= 2 else "NINF", r=0, k=update_freq, i=99991)]
    return Workload("transformer_big_enfr", transformer_tensors(1024, 4096, vocab), world, update_freq, 3,
                    inj, "exact", 5200)


WORKLOADS = {"tiny": tiny, "base": base_ende, "big_ende": big_ende, "big_enfr": big_enfr}
