"""Input generator (synth/) pins: published SplitMix64 vectors, recipe properties, model shapes."""
import numpy as np
import pytest

import synth
from synth import models


def test_splitmix64_published_vectors():
    # Vigna's SplitMix64 reference outputs: seed 0 -> first output 0xe220a8397b1dcdaf, seed 1 ->
    # 0x910a2dec89025cc1; stream of seed 1234567: 6457827717110365317, 3203168211198807973, ...
    assert synth.mix(0) == 0xE220A8397B1DCDAF
    assert synth.mix(1) == 0x910A2DEC89025CC1
    g = 0x9E3779B97F4A7C15
    st = 1234567
    outs = [synth.mix((st + j * g) & (2**64 - 1)) for j in range(3)]
    assert outs == [0x599ED017FB08FC85, 0x2C73F08458540FA5, 0x883EBCE5A3F27C77]


def test_parameter_counts_match_paper():
    # "210M parameters for the En-De dataset and 222M parameters for the En-Fr dataset"
    assert models.big_ende().n == 209_911_808
    assert models.big_enfr().n == 221_937_664
    assert models.base_ende().n == 60_915_712
    assert len(models.big_ende().tensors) == 181
    # ready order: tied embedding last (reading R18)
    assert models.big_ende().tensors[-1][0] == "embed_tokens.weight"
    assert models.big_ende().tensors[0][0].startswith("decoder.layers.5")


def test_real_generator_bounded_and_reproducible():
    wl = models.tiny()
    lay = synth.Layout(wl)
    g1 = synth.micro_grad_cpu(wl, lay, 1, 0, 1, 7)
    g2 = synth.micro_grad_cpu(wl, lay, 1, 0, 1, 7)
    assert np.array_equal(g1, g2)
    x = g1.view(np.float16).astype(np.float64)
    assert np.isfinite(x).all()
    assert np.abs(x).max() < 2.0 ** (-5 + 7)   # |g| < sigma * 2^e
    y = x / 2.0 ** (-5 + 7)   # back to q * 2^-17, Irwin-Hall(4)-shaped on (-1, 1): std = 2*65536/sqrt(12)/2^17 = 0.2887
    assert abs(y.mean()) < 0.005 and abs(y.std() - 0.2887) < 0.005
    idx = np.array([0, 5, 999_999, 123_457], dtype=np.int64)
    assert np.array_equal(synth.micro_grad_sample(wl, lay, idx, 1, 0, 1, 7), g1[idx])


def test_exact_generator_is_exactly_summable():
    wl = models.Workload("t", [("a", 4096, 0), ("b", 512, 1), ("c", 2048, 2)], world=4, update_freq=4,
                         family="exact")
    lay = synth.Layout(wl)
    gs = [synth.micro_grad_cpu(wl, lay, 1, r, k, 7) for r in range(4) for k in range(1, 5)]
    x = np.stack([g.view(np.float16).astype(np.float64) for g in gs])
    tot = x.sum(0)
    assert np.array_equal(tot.astype(np.float16).astype(np.float64), tot)  # every total exactly representable
    rng = np.random.default_rng(0)
    for _ in range(5):   # any order, fp16 rounding after each add: same bits
        perm = rng.permutation(len(gs))
        acc = np.zeros(lay.n, dtype=np.float16)
        for j in perm:
            acc = (acc.astype(np.float32) + x[j].astype(np.float32)).astype(np.float16)
        assert np.array_equal(acc.astype(np.float64), tot)


def test_ntokens_range():
    wl = models.big_ende()
    t = [synth.ntokens(wl, u, 0, k) for u in range(1, 50) for k in range(1, 17)]
    assert min(t) >= 2780 and max(t) <= 3500
    assert 3000 < np.mean(t) < 3280  # mean 3140 ~ 402k/128


def test_injection_overrides():
    wl = models.big_enfr(world=4)
    assert synth.overrides(wl, 2500, 0, 1) == [(777, synth.INF16)]
    assert synth.overrides(wl, 2502, 0, 1) == [(31337, 0x7BFF)]
    assert synth.overrides(wl, 2502, 1, 1) == [(31337, 0)]
    assert synth.overrides(wl, 2503, 2, 16) == [(99991, 0x78E2)]
    assert synth.overrides(wl, 2503, 2, 3) == [(99991, 0)]
    w2 = models.Workload("b", [("a", 10, 0)], 4, 2, injections=[dict(u=1, kind="BIG", i=3)])
    assert synth.overrides(w2, 1, 1, 2) == [(3, 0x74E2)] and synth.overrides(w2, 1, 2, 2) == [(3, 0)]
    assert np.uint16(0x74E2).view(np.float16) == 20000
    with pytest.raises(ValueError):
        synth.overrides(models.Workload("x", [("a", 10, 0)], 1, 2, injections=[dict(u=1, kind="RED_OVF", i=1)]),
                        1, 0, 2)


def test_row_sparse_embedding_zipf_rows():
    """SURVEY 8(d.2)'s row-sparse embedding: the rows drawn for a micro-batch follow Zipf(1.1) over the vocabulary.
    Pinned to the closed forms: E[distinct rows] = sum_v 1 - (1 - p_v)^T and P(row v drawn) = 1 - (1 - p_v)^T,
    over many micro-batches; inactive rows are exactly zero in the fill, active ones keep G_real's values."""
    V = 32_768
    wl = models.Workload("emb", [("w", 4096, 0), ("e", V * 64, 2)], 1, 1, embed_row=64)
    p = np.arange(1, V + 1, dtype=np.float64) ** -1.1
    p /= p.sum()
    ds, hits = [], np.zeros(V)
    Ts = []
    for k in range(1, 41):
        m = synth.embed_mask(wl, V, 1, 0, k).astype(bool)
        T = synth.ntokens(wl, 1, 0, k)
        Ts.append(T)
        ds.append(m.sum())
        hits += m
    T = np.mean(Ts)
    expect = np.sum(1 - (1 - p) ** T)
    assert abs(np.mean(ds) - expect) < 0.03 * expect, (np.mean(ds), expect)
    for v in (0, 9, 99, 999):       # per-row inclusion frequency over the 40 micro-batches
        pv = 1 - (1 - p[v]) ** T
        assert abs(hits[v] / 40 - pv) < 4 * np.sqrt(pv * (1 - pv) / 40) + 0.02, (v, hits[v], pv)
    lay = synth.Layout(wl)
    g = synth.micro_grad_cpu(wl, lay, 1, 0, 1, 7)
    dense = synth.micro_grad_cpu(models.Workload("emb", wl.tensors, 1, 1), lay, 1, 0, 1, 7)
    rows = g[4096:].reshape(V, 64)
    m = synth.embed_mask(wl, V, 1, 0, 1).astype(bool)
    assert not rows[~m].any()
    assert np.array_equal(rows[m], dense[4096:].reshape(V, 64)[m])
    assert np.array_equal(g[:4096], dense[:4096])
