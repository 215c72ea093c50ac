"""GPU input generator == CPU input generator, bit for bit (the two sides of the shared input recipe)."""
import numpy as np
import pytest

import synth
from synth import models

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("family", ["real", "exact"])
def test_gpu_generator_matches_cpu_full_tiny(family):
    import torch
    wl = models.Workload("t", [("a", 999_937, 0), ("b", 1023, 1), ("c", 65_536, 2)], 2, 3, family=family,
                         injections=[dict(u=3, kind="NAN", r=1, k=2, i=7)])
    lay = synth.Layout(wl)
    out = torch.empty(lay.n, dtype=torch.int16, device="cuda")
    for (u, r, k, e) in [(1, 0, 1, 7), (3, 1, 2, 5), (9, 1, 3, -5)]:
        synth.micro_grad_gpu(out, wl, lay, u, r, k, e)
        torch.cuda.synchronize()
        ref = synth.micro_grad_cpu(wl, lay, u, r, k, e)
        assert np.array_equal(out.cpu().numpy().view(np.uint16), ref)
    th = torch.empty(lay.n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(th, wl)
    assert np.array_equal(th.cpu().numpy(), synth.theta0_cpu(wl, lay))


def test_gpu_generator_matches_cpu_sampled_big():
    import torch
    wl = models.big_ende()
    lay = synth.Layout(wl)
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rng.integers(0, lay.n, 4096), lay.begin[1:-1], lay.begin[1:-1] - 1,
                                    [0, lay.n - 1]]))
    out = torch.empty(lay.n, dtype=torch.int16, device="cuda")
    synth.micro_grad_gpu(out, wl, lay, 2, 0, 16, 7)
    got = out[torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint16)
    assert np.array_equal(got, synth.micro_grad_sample(wl, lay, idx, 2, 0, 16, 7))


def test_gpu_generator_row_sparse_embedding_matches_cpu():
    """The row-sparse embedding option gives the same bits on both sides, partial last row too."""
    import torch
    wl = models.Workload("t", [("a", 70_001, 0), ("e", 4001 * 64 + 17, 2)], 2, 2, embed_row=64)
    lay = synth.Layout(wl)
    out = torch.empty(lay.n, dtype=torch.int16, device="cuda")
    for (u, r, k) in [(1, 0, 1), (2, 1, 2), (7, 0, 2)]:
        synth.micro_grad_gpu(out, wl, lay, u, r, k, 7)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint16), synth.micro_grad_cpu(wl, lay, u, r, k, 7))
