"""Hardware checks of the tcgen05 primitives (smem descriptors, instruction
descriptor, TMEM alloc/ld, mbarrier commit, bulk copy) the bf16 kernels use."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k", [(16, 16), (64, 64), (128, 64), (192, 64), (256, 256), (64, 512)])
def test_umma_selftest(n, k):
    import torch

    from paper_2603_15603_b200 import runtime as rt

    ctx = rt.default_context()
    rng = np.random.default_rng(n * 1000 + k)
    a = rng.standard_normal((128, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    ab, bb = rt.to_bf16_bits(a), rt.to_bf16_bits(b)
    da = torch.from_numpy(ab.view(np.int16)).cuda()
    db = torch.from_numpy(rt.pack_kmajor(bb).view(np.int16)).cuda()
    c = torch.empty((128, n), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.fsb_selftest_umma(ctx.h, rt.ptr(da), rt.ptr(db), n, k, rt.ptr(c), ctx.stream))
    got = c.cpu().numpy()
    want = rt.bf16_bits_to_f32(ab).astype(np.float64) @ rt.bf16_bits_to_f32(bb).astype(np.float64).T
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < 1e-5, err
