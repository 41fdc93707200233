"""Hardware checks of the tcgen05 primitives (smem descriptors, instruction
descriptor, TMEM alloc/ld, mbarrier commit, bulk copy) the bf16 kernels use."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bf16(rng, shape, scale=1.0):
    from paper_2603_15603_b200 import runtime as rt

    bits = rt.to_bf16_bits((rng.standard_normal(shape) * scale).astype(np.float32))
    return bits, rt.bf16_bits_to_f32(bits).astype(np.float64)


@pytest.mark.parametrize("m,n,k,kind", [(300, 256, 512, 0), (128, 384, 64, 1), (700, 1024, 1024, 2),
                                        (576 * 2, 1024, 768, 3), (20000, 768, 128, 2), (5000, 3072, 64, 0),
                                        (3000, 96, 256, 1)])
def test_tma_gemm(m, n, k, kind):
    """TMA (128B swizzle) + tcgen05 GEMM with each fused epilogue."""
    import ctypes

    import torch

    from paper_2603_15603_b200 import runtime as rt

    rng = np.random.default_rng(m + n + k)
    ab, a = _bf16(rng, (m, k))
    wb, w = _bf16(rng, (n, k), 0.05)
    bias = rng.standard_normal(n).astype(np.float32)
    ref = a @ w.T + bias
    lib = ctypes.CDLL(rt.LIB_PATH)
    da = torch.from_numpy(ab.view(np.int16)).cuda()
    dw = torch.from_numpy(wb.view(np.int16)).cuda()
    db = torch.from_numpy(bias).cuda()
    out = torch.zeros((m, n), dtype=torch.int16, device="cuda")
    x0 = rng.standard_normal((m, n)).astype(np.float32)
    x = torch.from_numpy(x0.copy()).cuda()
    pos = rng.standard_normal((576, n)).astype(np.float32)
    dpos = torch.from_numpy(pos).cuda()
    P = ctypes.c_void_p
    lib.fsb_debug_gemm.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P,
                                   ctypes.c_int, P]
    rc = lib.fsb_debug_gemm(da.data_ptr(), dw.data_ptr(), db.data_ptr(), m, n, k, kind, out.data_ptr(),
                            x.data_ptr(), dpos.data_ptr(), 576, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    if kind in (0, 1):
        got = rt.bf16_bits_to_f32(out.cpu().numpy().view(np.uint16))
        want = np.maximum(ref, 0.0) if kind == 1 else ref
        assert np.abs(got - want).max() <= 1e-2 * np.abs(want).max()
    else:
        got = x.cpu().numpy()
        want = x0 + ref if kind == 2 else ref + pos[np.arange(m) % 576]
        assert np.abs(got - want).max() <= 1e-4 * np.abs(want).max()


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
