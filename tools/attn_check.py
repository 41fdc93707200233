"""Run the C4 flash-attention kernel alone on one (crops, T, D) case and
compare with a float64 reference: python tools/attn_check.py crops T D"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    from paper_2603_15603_b200 import runtime as rt

    crops, T, D = (int(a) for a in sys.argv[1:4])
    H = D // 64
    rng = np.random.default_rng(T + D)
    x = (rng.standard_normal((crops * T, 3 * D)) * 1.5).astype(np.float32)
    bits = rt.to_bf16_bits(x)
    lib = ctypes.CDLL(rt.LIB_PATH)
    P = ctypes.c_void_p
    lib.fsb_debug_attention.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
    dq = torch.from_numpy(bits.view(np.int16)).cuda()
    out = torch.zeros((crops * T, D), dtype=torch.int16, device="cuda")
    t0 = time.time()
    assert lib.fsb_debug_attention(dq.data_ptr(), crops, T, D, H, out.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    print("ran in %.3f s" % (time.time() - t0), flush=True)
    qkv = rt.bf16_bits_to_f32(bits).astype(np.float64)
    got = rt.bf16_bits_to_f32(out.cpu().numpy().view(np.uint16)).astype(np.float64)
    err = 0.0
    for c in range(crops):
        r = slice(c * T, (c + 1) * T)
        for h in range(H):
            q = qkv[r, h * 64:(h + 1) * 64]
            k = qkv[r, D + h * 64:D + (h + 1) * 64]
            v = qkv[r, 2 * D + h * 64:2 * D + (h + 1) * 64]
            s = q @ k.T / 8.0
            p = np.exp(s - s.max(axis=1, keepdims=True))
            ref = (p / p.sum(axis=1, keepdims=True)) @ v
            e = np.abs(got[r, h * 64:(h + 1) * 64] - ref).max(axis=1)
            bad = np.nonzero(e > 0.1)[0]
            if len(bad) and c == 0 and h == 0:
                print("bad rows (crop 0, head 0): %d, first %s" % (len(bad), bad[:12]))
            err = max(err, e.max())
    print("crops %d T %d D %d max err %.4g" % (crops, T, D, err))
