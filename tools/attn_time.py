"""Time the C4 flash-attention kernel alone (fsb_debug_attention) with CUDA
events: python tools/attn_time.py [crops] [T] [D] [reps]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    from paper_2603_15603_b200 import runtime as rt

    crops, T, D, reps = (int(a) for a in (sys.argv[1:5] + ["256", "576", "1024", "20"][len(sys.argv) - 1:]))
    H = D // 64
    lib = ctypes.CDLL(rt.LIB_PATH)
    P = ctypes.c_void_p
    lib.fsb_debug_attention.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = (torch.randn((crops * T, 3 * D), device="cuda", generator=g) * 1.5).to(torch.bfloat16)
    out = torch.empty((crops * T, D), dtype=torch.bfloat16, device="cuda")
    st = torch.cuda.current_stream()
    call = lambda: lib.fsb_debug_attention(qkv.data_ptr(), crops, T, D, H, out.data_ptr(), st.cuda_stream)
    for _ in range(3):
        assert call() == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        call()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flop = 4.0 * T * T * 64 * H * crops
    print("%s attention crops %d T %d D %d: %.1f us/launch, %.0f TFLOP/s"
          % (os.path.basename(rt.LIB_PATH), crops, T, D, ms * 1e3, flop / ms / 1e9))
