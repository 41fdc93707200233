"""One CTA-pair GEMM launch through fsb_debug_gemm (for compute-sanitizer)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    from paper_2603_15603_b200 import runtime as rt

    m, n, k = 512, 512, 256
    a = torch.zeros((m, k), dtype=torch.int16, device="cuda")
    w = torch.zeros((n, k), dtype=torch.int16, device="cuda")
    b = torch.zeros(n, dtype=torch.float32, device="cuda")
    out = torch.zeros((m, n), dtype=torch.int16, device="cuda")
    lib = ctypes.CDLL(rt.LIB_PATH)
    P = ctypes.c_void_p
    lib.fsb_debug_gemm.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P,
                                   ctypes.c_int, P]
    rc = lib.fsb_debug_gemm(a.data_ptr(), w.data_ptr(), b.data_ptr(), m, n, k, 0, out.data_ptr(), None, None, 576,
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    print("rc", rc)
