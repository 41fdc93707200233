import ctypes, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2603_15603_b200 import runtime as rt
lib = ctypes.CDLL(rt.LIB_PATH)
P = ctypes.c_void_p
lib.fsb_debug_gemm.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int, P]
for kind in (0, 2, 3):
    m, n, k = 300, 256, 128
    a = torch.randn((m, k), device="cuda").to(torch.bfloat16); w = torch.randn((n, k), device="cuda").to(torch.bfloat16)
    b = torch.randn(n, device="cuda"); out = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    x = torch.randn((m, n), device="cuda"); pos = torch.randn((576, n), device="cuda")
    rc = lib.fsb_debug_gemm(a.data_ptr(), w.data_ptr(), b.data_ptr(), m, n, k, kind, out.data_ptr(), x.data_ptr(), pos.data_ptr(), 576, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize(); print("kind", kind, rc)
