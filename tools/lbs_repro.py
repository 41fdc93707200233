"""fsb_skin on a few meshes (debugging aid for the LBS kernels)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_15603_b200 import runtime as rt  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
pipe, _ = bench.build_models("bf16")
ctx = pipe.context()
ctx.reserve(B)
p = torch.from_numpy(np.random.default_rng(0).normal(0, 0.2, (B, 76)).astype(np.float32)).cuda()
v = torch.empty((B, pipe.mhr.num_vertices, 3), device="cuda")
ctx.check(ctx.lib.fsb_skin(ctx.h, 0, rt.ptr(p), B, rt.ptr(v), ctx.stream))
torch.cuda.synchronize()
print("ok", float(v.abs().max()))
