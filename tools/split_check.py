"""fp32 mode projector: split-bf16 tcgen05 MLP vs the CUDA-core fp32 GEMMs
(FSB_MLP_SIMT) on 4096 C3 meshes -- max |d theta| / max |theta| (run twice,
once per mode, comparing against a saved file):
    python tools/split_check.py save /tmp/simt.npy   (with FSB_MLP_SIMT=1)
    python tools/split_check.py cmp  /tmp/simt.npy"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    import bench
    from paper_2603_15603_b200 import runtime as rt

    pipe, _ = bench.build_models("fp32")
    ctx = pipe.context()
    n = 4096
    rng = np.random.default_rng(3)
    p = np.zeros((n, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(n, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(n, 10))
    ctx.reserve(n)
    poses = torch.from_numpy(p).cuda()
    v = torch.empty((n, pipe.mhr.num_vertices, 3), device="cuda")
    th = torch.empty((n, 76), device="cuda")
    j = torch.empty((n, 22, 3), device="cuda")
    ctx.check(ctx.lib.fsb_skin_project(ctx.h, rt.ptr(poses), n, rt.ptr(v), rt.ptr(th), rt.ptr(j), None,
                                       rt.PRECISIONS["fp32"], ctx.stream))
    torch.cuda.synchronize()
    t = th.cpu().numpy()
    if sys.argv[1] == "save":
        np.save(sys.argv[2], t)
    else:
        ref = np.load(sys.argv[2])
        print("split-bf16 vs fp32 SIMT: max|d|/max|theta| = %.3g, mean rel per mesh %.3g" % (
            np.abs(t - ref).max() / np.abs(ref).max(),
            (np.abs(t - ref).max(axis=1) / np.abs(ref).max(axis=1)).mean()))
