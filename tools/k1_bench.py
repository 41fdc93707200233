"""K1 microbench: fsb_boxes_crops on B frames resident in HBM (per-tap
kernel) and in pinned host memory (bulk-copy row-span kernel), timed as
CUDA-graph replays.

    python tools/k1_bench.py [B]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import numpy as np
    import torch

    import bench
    from paper_2603_15603_b200 import priors as pr
    from paper_2603_15603_b200 import runtime as rt
    from paper_2603_15603_b200 import synth

    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    _, smpl, _ = synth.make_toy_models(0, 1200, 600)
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, 8 * B))
    dimg = pr.render_scenes(scenes)
    dkp = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    himg = dimg.cpu().pin_memory()
    hkp = dkp.cpu().pin_memory()
    ctx = rt.Context()
    boxes = torch.empty((B, 3, 4), dtype=torch.float64, device="cuda")
    prompt = torch.empty((B, 8), device="cuda")
    crops = torch.empty((B, 3, 64, 64, 3), device="cuda")
    res = {"B": B}
    for name, img, kp in (("hbm", dimg, dkp), ("host", himg, hkp)):
        def run(i):
            s = i % 8
            ctx.check(ctx.lib.fsb_boxes_crops(ctx.h, rt.ptr(img[s * B:(s + 1) * B]), B, 512, 512,
                                              rt.ptr(kp[s * B:(s + 1) * B]), 3.0, 64, rt.ptr(boxes),
                                              rt.ptr(prompt), rt.ptr(crops), None, ctx.stream))
        for i in range(8):
            run(i)
        torch.cuda.synchronize()
        # 40 launches captured in one graph: device time, not host launch rate
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
                for i in range(40):
                    run(i)
        g.replay()
        torch.cuda.synchronize()
        ctx.input_bytes(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        n = 40 * reps
        us = e0.elapsed_time(e1) / n * 1e3
        nb = ctx.input_bytes(reset=True) / n
        res[name] = {"us": us, "bytes": nb, "GBps": nb / us / 1e3}
    print(json.dumps(res))
