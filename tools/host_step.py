"""Host cost of one bench step (Pipeline.launch -> fsb_frame_batch graph
replay) against the device time per step, at S in-flight streams."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    import bench
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr

    S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    B = 32
    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models("bf16")
    pipe.context().reserve(B)
    pipes = [pipe] + bench.extra_pipelines(pipe, S - 1, "bf16")
    for p_ in pipes[1:]:
        p_.context().reserve(B)
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, B * 4))
    images = pr.render_scenes(scenes)
    kps = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    streams = [torch.cuda.Stream() for _ in range(S)]
    outs = [p_.allocate_outputs(B, tail=True) for p_ in pipes]
    cfg = pl.fast_config()

    def step(i):
        j, s = i % S, i % 4
        with torch.cuda.stream(streams[j]):
            pipes[j].launch(images[s * B:(s + 1) * B], kps[s * B:(s + 1) * B], outs[j], cfg)

    for i in range(64):
        step(i)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for i in range(n):
        step(i)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("S=%d host us/step %.1f  wall us/step incl drain %.1f" % (S, 1e6 * (t1 - t0) / n, 1e6 * (t2 - t0) / n))
    # pieces
    ctx = pipe.context()
    t0 = time.perf_counter()
    for i in range(n):
        with torch.cuda.stream(streams[0]):
            pass
    t1 = time.perf_counter()
    print("stream ctx mgr us %.2f" % (1e6 * (t1 - t0) / n))
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt
    t0 = time.perf_counter()
    for i in range(n):
        dc.selection_mask(cfg.selection, 5)
        dc.selection_mask(cfg.hand_selection, 5, "hand selection")
    t1 = time.perf_counter()
    print("selection masks us %.2f" % (1e6 * (t1 - t0) / n))
    o = outs[0]
    t0 = time.perf_counter()
    for i in range(n):
        rt.FrameOutputsC(*[rt.ptr(o.get(k)) for k, _ in rt.FrameOutputsC._fields_])
    t1 = time.perf_counter()
    print("FrameOutputsC us %.2f" % (1e6 * (t1 - t0) / n))
    # the bare C call with prebuilt arguments
    import ctypes
    sh = ctypes.c_void_p(streams[0].cuda_stream)
    img0, kp0 = images[0:B], kps[0:B]
    fo = rt.FrameOutputsC(*[rt.ptr(outs[0].get(k)) for k, _ in rt.FrameOutputsC._fields_])
    bsel, _ = dc.selection_mask(cfg.selection, 5)
    hsel, _ = dc.selection_mask(cfg.hand_selection, 5, "hand selection")
    args = (ctx.h, rt.ptr(img0), B, 512, 512, rt.ptr(kp0), float(cfg.alpha), bsel, hsel, rt.PRECISIONS["bf16"], fo, sh)
    for _ in range(10):
        ctx.lib.fsb_frame_batch(*args)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        ctx.lib.fsb_frame_batch(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("bare fsb_frame_batch us/call %.1f (incl drain %.1f)" % (1e6 * (t1 - t0) / n, 1e6 * (t2 - t0) / n))
    t0 = time.perf_counter()
    for i in range(n):
        pipe.context()
    t1 = time.perf_counter()
    print("pipe.context() us %.2f" % (1e6 * (t1 - t0) / n))
    t0 = time.perf_counter()
    for i in range(n):
        images[0:B]; kps[0:B]
    t1 = time.perf_counter()
    print("2 slices us %.2f" % (1e6 * (t1 - t0) / n))
