"""Device time of the K3 decoder on body CTAs only, hand CTAs only and both,
of the encoder + K / V projection launch and of the decoders on projected
K / V (B frames, default 32, bf16, CUDA-graph replays): python tools/k3_split.py [B]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    import bench
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt

    pipe, _ = bench.build_models("bf16")
    ctx = pipe.context()
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    feats = torch.randn((B, 3, 64, 64), device="cuda")
    prompts = torch.rand((B, 8), device="cuda")
    params = torch.empty((B, 76), device="cuda")
    cam = torch.empty((B, 3), device="cuda")
    rots = torch.empty((B, 2, 3), device="cuda")
    merged = torch.empty((B, 76), device="cuda")
    bsel, _ = dc.selection_mask((0, 1, 2), 5)
    prec = rt.PRECISIONS["bf16"]
    hfeat = feats[:, 1:3].contiguous().reshape(2 * B, 64, 64)

    def body():
        ctx.check(ctx.lib.fsb_decode_body(ctx.h, rt.ptr(feats), B, 3, rt.ptr(prompts), bsel, rt.ptr(params),
                                          rt.ptr(cam), None, prec, ctx.stream))

    def hands():
        ctx.check(ctx.lib.fsb_decode_hands(ctx.h, rt.ptr(hfeat), 2 * B, 0, rt.ptr(rots), prec, ctx.stream))

    def both():
        ctx.check(ctx.lib.fsb_decode_frames(ctx.h, rt.ptr(feats), B, rt.ptr(prompts), bsel, 0, rt.ptr(params),
                                            rt.ptr(cam), rt.ptr(rots), rt.ptr(merged), prec, ctx.stream))

    crops = torch.rand((B, 3, 64, 64, 3), device="cuda")

    def enc():  # encoder + K / V projection (fsb_encode_frames)
        ctx.check(ctx.lib.fsb_encode_frames(ctx.h, rt.ptr(crops), B, rt.ptr(feats), prec, ctx.stream))

    # body / hands / both: the decode API on given features (K / V projection
    # + decoders); "decoders": the decoders alone on K / V projected by the
    # encoder launch (the frame path)
    for name, fn in (("body", body), ("hands", hands), ("both", both), ("encoder+kv", enc), ("decoders", both)):
        if name == "decoders":
            enc()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
                for _ in range(20):
                    fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(name, "%.1f us" % (e0.elapsed_time(e1) / 60 * 1e3))
