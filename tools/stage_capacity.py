"""Throughput capacity of each stage kernel when N copies run concurrently.

Each stage's C-ABI call is captured R times on each of N forked streams into
one CUDA graph (inputs shared, outputs overwritten: timing only), and the
graph is replayed between CUDA events.  us/batch at N=1 is the stage's
latency; at N=8 it is the device time one batch of that stage costs when the
GPU is kept full with it, i.e. its share of the SM budget.

    python tools/stage_capacity.py [--batch 32] [--reps 8]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--streams", default="1,2,4,8")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr
    from paper_2603_15603_b200 import runtime as rt

    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models("bf16")
    ctx = pipe.context()
    B = args.batch
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, B))
    img = pr.render_scenes(scenes)
    kp = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    outs = pipe.allocate_outputs(B, tail=True)
    cfg = pl.fast_config()
    pipe.launch(img, kp, outs, cfg)
    torch.cuda.synchronize()
    lib, h = ctx.lib, ctx.h
    prec = rt.PRECISIONS["bf16"]
    dev = img.device
    crops = torch.empty((B, 3, 64, 64, 3), dtype=torch.float32, device=dev)
    feats = torch.empty((B, 3, 64, 64), dtype=torch.float32, device=dev)
    bsel, _ = dc.selection_mask(cfg.selection, 5)
    cur = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731

    def k1():
        ctx.check(lib.fsb_boxes_crops(h, rt.ptr(img), B, 512, 512, rt.ptr(kp), 3.0, 64, rt.ptr(outs["boxes"]),
                                      rt.ptr(outs["prompt"]), rt.ptr(crops), None, cur()))

    def k2():
        ctx.check(lib.fsb_encode(h, rt.ptr(crops), 3 * B, rt.ptr(feats), prec, cur()))

    def k3():
        ctx.check(lib.fsb_decode_frames(h, rt.ptr(feats), B, rt.ptr(outs["prompt"]), bsel, 0,
                                        rt.ptr(outs["body_params"]), rt.ptr(outs["body_cam"]),
                                        rt.ptr(outs["hand_rots"]), rt.ptr(outs["merged"]), prec, cur()))

    def k4a():
        ctx.check(lib.fsb_skin(h, 0, rt.ptr(outs["merged"]), B, rt.ptr(outs["v_mhr"]), cur()))

    def k4b():
        ctx.check(lib.fsb_skin_project(h, rt.ptr(outs["merged"]), B, None, rt.ptr(outs["theta"]),
                                       rt.ptr(outs["j_smpl"]), None, prec, cur()))

    stages = [("k1", k1), ("k2", k2), ("k3", k3), ("k4_lbs", k4a), ("k4_proj", k4b)]
    ctx.set_graphs(False)
    for _, fn in stages:
        fn()
    torch.cuda.synchronize()
    res = {}
    for name, fn in stages:
        row = {}
        for n in [int(x) for x in args.streams.split(",")]:
            side = [torch.cuda.Stream(device=dev) for _ in range(n)]
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap, capture_error_mode="relaxed"):
                    for s in side:
                        s.wait_stream(cap)
                        with torch.cuda.stream(s):
                            for _ in range(args.reps):
                                fn()
                    for s in side:
                        cap.wait_stream(s)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            row[n] = round(1e3 * e0.elapsed_time(e1) / (5 * n * args.reps), 2)
        res[name] = row
        print(name, "us/batch by concurrent streams:", row, flush=True)
    tot = {n: round(sum(r[n] for r in res.values()), 2) for n in res["k1"]}
    print("sum", tot)


if __name__ == "__main__":
    main()
