"""Host cost of one Pipeline.launch (graph replay through the C ABI) vs the
device time per batch: python tools/host_rate.py"""
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

    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models("bf16")
    B = 32
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, 64))
    images = pr.render_scenes(scenes)
    kps = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    outs = pipe.allocate_outputs(B, tail=True)
    cfg = pl.fast_config()
    for i in range(10):
        pipe.launch(images[:B], kps[:B], outs, cfg)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for i in range(n):
        pipe.launch(images[:B], kps[:B], outs, cfg)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("host %.1f us per launch; wall incl. drain %.1f us per batch" % ((t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6))
