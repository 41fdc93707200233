"""One-frame device path (the p50 graph) for an ncu launch list:
python tools/prof_b1.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    import bench
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr

    pipe, _ = bench.build_models("bf16")
    pipe.context().set_graphs(False)
    scenes = bench.make_scenes(pipe.decoder.template, bench.frame_seeds(0, 1))
    images = pr.render_scenes(scenes)
    kps = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    outs = pipe.allocate_outputs(1, tail=True)
    for _ in range(3):
        pipe.launch(images, kps, outs, pl.fast_config())
    torch.cuda.synchronize()
