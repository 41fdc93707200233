"""Launch each stage kernel of the frame -> SMPL path a few times on one batch
(no graphs) so ncu can capture them by name:

    ncu --set full --import-source on -k regex:k_decoders_tc -s 2 -c 1 \
        -o gpurun_out/dec python tools/prof_stages.py --precision bf16
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr

    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models(args.precision)
    ctx = pipe.context()
    ctx.set_graphs(False)
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, args.batch))
    images = pr.render_scenes(scenes)
    kps = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    outs = pipe.allocate_outputs(args.batch, tail=True)
    cfg = pl.fast_config()
    for _ in range(args.reps):
        pipe.launch(images, kps, outs, cfg)
    torch.cuda.synchronize()
    ctx.check_finite("prof")
    print("ok", ctx.launches())


if __name__ == "__main__":
    main()
