"""K1 on pinned host frames (the e2e path): bytes the kernel counts as read
from host memory (fsb_input_bytes) -- run under ncu with pcie__read_bytes /
syslts__d_sectors_fill_sysmem to show they cross PCIe:
    ncu --metrics pcie__read_bytes.sum,syslts__d_sectors_fill_sysmem.sum -k regex:k_crops_stream \
        python tools/pcie_proof.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    import bench
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr

    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models("bf16")
    pipe.context().set_graphs(False)
    B = 32
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, B))
    images = pr.render_scenes(scenes)
    h_img = images.cpu().pin_memory()
    h_kp = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).pin_memory()
    cfg = pl.fast_config()
    ctx = pipe.context()
    for i in range(3):
        ctx.input_bytes(reset=True)
        pipe.run_batch(h_img, h_kp, cfg)
        torch.cuda.synchronize()
        n = ctx.input_bytes(reset=True)
        print("batch %d: K1 read %d bytes of pinned host frames (%.1f%% of the %d frame bytes)"
              % (i, n, 100.0 * n / (h_img.numel() * 4), h_img.numel() * 4))
