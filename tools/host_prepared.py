"""Host cost of PreparedBatch.launch (one C call: graph lookup + launch)
round-robin over 16 streams, as bench.py's C2 loop issues them."""
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

    pipe, _ = bench.build_models("bf16")
    B, S = 32, 16
    scenes = bench.make_scenes(pipe.template, bench.frame_seeds(0, B))
    images = pr.render_scenes(scenes)
    kps = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).cuda()
    pipes = [pipe] + [pipe.fork() for _ in range(S - 1)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    pbs = []
    for p_ in pipes:
        p_.context().reserve(B)
        pbs.append(p_.prepare(images, kps, p_.allocate_outputs(B, tail=True), pl.fast_config()))
    for _ in range(3):
        for j in range(S):
            pbs[j].launch(streams[j])
    torch.cuda.synchronize()
    n = 100
    t0 = time.perf_counter()
    for _ in range(n):
        for j in range(S):
            pbs[j].launch(streams[j])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("host %.1f us per launch; device-bound time per batch %.1f us" % ((t1 - t0) / (n * S) * 1e6,
                                                                            (t2 - t0) / (n * S) * 1e6))
