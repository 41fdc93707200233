"""Where the host time of one Pipeline.run_smpl goes (the steps of
Pipeline._run_one timed separately): python tools/api_profile.py"""
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
    from paper_2603_15603_b200.numkit import check_finite

    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models("bf16")
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, 8))
    images = pr.render_scenes(scenes)
    host = [images[i].cpu().numpy() for i in range(8)]
    cfg = pl.fast_config()
    import ctypes

    from paper_2603_15603_b200 import runtime as rt

    lib = pipe.context().lib
    for i in range(10):
        pipe.run_smpl(host[i % 8], scenes[i % 8], cfg)
    T = {}

    def tick(name, t0):
        t1 = time.perf_counter()
        T.setdefault(name, []).append((t1 - t0) * 1e6)
        return t1

    for r in range(200):
        img, sc = host[r % 8], scenes[r % 8]
        t = time.perf_counter()
        t0 = t
        st = pipe._frame_state(512, 512, True)
        bad = ctypes.c_int(0)
        lib.fsb_stage_frame(img.ctypes.data, st["img_np"].ctypes.data, img.size, ctypes.byref(bad))
        t = tick("fsb_stage_frame (check + copy)", t)
        check_finite(img, "x")
        t = tick("numpy check_finite (ref)", t)
        np.copyto(st["img_np"], img)
        t = tick("numpy copyto (ref)", t)
        st["kp_np"][...] = sc.keypoints2d
        t = tick("copy to pinned", t)
        stream = torch.cuda.current_stream()
        pipe.launch(st["h_img"], st["h_kp"], st["out"], cfg)
        t = tick("launch (graph replay)", t)
        for k, hb in st["host"].items():
            hb.copy_(st["out"][k], non_blocking=True)
        t = tick("D2H enqueue", t)
        torch.cuda.current_stream().synchronize()
        t = tick("sync (device work)", t)
        pipe.context().check_finite("run")
        t = tick("nonfinite flag", t)
        tick("total", t0)
        t = time.perf_counter()
        pipe.run_smpl(img, sc, cfg)
        tick("run_smpl", t)
    for k, v in T.items():
        v.sort()
        print("%-24s p50 %8.1f us" % (k, v[len(v) // 2]))
