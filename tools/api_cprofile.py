"""cProfile of Pipeline.run_smpl (host side of the single-frame API):
python tools/api_cprofile.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import bench
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr

    pipe, (mhr, smpl, gt, dec, proj) = bench.build_models("bf16")
    scenes = bench.make_scenes(smpl, bench.frame_seeds(0, 8))
    images = pr.render_scenes(scenes)
    host = [images[i].cpu().numpy() for i in range(8)]
    cfg = pl.fast_config()
    for i in range(20):
        pipe.run_smpl(host[i % 8], scenes[i % 8], cfg)
    ts = []
    for i in range(300):
        t0 = time.perf_counter()
        pipe.run_smpl(host[i % 8], scenes[i % 8], cfg)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print("run_smpl p50 %.1f us" % (ts[150] * 1e6))
    pr_ = cProfile.Profile()
    pr_.enable()
    for i in range(300):
        pipe.run_smpl(host[i % 8], scenes[i % 8], cfg)
    pr_.disable()
    st = pstats.Stats(pr_)
    st.sort_stats("tottime").print_stats(25)
