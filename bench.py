#!/usr/bin/env python
"""Benchmark of the frame -> SMPL hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B]
                    [--precision fp32|bf16] [--impl ours|reference]

One step = one batch of B synthetic 512x512 frames per GPU through the whole
path (K1 boxes+crops -> K2 encoder -> K3 decoders+merge -> K4 MHR LBS,
bridge, projector, SMPL FK), replayed from a CUDA graph; with N > 1 every
rank runs its own frames (weak scaling, one process per GPU under torchrun)
and the per-step SMPL outputs (theta + joints) are all-gathered over NCCL,
the path's only collective.  Rank 0 prints one JSON line.

`value` is device-timed throughput with inputs resident in HBM; `e2e` is
the same metric through Pipeline.run_batch with pinned host frames copied
in and SMPL results copied out every step.  `--impl reference` times the
CPU restatement of the reference (oracle/) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1/2/4/8 B200 and p50 frame latency (crop→encode→SMPL)"
UNIT = "frames/s"

# algorithmic work per unit; see DESIGN.md
FLOP_ENC_FRAME = 48_758_784
FLOP_DEC_FRAME = 57_853_440
BYTES_K1_FRAME = 737_280 + 304
BYTES_LBS_MESH = 221_268 + 304 + 1_056
FLOP_MLP_MESH = 4_909_056
# C4 (ViT-L-sized encoder, S=384, p=16, T=576, D=1024, 24 layers), per crop:
# 2*T*(3p^2)*D + L*(24*T*D^2 + 4*T^2*D)
FLOP_C4_CROP = 2 * 576 * 768 * 1024 + 24 * (24 * 576 * 1024 ** 2 + 4 * 576 ** 2 * 1024)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--batch", type=int, default=32, help="frames per GPU per step (C2: 32)")
    ap.add_argument("--bank", type=int, default=256, help="distinct frames per GPU cycled through")
    ap.add_argument("--precision", default="bf16", choices=("fp32", "bf16"))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--streams", type=int, default=16,
                    help="in-flight batches per GPU: independent pipeline contexts on their own streams")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 LBS + projector microbench")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 ViT-L-sized encoder microbench")
    ap.add_argument("--no-fit", action="store_true", help="skip the iterative-fit conversion microbench")
    ap.add_argument("--stream-frames", type=int, default=8192,
                    help="C5: frames of the synthetic video stream sharded across the ranks (0: skip)")
    ap.add_argument("--c4-crops", type=int, default=768, help="C4: 3 crops x 256 frames")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing


def dist_setup(torch, want):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return dist, rank, ws, local
    return None, 0, 1, 0


def frame_seeds(rank, bank):
    """Rank r's frames are scenes 5000 + r * bank + i (disjoint per rank)."""
    return [5000 + rank * bank + i for i in range(bank)]


def shard_bounds(n_frames, rank, world):
    """Contiguous shard of a frame stream: [r*n/G, (r+1)*n/G)."""
    return rank * n_frames // world, (rank + 1) * n_frames // world


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)

_REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            mx = m
            if s > 0.5 * m:  # under load
                sm.append(s)
            for name, val in zip(_REASONS, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(self.lines)}


# ---------------------------------------------------------------------------
# models and synthetic frames


def build_models(precision):
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = synth.make_toy_models(0, 18439, 6890)
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    proj = pj.init_projector(pj.make_subsample(6890, 1500), (512, 256), seed=0)
    return pl.Pipeline(dec, mhr=mhr, bmap=gt, projector=proj, precision=precision), (mhr, smpl, gt, dec, proj)


def extra_pipelines(pipe, n, precision):
    """n more pipeline instances over the same models, each with its own
    fsb context (weights, workspace, CUDA graphs): one per in-flight batch
    (pipelines are not shared between concurrent users)."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl

    out = []
    for _ in range(n):
        d = dc.Decoder(pipe.decoder.template, pipe.decoder.config, seed=40)
        out.append(pl.Pipeline(d, mhr=pipe.mhr, bmap=pipe.bmap, projector=pipe.projector, precision=precision))
    return out


def make_scenes(smpl, seeds):
    from paper_2603_15603_b200 import synth

    return [synth.random_scene(np.random.default_rng(s), smpl, (512, 512)) for s in seeds]


# ---------------------------------------------------------------------------
# CPU oracle (baseline / reference arm)


def _cpu_worker(args):
    frames, kps, deadline_s, min_frames, warm = args
    os.environ["OMP_NUM_THREADS"] = "1"
    import oracle as orc
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = synth.make_toy_models(0, 18439, 6890)
    cfg = dc.DecoderConfig()
    w = synth.decoder_weights(cfg, 40)
    p = pj.init_projector(pj.make_subsample(6890, 1500), (512, 256), seed=0)
    pw = dict(w1=p.w1, b1=p.b1, w2=p.w2, b2=p.b2, w3=p.w3, b3=p.b3, subsample=p.subsample, mask=p.mask)
    for i in range(max(1, warm)):  # untimed warm-up frames
        orc.frame_to_smpl(frames[i % len(frames)], kps[i % len(frames)], w, cfg, mhr, smpl, gt, pw)
    done, lat = 0, []
    t0 = time.perf_counter()
    while done < min_frames or (time.perf_counter() - t0) < deadline_s:
        i = done % len(frames)
        a = time.perf_counter()
        orc.frame_to_smpl(frames[i], kps[i], w, cfg, mhr, smpl, gt, pw)
        lat.append(time.perf_counter() - a)
        done += 1
    return done, time.perf_counter() - t0, lat


def cpu_oracle_run(frames, kps, seconds, min_frames=1, workers=None, warm=1):
    """Oracle frames/s on `workers` host processes (spawn), disjoint frames."""
    n = workers or len(os.sched_getaffinity(0))
    n = max(1, min(n, 64))
    chunks = [(frames[i::n] if len(frames[i::n]) else frames[:1], kps[i::n] if len(kps[i::n]) else kps[:1],
               seconds, min_frames, warm) for i in range(n)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(n) as pool:
        res = pool.map(_cpu_worker, chunks)
    frames_done = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    lat = [x for r in res for x in r[2]]
    return frames_done / wall, n, frames_done, statistics.median(lat) * 1e3


def reference_arm(args):
    """--impl reference: the oracle port on all host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_2603_15603_b200 import synth

    _, smpl, _ = synth.make_toy_models(0, 18439, 6890)
    n = len(os.sched_getaffinity(0))
    scenes = make_scenes(smpl, frame_seeds(0, max(8, min(n, 32))))
    frames = np.stack([synth.render_scene(s, smpl) for s in scenes])
    kps = np.stack([s.keypoints2d for s in scenes])
    # one step = one frame on every host worker; W untimed warm-up frames per
    # worker, then K timed frames per worker (capped so the run stays short)
    warm = max(0, args.warmup)
    steps = max(1, min(args.steps, 600))
    fps, cores, done, p50 = cpu_oracle_run(frames, kps, 0.0, min_frames=steps, workers=n, warm=warm)
    per_step_s = n / fps
    line = {"impl": "reference", "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": ws, "steps": steps,
            "warmup": warm, "ms_per_step": per_step_s * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 frame->SMPL, 512x512 frames, default encoder/decoders, full-size "
                                   "MHR 18439 / SMPL 6890 tail (CPU oracle restatement of the reference)",
                       "frames_per_step": n},
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": "%d timed frames on %d host processes (one frame per process per step, %d "
                                       "steps), p50 %.1f ms/frame" % (done, cores, steps, p50)},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "p50_frame_latency_ms": p50}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the GPU arm


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch

    dist, rank, world, local = dist_setup(torch, args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2603_15603_b200 import priors as pr

    pipe, (mhr, smpl, gt, dec, proj) = build_models(args.precision)
    ctx = pipe.context()
    B, bank = args.batch, max(args.bank, args.batch)
    bank -= bank % B
    ctx.reserve(max(B, 1))

    scenes = make_scenes(smpl, frame_seeds(rank, bank))
    images = pr.render_scenes(scenes)                      # (bank, 512, 512, 3) resident in HBM
    kps = torch.from_numpy(np.stack([s.keypoints2d for s in scenes])).to(dev)
    nslot = bank // B
    S = max(1, args.streams)
    pipes = [pipe] + extra_pipelines(pipe, S - 1, args.precision)
    for p_ in pipes[1:]:
        p_.context().reserve(max(B, 1))
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream(device=dev) for _ in range(S - 1)]
    outs_s = [p_.allocate_outputs(B, tail=True) for p_ in pipes]
    outs = outs_s[0]
    from paper_2603_15603_b200 import pipeline as pl

    cfg = pl.fast_config()
    gathered = None
    if dist is not None:
        gathered = [torch.empty((world * B, 76 + 66), dtype=torch.float32, device=dev) for _ in range(S)]
        packed = [torch.empty((B, 76 + 66), dtype=torch.float32, device=dev) for _ in range(S)]

    def step(i):
        j, s = i % S, i % nslot
        with torch.cuda.stream(streams[j]):
            pipes[j].launch(images[s * B:(s + 1) * B], kps[s * B:(s + 1) * B], outs_s[j], cfg)
            if dist is not None:
                packed[j][:, :76].copy_(outs_s[j]["theta"])
                packed[j][:, 76:].copy_(outs_s[j]["j_smpl"].reshape(B, 66))
                dist.all_gather_into_tensor(gathered[j], packed[j])

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (captures one graph per input slot and stream)
    for i in range(max(args.warmup, 3, nslot * S)):
        step(i)
    for p_ in pipes:
        p_.context().check_finite("bench warm-up")
    barrier()
    launches0 = sum(p_.context().launches() for p_ in pipes)
    st = streams[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    joins = [torch.cuda.Event() for _ in range(S)]
    with ClockSampler(local) as clk:
        barrier()
        e0.record(st)
        for q in streams[1:]:
            q.wait_event(e0)
        for i in range(args.steps):
            step(i)
        for j in range(1, S):
            joins[j].record(streams[j])
            st.wait_event(joins[j])
        e1.record(st)
        barrier()
    launches = sum(p_.context().launches() for p_ in pipes) - launches0
    ms = e0.elapsed_time(e1)
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    frames_total = world * B * args.steps
    value = frames_total / (ms / 1e3)
    for p_ in pipes:
        p_.context().check_finite("bench")
    # the concurrent batches computed what one pipeline computes alone
    verified = verify_streams(torch, pipes, outs_s, images, kps, cfg, B, args.steps, nslot, S)

    # -- C5: an 8192-frame stream sharded across the ranks, one NCCL gather ----
    c5 = None if args.stream_frames <= 0 else stream_run(torch, pipes, streams, images, kps, cfg, B, dist, world,
                                                          rank, args.stream_frames)

    # -- per-stage attribution (graphs off, CUDA events between stages) -------
    stage_sat = {}
    stage_ms = attribute_stages(torch, pipe, ctx, images[:B], kps[:B], outs, cfg, reps=20, saturated=16,
                                saturated_out=stage_sat)
    stage_sat["sum"] = round(sum(stage_sat.values()), 2)

    # -- p50 single-frame latency (B = 1 graph replay) -------------------------
    lat = frame_latency(torch, pipe, images, kps, cfg, reps=200)

    # -- end-to-end through the public API with host buffers -------------------
    e2e = None if args.no_e2e else end_to_end(torch, pipes, images, kps, cfg, B, args.steps, args.warmup, dist,
                                              world)
    e2e_copy = None if args.no_e2e else end_to_end_full_copy(torch, pipe, images, kps, cfg, B, args.steps,
                                                             args.warmup, dist, world)

    # -- C3 microbench: LBS + projector on 4096 full-size meshes ---------------
    c3 = None if args.no_c3 else c3_microbench(torch, pipe, ctx, meshes=4096, reps=10)

    # -- conversion: iterative fit (the paper's slow baseline) vs projector ----
    conv = None if args.no_fit else fit_microbench(torch, pipe, meshes=148, steps=300,
                                                   projector_meshes_per_s=(c3 or {}).get("meshes_per_s"))

    # -- C4 microbench: ViT-L-sized encoder, 3 crops x 256 frames --------------
    c4 = None if args.no_c4 else c4_microbench(torch, crops=args.c4_crops, reps=3)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    roof = roofline(stage_ms, B)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        n_host = min(len(scenes), 64)
        fr = images[:n_host].cpu().numpy()
        kk = kps[:n_host].cpu().numpy()
        fps, cores, done, p50c = cpu_oracle_run(fr, kk, args.cpu_seconds)
        cpu = {"value": fps, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": "%d frames (C2 frame->SMPL, full-size tail) on %d host processes over ~%.0f s; "
                         "p50 %.1f ms/frame single process" % (done, cores, args.cpu_seconds, p50c)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "bf16", "data": "synthetic",
        "config": {"workload": "C2: %d synthetic 512x512 frames per GPU per step, body + 2 hand crops -> "
                               "encoder -> pruned decoders -> MHR LBS (18439 v) -> projector -> SMPL FK" % B,
                   "frames_per_gpu_per_step": B, "global_batch": B * world,
                   "parallelism": "dp%d (frame sharding, NCCL all-gather of SMPL outputs)" % world
                   if world > 1 else "single GPU",
                   "l2": "inputs cycle through a %d-frame bank (%.0f MB in HBM) > 126 MB L2" %
                         (bank, bank * 512 * 512 * 12 / 1e6),
                   "precision": args.precision, "graphs": True,
                   "in_flight_batches": S, "concurrent_outputs_match_single_stream": verified},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_full_frame_copy": e2e_copy,
        "gpu_launches": launches,
        "clocks": clk.summary(), "p50_frame_latency_ms": lat["p50_ms"], "frame_latency": lat,
        "stage_ms": stage_ms,
        "stage_saturated_us_per_batch": stage_sat,  # 16 concurrent copies of each stage alone
        "c3": c3, "c4": c4, "c5": c5, "conversion": conv,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def c3_microbench(torch, pipe, ctx, meshes, reps):
    """C3: MHR LBS of `meshes` full-size meshes (18,439 v) plus
    the MHR -> SMPL projector and SMPL FK, poses from rng(3) as the
    acceptance suite draws them.  LBS is timed alone for its HBM roofline
    (222,628 algorithmic bytes per mesh: V_mhr written + pose/transforms)."""
    from paper_2603_15603_b200 import runtime as rt

    rng = np.random.default_rng(3)
    p = np.zeros((meshes, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(meshes, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(meshes, 10))
    p[:, 51:54] = 0.0
    p[:, 63:66] = 0.0
    dev = torch.device("cuda", torch.cuda.current_device())
    poses = torch.from_numpy(p).to(dev)
    nv = pipe.mhr.num_vertices
    v = torch.empty((meshes, nv, 3), dtype=torch.float32, device=dev)
    th = torch.empty((meshes, 76), dtype=torch.float32, device=dev)
    j = torch.empty((meshes, 22, 3), dtype=torch.float32, device=dev)
    ctx.reserve(meshes)
    prec = rt.PRECISIONS[pipe.precision]
    st = torch.cuda.current_stream()

    def full():
        ctx.check(ctx.lib.fsb_skin_project(ctx.h, rt.ptr(poses), meshes, rt.ptr(v), rt.ptr(th), rt.ptr(j), None, prec,
                                           ctx.stream))

    def lbs():
        ctx.check(ctx.lib.fsb_skin(ctx.h, 0, rt.ptr(poses), meshes, rt.ptr(v), ctx.stream))

    out = {}
    for name, fn in (("full", full), ("lbs", lbs)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    ctx.check_finite("c3")
    peak = 6550.7
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    lbs_gbs = meshes * BYTES_LBS_MESH / (out["lbs"] / 1e3) / 1e9
    return {"workload": "C3: %d full-size meshes (MHR 18439 v) LBS + projector + SMPL FK, %s" % (meshes, pipe.precision),
            "meshes_per_s": meshes / (out["full"] / 1e3), "ms_full": out["full"], "ms_lbs_fk": out["lbs"],
            "lbs_achieved_gbs": lbs_gbs, "lbs_frac_of_hbm": lbs_gbs / peak,
            "lbs_algorithmic_bytes": meshes * BYTES_LBS_MESH}


def fit_microbench(torch, pipe, meshes, steps, projector_meshes_per_s=None):
    """MHR -> SMPL conversion two ways on full-size meshes (PAPER.md:500-504's
    comparison): projection.fit_batch (`steps` Adam iterations per mesh,
    projection.py:321-370, one CTA per mesh on the GPU) against the
    feed-forward projector (the C3 number)."""
    from paper_2603_15603_b200 import bodymodel as bm
    from paper_2603_15603_b200 import projection as pj

    rng = np.random.default_rng(3)
    p = np.zeros((meshes, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(meshes, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(meshes, 10))
    p[:, 51:54] = 0.0
    p[:, 63:66] = 0.0
    dev = torch.device("cuda", torch.cuda.current_device())
    v = bm.skin_batch(pipe.mhr, torch.from_numpy(p).to(dev))
    pj.fit_batch(v[:2], pipe.bmap, pipe.decoder.template, pj.FitConfig(steps=3))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = pj.fit_batch(v, pipe.bmap, pipe.decoder.template, pj.FitConfig(steps=steps))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out = {"workload": "fit_batch: %d full-size MHR meshes -> SMPL, %d Adam steps each (GPU)" % (meshes, steps),
           "ms": ms, "fit_meshes_per_s": meshes / (ms / 1e3), "mean_vertex_gap": float(res.vertex_error.mean())}
    if projector_meshes_per_s:
        out["projector_meshes_per_s"] = projector_meshes_per_s
        out["projector_over_fit"] = projector_meshes_per_s / out["fit_meshes_per_s"]
    return out


def c4_microbench(torch, crops, reps, layers=24):
    """C4: Decoder.encode (decoder.py:231-260) at ViT-L size,
    DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16,
    enc_layers=24), on `crops` U[0,1) crops (768 = 3 crops x 256 frames),
    bf16 operands with fp32 accumulation on the tcgen05 path.  Tensor-bound:
    FLOP_C4_CROP algorithmic FLOPs per crop, against the sustained bf16 peak
    (a ~0.2 s launch sequence under the power cap)."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt
    from paper_2603_15603_b200 import synth

    cfg = dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16, enc_layers=layers, body_layers=1,
                           hand_layers=1)
    ctx = rt.Context()
    ctx.load_decoder(cfg, synth.decoder_weights(cfg, 40, encoder_only=True))
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    x = torch.rand((crops, 384, 384, 3), generator=g, dtype=torch.float32, device=dev)
    out = torch.empty((crops, 576, 1024), dtype=torch.float32, device=dev)
    prec = rt.PRECISIONS["bf16"]

    def run():
        ctx.check(ctx.lib.fsb_encode(ctx.h, rt.ptr(x), crops, rt.ptr(out), prec, ctx.stream), "c4 encode")

    run()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    ctx.check_finite("c4")
    ms = e0.elapsed_time(e1) / reps
    peak, src = 1396.7, "fallback"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak, src = float(json.load(fh)["bf16_tflops_sustained"]), "measured sustained"
    except (OSError, KeyError, ValueError):
        pass
    tf = crops * FLOP_C4_CROP / (ms / 1e3) / 1e12
    del ctx
    return {"workload": "C4: ViT-L-sized encoder (S=384, p=16, T=576, D=1024, 16 heads, %d layers) on %d crops "
                        "(3 crops x %d frames), bf16 tcgen05" % (layers, crops, crops // 3),
            "ms_per_batch": ms, "crops_per_s": crops / (ms / 1e3), "frames_per_s": crops / 3 / (ms / 1e3),
            "achieved_tflops": tf, "peak_tflops": peak, "peak_source": src, "frac": tf / peak,
            "algorithmic_flop_per_batch": crops * FLOP_C4_CROP}


def attribute_stages(torch, pipe, ctx, img, kp, outs, cfg, reps, saturated=None, saturated_out=None):
    """Average device time of each stage kernel on one batch.  Each stage's
    launches are captured `reps` times into its own CUDA graph and the graph
    is replayed between CUDA events, so the numbers are device time, not the
    host's ctypes launch rate."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt

    B = img.shape[0]
    lib, h = ctx.lib, ctx.h
    prec = rt.PRECISIONS[pipe.precision]
    dev = img.device
    crops = torch.empty((B, 3, 64, 64, 3), dtype=torch.float32, device=dev)
    feats = torch.empty((B, 3, 64, 64), dtype=torch.float32, device=dev)
    bsel, _ = dc.selection_mask(cfg.selection, 5)

    def k1():
        ctx.check(lib.fsb_boxes_crops(h, rt.ptr(img), B, 512, 512, rt.ptr(kp), 3.0, 64, rt.ptr(outs["boxes"]),
                                      rt.ptr(outs["prompt"]), rt.ptr(crops), None, ctx.stream))

    def k2():
        ctx.check(lib.fsb_encode(h, rt.ptr(crops), 3 * B, rt.ptr(feats), prec, ctx.stream))

    def k3():
        ctx.check(lib.fsb_decode_frames(h, rt.ptr(feats), B, rt.ptr(outs["prompt"]), bsel, 0,
                                        rt.ptr(outs["body_params"]), rt.ptr(outs["body_cam"]),
                                        rt.ptr(outs["hand_rots"]), rt.ptr(outs["merged"]), prec, ctx.stream))

    def k4a():
        ctx.check(lib.fsb_skin(h, 0, rt.ptr(outs["merged"]), B, rt.ptr(outs["v_mhr"]), ctx.stream))

    def k4b():  # projector input bridged from V_mhr + the MLP, as in the frame path
        ctx.check(lib.fsb_project_vertices(h, rt.ptr(outs["v_mhr"]), B, pipe.mhr.num_vertices, rt.ptr(outs["theta"]),
                                           prec, ctx.stream))

    stages = [("k1_boxes_crops", k1), ("k2_encoder", k2), ("k3_decoders", k3), ("k4_fk_lbs", k4a),
              ("k4_proj_mlp", k4b)]
    for _, fn in stages:  # eager warm-up (workspace allocation happens here)
        fn()
    torch.cuda.synchronize()
    out = {}
    side = torch.cuda.Stream(device=dev)
    for name, fn in stages:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side, capture_error_mode="relaxed"):
                for _ in range(reps):
                    fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = float(e0.elapsed_time(e1) / (3 * reps))
    if saturated is not None:
        # the same stages with `saturated` concurrent copies (forked streams in
        # one graph): device time one batch of the stage costs when the GPU is
        # kept full with it -- its share of the SM budget the pipeline runs on
        n = saturated
        for name, fn in stages:
            branches = [torch.cuda.Stream(device=dev) for _ in range(n)]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side, capture_error_mode="relaxed"):
                    for q in branches:
                        q.wait_stream(side)
                        with torch.cuda.stream(q):
                            for _ in range(4):
                                fn()
                    for q in branches:
                        side.wait_stream(q)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            saturated_out[name] = round(float(1e3 * e0.elapsed_time(e1) / (3 * 4 * n)), 2)
    return out


def roofline(stage_ms, B):
    """Roofline of the dominant stage kernel against MEASURED_PEAKS.json."""
    peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        peaks = {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]), "src": "measured"}
    except (OSError, KeyError, ValueError):
        pass
    work = {  # name -> (bound, algorithmic units per launch, unit)
        "k1_boxes_crops": ("hbm", BYTES_K1_FRAME * B),
        "k2_encoder": ("tensor", FLOP_ENC_FRAME * B),
        "k3_decoders": ("tensor", FLOP_DEC_FRAME * B),
        "k4_fk_lbs": ("hbm", BYTES_LBS_MESH * B),
        "k4_proj_mlp": ("tensor", FLOP_MLP_MESH * B),
    }
    dom = max(stage_ms, key=stage_ms.get)
    bound, amount = work[dom]
    sec = stage_ms[dom] / 1e3
    if bound == "hbm":
        achieved, peak, unit = amount / sec / 1e9, peaks["hbm_gbs"], "GB/s"
    else:
        achieved, peak, unit = amount / sec / 1e12, peaks["bf16_tflops"], "TFLOP/s"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        if dom in tr:
            traffic = tr[dom].get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    return {"kernel": dom, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": traffic, "peak_source": peaks["src"],
            "share_of_step": stage_ms[dom] / sum(stage_ms.values()),
            "algorithmic_per_launch": amount, "launch_ms": stage_ms[dom]}


def frame_latency(torch, pipe, images, kps, cfg, reps):
    """p50 latency of one frame through the whole path (graph replay)."""
    outs = pipe.allocate_outputs(1, tail=True)
    st = torch.cuda.current_stream()
    for i in range(5):
        pipe.launch(images[i:i + 1], kps[i:i + 1], outs, cfg)
    torch.cuda.synchronize()
    ts = []
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        pipe.launch(images[0:1], kps[0:1], outs, cfg)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return {"p50_ms": ts[len(ts) // 2], "p95_ms": ts[int(len(ts) * 0.95)], "reps": reps, "batch": 1}


def stream_run(torch, pipes, streams, images, kps, cfg, B, dist, world, rank, total):
    """C5: a stream of `total` synthetic frames, rank r taking
    the contiguous block [r*total/G, (r+1)*total/G) (frame i is bank frame
    i % bank), batches of B spread over the in-flight pipelines, the SMPL
    outputs (theta + joints, 142 floats per frame) collected per rank and
    all-gathered over NCCL once at the end.  Strong scaling: frames/s of the
    whole stream, first frame to gathered result, max over ranks."""
    lo, hi = shard_bounds(total, rank, world)
    n = hi - lo
    dev = images.device
    bank = images.shape[0]
    res = torch.empty((max(n, 1), 142), dtype=torch.float32, device=dev)
    S = len(pipes)
    outs = [p_.allocate_outputs(B, tail=True) for p_ in pipes]
    gathered = torch.empty((world * max(n, 1), 142), dtype=torch.float32, device=dev) if dist is not None else None

    def batch(k, f0, nb):
        j = k % S
        with torch.cuda.stream(streams[j]):
            s0 = f0 % bank
            if s0 + nb <= bank:
                img, kp = images[s0:s0 + nb], kps[s0:s0 + nb]
            else:
                idx = torch.arange(f0, f0 + nb, device=dev) % bank
                img, kp = images[idx], kps[idx]
            o = outs[j] if nb == B else pipes[j].allocate_outputs(nb, tail=True)
            pipes[j].launch(img, kp, o, cfg)
            r = f0 - lo
            res[r:r + nb, :76].copy_(o["theta"])
            res[r:r + nb, 76:].copy_(o["j_smpl"].reshape(nb, 66))

    # warm-up: every (pipeline, input slot) pair the timed pass will use
    # gets its CUDA graph captured first -- the input ring repeats with period
    # lcm(pipelines, bank / B) batches, as a deployment's ring of frame buffers would
    import math

    nslot = max(1, bank // B)
    period = S * nslot // math.gcd(S, nslot)
    for k in range(min(period, max(1, (n + B - 1) // B))):
        f0 = lo + k * B
        batch(k, f0, min(B, hi - f0))
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    st = streams[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for q in streams[1:]:
        q.wait_event(e0)
    k = 0
    for f0 in range(lo, hi, B):
        batch(k, f0, min(B, hi - f0))
        k += 1
    for q in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(q)
        st.wait_event(ev)
    if dist is not None:
        with torch.cuda.stream(st):
            dist.all_gather_into_tensor(gathered, res)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"workload": "C5: %d-frame synthetic stream sharded over %d GPU(s) (%d frames on this rank), batches of %d "
                        "on %d in-flight pipelines, one all-gather of the SMPL outputs (theta + joints)"
                        % (total, world, n, B, S),
            "ms": ms, "frames_per_s": total / (ms / 1e3), "scaling": "strong",
            "gathered_bytes_per_rank": int(n * 142 * 4)}


def verify_streams(torch, pipes, outs_s, images, kps, cfg, B, steps, nslot, S):
    """Re-run the last step of every stream alone on pipeline 0 and compare
    bit for bit with what the concurrent run produced."""
    torch.cuda.synchronize()
    ref = pipes[0].allocate_outputs(B, tail=True)
    ok = True
    for j in range(S):
        last = max(i for i in range(steps) if i % S == j) if steps > j else None
        if last is None:
            continue
        s = last % nslot
        got = {k: outs_s[j][k].clone() for k in ("merged", "theta", "j_smpl")}
        pipes[0].launch(images[s * B:(s + 1) * B], kps[s * B:(s + 1) * B], ref, cfg)
        torch.cuda.synchronize()
        ok = ok and all(torch.equal(got[k], ref[k]) for k in got)
    return bool(ok)


E2E_STREAMS = int(os.environ.get("FSB_E2E_STREAMS", "6"))


def end_to_end(torch, pipes, images, kps, cfg, B, steps, warmup, dist, world):
    """Pipeline.run_batch on frames that live in pinned host memory (the
    reference's images are host float32 arrays).  K1 reads each frame in
    place over PCIe -- only the crop footprints (the rows and x-spans the
    three crops tap) cross the bus -- so there is no separate whole-frame
    H2D copy; steps rotate over E2E_STREAMS streams so one batch's gather
    overlaps the others' compute.  Every step ends with a D2H read
    of merged/theta/j_smpl into pinned host buffers.  h2d_bytes_per_step is
    counted on the device by K1 (fsb_input_bytes) plus the keypoints.  Each
    stream drives its own pipeline context (own workspace and graphs)."""
    NS = E2E_STREAMS
    pipes = list(pipes[:NS])
    if len(pipes) < NS:
        pipes += extra_pipelines(pipes[0], NS - len(pipes), pipes[0].precision)
    ctxs = [p_.context() for p_ in pipes]
    dev = images.device
    nhost = min(images.shape[0], 4 * B)
    h_img = images[:nhost].cpu().pin_memory()
    h_kp = kps[:nhost].cpu().pin_memory()
    nslot = nhost // B
    streams = [torch.cuda.Stream(device=dev) for _ in range(NS)]
    outs = [pipes[j].allocate_outputs(B, tail=True) for j in range(NS)]
    h_out = [{k: torch.empty(outs[0][k].shape, dtype=torch.float32).pin_memory()
              for k in ("merged", "theta", "j_smpl")} for _ in range(NS)]

    def run(i):
        j, s = i % NS, i % nslot
        with torch.cuda.stream(streams[j]):
            pipes[j].run_batch(h_img[s * B:(s + 1) * B], h_kp[s * B:(s + 1) * B], cfg, outputs=outs[j], sync=False)
            for k in ("merged", "theta", "j_smpl"):
                h_out[j][k].copy_(outs[j][k], non_blocking=True)

    for i in range(max(warmup, NS * nslot)):
        run(i)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    for c in ctxs:
        c.input_bytes(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tail = [torch.cuda.Event() for _ in range(NS)]
    e0.record(streams[0])
    for q in streams[1:]:
        q.wait_event(e0)
    for i in range(steps):
        run(i)
    for j in range(NS):
        tail[j].record(streams[j])
        streams[0].wait_event(tail[j])
    e1.record(streams[0])
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    frame_bytes = sum(c.input_bytes(reset=True) for c in ctxs)
    # the host-side results of the last step of each stream equal a fresh
    # device-frame run of the same frames
    ok = True
    ref = pipes[0].allocate_outputs(B, tail=True)
    for j in range(min(NS, steps)):
        last = max(i for i in range(steps) if i % NS == j)
        s = last % nslot
        pipes[0].launch(images[s * B:(s + 1) * B], kps[s * B:(s + 1) * B], ref, cfg)
        torch.cuda.synchronize()
        ok = ok and all(torch.equal(h_out[j][k], ref[k].cpu()) for k in ("merged", "theta", "j_smpl"))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    h2d_b = frame_bytes // steps + B * 44 * 4
    d2h_b = B * (76 + 76 + 66) * 4
    full = B * (images[0].numel() + 44) * 4
    return {"value": world * B * steps / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d_b,
            "d2h_bytes_per_step": d2h_b, "ms_per_step": ms / steps,
            "api": "Pipeline.run_batch on pinned host frames (K1 gathers the crop footprints over PCIe in "
                   "place; %d streams)" % NS,
            "h2d_fraction_of_frames": h2d_b / full, "outputs_verified": bool(ok)}


def end_to_end_full_copy(torch, pipe, images, kps, cfg, B, steps, warmup, dist, world):
    """Variant kept for comparison: whole frames copied H2D (copy stream,
    double-buffered) before Pipeline.run_batch on device frames."""
    dev = images.device
    nhost = min(images.shape[0], 4 * B)
    h_img = images[:nhost].cpu().pin_memory()
    h_kp = kps[:nhost].cpu().pin_memory()
    nslot = nhost // B
    d_img = [torch.empty((B,) + tuple(images.shape[1:]), dtype=torch.float32, device=dev) for _ in range(2)]
    d_kp = [torch.empty((B, 22, 2), dtype=torch.float32, device=dev) for _ in range(2)]
    outs = [pipe.allocate_outputs(B, tail=True) for _ in range(2)]
    h_out = [{k: torch.empty(outs[0][k].shape, dtype=torch.float32).pin_memory()
              for k in ("merged", "theta", "j_smpl")} for _ in range(2)]
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    for d in done:
        d.record(comp)

    def h2d(i):
        j = i % 2
        s = i % nslot
        with torch.cuda.stream(copy):
            copy.wait_event(done[j])
            d_img[j].copy_(h_img[s * B:(s + 1) * B], non_blocking=True)
            d_kp[j].copy_(h_kp[s * B:(s + 1) * B], non_blocking=True)
            ready[j].record(copy)

    def run(i):
        j = i % 2
        comp.wait_event(ready[j])
        pipe.run_batch(d_img[j], d_kp[j], cfg, outputs=outs[j], sync=False)
        for k in ("merged", "theta", "j_smpl"):
            h_out[j][k].copy_(outs[j][k], non_blocking=True)
        done[j].record(comp)

    total = warmup + steps
    h2d(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(total):
        if i == warmup:
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            e0.record(comp)
        if i + 1 < total:
            h2d(i + 1)
        run(i)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    h2d_b = B * (images[0].numel() + 44) * 4
    d2h_b = B * (76 + 76 + 66) * 4
    return {"value": world * B * steps / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d_b,
            "d2h_bytes_per_step": d2h_b, "ms_per_step": ms / steps,
            "api": "Pipeline.run_batch after whole-frame H2D copies (copy stream double-buffered)"}


if __name__ == "__main__":
    main()
