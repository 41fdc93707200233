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
import math
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


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32, help="frames per batch (C2: 32)")
    ap.add_argument("--bank", type=int, default=512,
                    help="distinct frames per GPU cycled through (>= streams x batch: no two in-flight batches "
                         "read the same frames)")
    ap.add_argument("--precision", default="bf16", choices=("fp32", "bf16"))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--streams", type=int, default=16,
                    help="in-flight batches per GPU: pipelines sharing one uploaded model, each with its own "
                         "context (workspace, CUDA graphs) and stream; one step = one batch on each")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 LBS + projector microbench")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 ViT-L-sized encoder microbench")
    ap.add_argument("--no-fit", action="store_true", help="skip the iterative-fit conversion microbench")
    ap.add_argument("--stream-frames", type=int, default=8192,
                    help="C5: frames of the synthetic video stream sharded across the ranks (0: skip)")
    ap.add_argument("--c4-crops", type=int, default=768, help="C4: 3 crops x 256 frames")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# distributed plumbing


def torchrun_argv(argv, n, port):
    """`python bench.py --gpus N ...` without a torchrun environment re-executes
    itself under torchrun: one process per GPU on this node (127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def maybe_spawn(args, argv):
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    if args.impl == "ours":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write("bench.py: --gpus %d but only %d CUDA device(s) visible\n" % (args.gpus, have))
            sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = torchrun_argv(argv, args.gpus, port)
    sys.stderr.write("bench.py: spawning %d ranks: %s\n" % (args.gpus, " ".join(cmd)))
    sys.exit(subprocess.call(cmd))


def dist_setup(torch, want):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "VERSION")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if rank == 0:
            sys.stderr.write("bench.py: NCCL process group, %d ranks\n" % dist.get_world_size())
        return dist, rank, ws, local
    return None, 0, 1, 0


def frame_seeds(rank, bank):
    """Rank r's frames are scenes 5000 + r * bank + i (disjoint per rank)."""
    return [5000 + rank * bank + i for i in range(bank)]


def shard_bounds(n_frames, rank, world):
    """Contiguous shard of a frame stream: [r*n/G, (r+1)*n/G)."""
    return rank * n_frames // world, (rank + 1) * n_frames // world


def gather_rows(dist, torch, rows, world):
    """All ranks' (n, k) result rows -> (world * n, k) on every rank: NCCL
    all_gather_into_tensor on the GPU, the list form on gloo/CPU."""
    if dist is None:
        return rows
    if rows.is_cuda:
        out = torch.empty((world * rows.shape[0],) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
        dist.all_gather_into_tensor(out, rows)
        return out
    parts = [torch.empty_like(rows) for _ in range(world)]
    dist.all_gather(parts, rows)
    return torch.cat(parts)


def max_over_ranks(dist, torch, ms, device):
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class Lanes:
    """In-flight lanes of one rank: CUDA streams timed with CUDA events on the
    device (cuda=True), or sequential CPU execution timed on the host (the
    gloo tests drive the same stream/shard/gather code with a stand-in
    pipeline)."""

    def __init__(self, torch, n, device, streams=None):
        self.torch, self.n, self.device = torch, n, device
        self.cuda = device.type == "cuda"
        if self.cuda:
            self.streams = streams or ([torch.cuda.current_stream(device)] +
                                       [torch.cuda.Stream(device=device) for _ in range(n - 1)])

    def lane(self, j):
        import contextlib

        return self.torch.cuda.stream(self.streams[j]) if self.cuda else contextlib.nullcontext()

    def main(self):
        import contextlib

        return self.torch.cuda.stream(self.streams[0]) if self.cuda else contextlib.nullcontext()

    def start(self):
        if self.cuda:
            self.e0 = self.torch.cuda.Event(enable_timing=True)
            self.e0.record(self.streams[0])
            for q in self.streams[1:]:
                q.wait_event(self.e0)
        else:
            self.t0 = time.perf_counter()

    def join(self):
        """Everything every lane enqueued so far happens before what the main
        lane enqueues next."""
        if self.cuda:
            for q in self.streams[1:]:
                ev = self.torch.cuda.Event()
                ev.record(q)
                self.streams[0].wait_event(ev)

    def stop(self):
        self.join()
        if self.cuda:
            self.e1 = self.torch.cuda.Event(enable_timing=True)
            self.e1.record(self.streams[0])
            self.torch.cuda.synchronize(self.device)
            return self.e0.elapsed_time(self.e1)
        return (time.perf_counter() - self.t0) * 1e3


def stream_shard(lanes, launch, frames_fn, B, dist, world, rank, total, out_width=142, result=None):
    """C5: a stream of `total` frames, rank r taking the
    contiguous block [r*total/G, (r+1)*total/G); batches of B round-robin over
    the lanes; each batch's SMPL outputs (theta + joints) land in the rank's
    result rows; ONE all-gather of the rows at the end (the path's only
    collective).  `launch(j, img, kp, nb, res, r)` enqueues a batch on lane j
    and places its (theta (nb, 76) | joints (nb, 66)) into res[r:r + nb];
    `frames_fn(f0, nb)` gives the batch's frames.  `result` = (alloc(n),
    finish(res, n)) replaces the default (n, 142) row buffer (alloc) and
    turns the launch's result object into those rows before the gather
    (finish, inside the timed region).  Returns (gathered rows (total, 142),
    ms)."""
    torch = lanes.torch
    lo, hi = shard_bounds(total, rank, world)
    n = hi - lo
    if result is None:
        res = torch.zeros((max(n, 1), out_width), dtype=torch.float32, device=lanes.device)
        finish = None
    else:
        res = result[0](n)
        finish = result[1]
    lanes.start()
    k = 0
    for f0 in range(lo, hi, B):
        nb = min(B, hi - f0)
        img, kp = frames_fn(f0, nb)
        launch(k % lanes.n, img, kp, nb, res, f0 - lo)
        k += 1
    lanes.join()
    with lanes.main():
        rows = finish(res, n) if finish is not None else (res[:n] if n else res)
        gathered = gather_rows(dist, torch, rows, world)
    ms = lanes.stop()
    return gathered, max_over_ranks(dist, torch, ms, lanes.device)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md): NVML polled from a
# thread (sub-millisecond), nvidia-smi as the fallback

_REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.stop_ev = threading.Event()
        self.t = None
        self.src = "nvml"

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, rs))
                    except pynvml.NVMLError:
                        pass
                    time.sleep(0.0005)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:  # no NVML: nvidia-smi at its 10 ms minimum
            self.src = "nvidia-smi"
            self._smi()
        return self

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def read():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                try:
                    sm, mx = float(parts[0]), float(parts[1])
                except (ValueError, IndexError):
                    continue
                self.max_mhz = mx
                bits = 0
                for (name, bit), v in zip(_REASONS.items(), parts[2:6]):
                    bits |= bit if v.lower() == "active" else 0
                self.samples.append((sm, bits))

        self.t = threading.Thread(target=read, daemon=True)
        self.t.start()

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.src == "nvidia-smi" and getattr(self, "proc", None) is not None:
            self.proc.terminate()
        if self.t is not None:
            self.t.join(timeout=5)

    def summary(self, samples=None):
        samples = self.samples if samples is None else samples
        sm = [s for s, _ in samples if self.max_mhz and s > 0.5 * self.max_mhz]
        reasons = sorted(name for name, bit in _REASONS.items() if any(r & bit for _, r in samples))
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(samples), "source": self.src}


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


def make_scenes(smpl, seeds):
    from paper_2603_15603_b200 import synth

    return [synth.random_scene(np.random.default_rng(s), smpl, (512, 512)) for s in seeds]


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


# ---------------------------------------------------------------------------
# CPU oracle (baseline / reference arm)

PORT_NOTE = ("oracle/ restatement of the reference (numpy + the two numba kernels restated in C); in the survey "
             "container the reference package itself ran this composition 1.3-1.8x slower per frame, so ratios "
             "against this arm understate the gap to the reference")


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
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                             "sample": "%d timed frames on %d host processes (one frame per process per step, %d "
                                       "steps), p50 %.1f ms/frame; %s" % (done, cores, steps, p50, PORT_NOTE)},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "p50_frame_latency_ms": p50}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the GPU arm


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    maybe_spawn(args, argv)
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch

    dist, rank, world, local = dist_setup(torch, args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import priors as pr

    clk = ClockSampler(local).__enter__()  # whole run; the timed regions are marked below
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
    pipes = [pipe] + [pipe.fork() for _ in range(S - 1)]   # one uploaded model, S contexts
    for p_ in pipes:
        p_.context().reserve(max(B, 1))
    lanes = Lanes(torch, S, dev)
    outs_s = [p_.allocate_outputs(B, tail=True) for p_ in pipes]
    cfg = pl.fast_config()

    prepared = {}  # (lane, input slot) -> PreparedBatch (arguments bound once)

    def step(i):
        """One step: batch j of every in-flight pipeline (S * B frames),
        inputs cycling through the HBM bank (larger than L2)."""
        for j in range(S):
            s = (i * S + j) % nslot
            pb = prepared.get((j, s))
            if pb is None:
                pb = prepared[(j, s)] = pipes[j].prepare(images[s * B:(s + 1) * B], kps[s * B:(s + 1) * B],
                                                         outs_s[j], cfg)
            pb.launch(lanes.streams[j])

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up: every (pipeline, input slot) pair gets its CUDA graph captured
    period = nslot // math.gcd(nslot, S)
    for i in range(max(args.warmup, 3, period)):
        step(i)
    for p_ in pipes:
        p_.context().check_finite("bench warm-up")
    barrier()
    launches0 = sum(p_.context().launches() for p_ in pipes)
    n0 = len(clk.samples)
    barrier()
    lanes.start()
    for i in range(args.steps):
        step(i)
    lanes.join()
    # the path's only collective: the final gather of the SMPL outputs
    # (theta + joints) of the last round, on the main lane
    if dist is not None:
        with lanes.main():
            rows = torch.cat([torch.cat([o["theta"], o["j_smpl"].reshape(B, 66)], 1) for o in outs_s])
            gather_rows(dist, torch, rows, world)
    ms = lanes.stop()
    barrier()
    timed_clocks = clk.samples[n0:]
    launches = sum(p_.context().launches() for p_ in pipes) - launches0
    ms = max_over_ranks(dist, torch, ms, dev)
    frames_step = S * B
    frames_total = world * frames_step * args.steps
    value = frames_total / (ms / 1e3)
    for p_ in pipes:
        p_.context().check_finite("bench")
    # the concurrent batches computed what one pipeline computes alone
    verified = verify_streams(torch, pipes, outs_s, images, kps, cfg, B, args.steps, nslot, S)

    # -- C5: an 8192-frame stream sharded across the ranks, one NCCL gather ----
    c5 = None if args.stream_frames <= 0 else stream_run(torch, pipes, lanes, images, kps, cfg, B, dist, world,
                                                          rank, args.stream_frames)

    # -- per-stage attribution (each stage alone in a CUDA graph) -------------
    stage_sat = {}
    stage_ms = attribute_stages(torch, pipe, ctx, images, kps, outs_s[0], cfg, reps=20, saturated=16,
                                saturated_out=stage_sat)
    stage_sat["sum"] = round(sum(stage_sat.values()), 2)

    # -- p50 single-frame latency ----------------------------------------------
    lat = frame_latency(torch, pipe, images, kps, cfg, reps=200)
    lat_api = api_latency(torch, pipe, images, scenes, cfg, reps=100)

    # -- end-to-end through the public API with host buffers -------------------
    e2e = None if args.no_e2e else end_to_end(torch, pipes, images, kps, cfg, B, args.steps, args.warmup, dist,
                                              world)

    # -- C3 microbench: LBS + projector on 4096 full-size meshes ---------------
    c3 = None if args.no_c3 else c3_microbench(torch, pipe, ctx, meshes=4096, reps=10)

    # -- conversion: iterative fit (the paper's slow baseline) vs projector ----
    conv = None if args.no_fit else fit_microbench(torch, pipe, meshes=148, steps=300,
                                                   projector_meshes_per_s=(c3 or {}).get("meshes_per_s"))

    # -- C4 microbench: ViT-L-sized encoder, 3 crops x 256 frames --------------
    c4 = None if args.no_c4 else c4_microbench(torch, crops=args.c4_crops, reps=3)
    clk.__exit__()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    roof = roofline(stage_ms, stage_sat, B)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        n_host = min(len(scenes), 64)
        fr = images[:n_host].cpu().numpy()
        kk = kps[:n_host].cpu().numpy()
        fps, cores, done, p50c = cpu_oracle_run(fr, kk, args.cpu_seconds)
        cpu = {"value": fps, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
               "sample": "%d frames (C2 frame->SMPL, full-size tail) on %d host processes over ~%.0f s; "
                         "p50 %.1f ms/frame single process; %s" % (done, cores, args.cpu_seconds, p50c, PORT_NOTE)}
    clocks = clk.summary(timed_clocks)  # samples taken inside the timed region
    clocks["whole_run"] = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "bf16", "data": "synthetic",
        "config": {"workload": "C2: batches of %d synthetic 512x512 frames, body + 2 hand crops -> encoder -> "
                               "pruned decoders -> MHR LBS (18439 v) -> projector -> SMPL FK; one step = one batch "
                               "on each of %d in-flight pipelines" % (B, S),
                   "batch": B, "in_flight_batches": S, "frames_per_gpu_per_step": frames_step,
                   "global_batch": frames_step * world,
                   "parallelism": "dp%d (frame sharding, one NCCL all-gather of the SMPL outputs after the "
                                  "timed steps)" % world if world > 1 else "single GPU",
                   "l2": "inputs cycle through a %d-frame bank (%.0f MB in HBM) > 126 MB L2" %
                         (bank, bank * 512 * 512 * 12 / 1e6),
                   "precision": args.precision, "graphs": True, "shared_model": True,
                   "concurrent_outputs_match_single_stream": verified},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks, "p50_frame_latency_ms": lat_api["p50_ms"], "frame_latency_api": lat_api,
        "frame_latency_device": lat,
        "stage_ms": stage_ms,
        "stage_saturated_us_per_batch": stage_sat,  # 16 concurrent copies of each stage alone, distinct frames
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


def attribute_stages(torch, pipe, ctx, images, kps, outs, cfg, reps, saturated=None, saturated_out=None):
    """Average device time of each stage kernel on one batch.  Each stage's
    launches are captured `reps` times into its own CUDA graph and the graph
    is replayed between CUDA events, so the numbers are device time, not the
    host's ctypes launch rate.  With `saturated`, the same stage runs as
    `saturated` concurrent copies (forked streams in one graph), each copy on
    DISTINCT frames and its own buffers: the device time one batch of the
    stage costs when the GPU is kept full of it."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt

    B = outs["merged"].shape[0]
    lib, h = ctx.lib, ctx.h
    prec = rt.PRECISIONS[pipe.precision]
    dev = images.device
    nv = pipe.mhr.num_vertices
    bsel, _ = dc.selection_mask(cfg.selection, 5)
    n_copies = saturated or 1
    nslot = images.shape[0] // B
    bufs = []
    for q in range(n_copies):
        o = outs if q == 0 else {k: torch.empty_like(v) for k, v in outs.items()}
        s = q % nslot
        bufs.append({"img": images[s * B:(s + 1) * B], "kp": kps[s * B:(s + 1) * B], "o": o,
                     "crops": torch.empty((B, 3, 64, 64, 3), dtype=torch.float32, device=dev),
                     "feats": torch.empty((B, 3, 64, 64), dtype=torch.float32, device=dev)})
    # each concurrent copy needs its own workspace: one forked context per copy
    ctxs = [ctx] + [rt.Context(share=ctx) for _ in range(n_copies - 1)]
    for c in ctxs:
        c.reserve(B)

    def k1(c, b):
        c.check(lib.fsb_boxes_crops(c.h, rt.ptr(b["img"]), B, 512, 512, rt.ptr(b["kp"]), 3.0, 64,
                                    rt.ptr(b["o"]["boxes"]), rt.ptr(b["o"]["prompt"]), rt.ptr(b["crops"]), None,
                                    c.stream))

    def k2(c, b):  # encoder + the decoders' cross-attention K / V (one launch, as in the frame path)
        c.check(lib.fsb_encode_frames(c.h, rt.ptr(b["crops"]), B, rt.ptr(b["feats"]), prec, c.stream))

    def k3(c, b):
        o = b["o"]
        c.check(lib.fsb_decode_frames(c.h, rt.ptr(b["feats"]), B, rt.ptr(o["prompt"]), bsel, 0,
                                      rt.ptr(o["body_params"]), rt.ptr(o["body_cam"]), rt.ptr(o["hand_rots"]),
                                      rt.ptr(o["merged"]), prec, c.stream))

    def k4a(c, b):
        c.check(lib.fsb_skin(c.h, 0, rt.ptr(b["o"]["merged"]), B, rt.ptr(b["o"]["v_mhr"]), c.stream))

    def k4b(c, b):  # projector input bridged from V_mhr + the MLP, as in the frame path
        c.check(lib.fsb_project_vertices(c.h, rt.ptr(b["o"]["v_mhr"]), B, nv, rt.ptr(b["o"]["theta"]), prec,
                                         c.stream))

    stages = [("k1_boxes_crops", k1), ("k2_encoder", k2), ("k3_decoders", k3), ("k4_fk_lbs", k4a),
              ("k4_proj_mlp", k4b)]
    for q in range(n_copies):  # eager pass: real inputs for every stage of every copy
        for _, fn in stages:
            fn(ctxs[q], bufs[q])
    torch.cuda.synchronize()
    out = {}
    side = torch.cuda.Stream(device=dev)
    for name, fn in stages:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side, capture_error_mode="relaxed"):
                for _ in range(reps):
                    fn(ctx, bufs[0])
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = float(e0.elapsed_time(e1) / (3 * reps))
    if saturated:
        branches = [torch.cuda.Stream(device=dev) for _ in range(n_copies)]
        for name, fn in stages:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side, capture_error_mode="relaxed"):
                    for q, br in enumerate(branches):
                        br.wait_stream(side)
                        with torch.cuda.stream(br):
                            for _ in range(4):
                                fn(ctxs[q], bufs[q])
                    for br in branches:
                        side.wait_stream(br)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            saturated_out[name] = round(float(1e3 * e0.elapsed_time(e1) / (3 * 4 * n_copies)), 2)
    return out


def _peaks():
    peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        peaks = {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]), "src": "measured"}
    except (OSError, KeyError, ValueError):
        pass
    return peaks


def roofline(stage_ms, stage_sat, B):
    """Roofline of the dominant stage kernel against MEASURED_PEAKS.json:
    `achieved` from the stage's isolated launch time (one batch alone on the
    GPU), `achieved_saturated` from its per-batch cost with 16 concurrent
    copies (how the pipeline runs it)."""
    peaks = _peaks()
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
    sat_s = stage_sat.get(dom, 0.0) / 1e6
    if bound == "hbm":
        scale, peak, unit = 1e9, peaks["hbm_gbs"], "GB/s"
    else:
        scale, peak, unit = 1e12, peaks["bf16_tflops"], "TFLOP/s"
    achieved = amount / sec / scale
    achieved_sat = amount / sat_s / scale if sat_s > 0 else None
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
            "achieved_saturated": achieved_sat, "frac_saturated": achieved_sat / peak if achieved_sat else None,
            "share_of_step": stage_ms[dom] / sum(stage_ms.values()),
            "share_of_saturated_step": stage_sat.get(dom, 0.0) / max(stage_sat.get("sum", 0.0), 1e-9),
            "algorithmic_per_launch": amount, "launch_ms": stage_ms[dom]}


def frame_latency(torch, pipe, images, kps, cfg, reps):
    """p50 device latency of one HBM-resident frame through the whole path
    (graph replay, CUDA events)."""
    outs = pipe.allocate_outputs(1, tail=True)
    st = torch.cuda.current_stream()
    for i in range(5):
        pipe.launch(images[i:i + 1], kps[i:i + 1], outs, cfg)
    torch.cuda.synchronize()
    ts = []
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        pipe.launch(images[r % 8:r % 8 + 1], kps[r % 8:r % 8 + 1], outs, cfg)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return {"p50_ms": ts[len(ts) // 2], "p95_ms": ts[int(len(ts) * 0.95)], "reps": reps, "batch": 1,
            "api": "graph replay of one HBM-resident frame (device time)"}


def api_latency(torch, pipe, images, scenes, cfg, reps):
    """p50 single-frame latency through the reference-shaped API:
    Pipeline.run_smpl(image numpy (512, 512, 3), scene) -> host theta / SMPL
    joints: host finiteness check, staging into pinned memory, one graph
    replay (K1 gathers the crop footprints over PCIe), results read back.
    Host wall clock around the call."""
    host = [images[i].cpu().numpy() for i in range(8)]
    for i in range(5):
        pipe.run_smpl(host[i % 8], scenes[i % 8], cfg)
    ts = []
    for r in range(reps):
        t0 = time.perf_counter()
        pipe.run_smpl(host[r % 8], scenes[r % 8], cfg)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    return {"p50_ms": ts[len(ts) // 2], "p95_ms": ts[int(len(ts) * 0.95)], "reps": reps, "batch": 1,
            "api": "Pipeline.run_smpl(numpy image, scene) -> numpy theta/joints (host wall clock)"}


def stream_run(torch, pipes, lanes, images, kps, cfg, B, dist, world, rank, total):
    """C5 on the GPU: stream_shard with the real pipelines.
    Frame i of the stream is bank frame i % bank; batches of B spread over the
    in-flight pipelines; the SMPL outputs all-gathered over NCCL once at the
    end.  Strong scaling: frames/s of the whole stream, first frame to
    gathered result, max over ranks."""
    lo, hi = shard_bounds(total, rank, world)
    dev = images.device
    bank = images.shape[0]
    S = len(pipes)
    outs = [p_.allocate_outputs(B, tail=True) for p_ in pipes]

    views = {}  # bank offset -> (frames, keypoints) views, built once

    def frames_fn(f0, nb):
        s0 = f0 % bank
        if s0 + nb <= bank:
            v = views.get((s0, nb))
            if v is None:
                v = views[(s0, nb)] = (images[s0:s0 + nb], kps[s0:s0 + nb])
            return v
        idx = torch.arange(f0, f0 + nb, device=dev) % bank
        return images[idx], kps[idx]

    # every batch writes theta / joints straight into the stream's result
    # arrays (its outputs are row slices of them): one prepared graph per
    # (lane, frame slot, result rows), captured in an untimed pass of the
    # same stream, then one C call per batch in the timed pass -- no per-batch
    # copies (the row copies of the first version made C5 host-bound)
    n = hi - lo
    theta_all = torch.zeros((max(n, 1), 76), dtype=torch.float32, device=dev)
    j_all = torch.zeros((max(n, 1), 22, 3), dtype=torch.float32, device=dev)
    prepared = {}

    def launch(j, img, kp, nb, res, r):
        st = lanes.streams[j]
        th, jj = res
        key = (j, img.data_ptr(), r, nb)
        pb = prepared.get(key)
        if pb is None:
            o = dict(outs[j]) if nb == B else pipes[j].allocate_outputs(nb, tail=True)
            o["theta"], o["j_smpl"] = th[r:r + nb], jj[r:r + nb]
            pb = prepared[key] = pipes[j].prepare(img, kp, o, cfg)
        pb.launch(st)

    result = (lambda n_: (theta_all, j_all),
              lambda res, n_: torch.cat([res[0][:n_], res[1][:n_].reshape(n_, 66)], 1))
    # warm-up: the whole stream once, untimed (captures every batch's graph)
    stream_shard(lanes, launch, frames_fn, B, dist, world, rank, total, result=result)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    gathered, ms = stream_shard(lanes, launch, frames_fn, B, dist, world, rank, total, result=result)
    # the rows this rank gathered for its first and last batch equal a fresh
    # single-stream run of the same frames
    ok = True
    chk = pipes[0].allocate_outputs(B, tail=True)
    for f0 in sorted({lo, lo + ((n - 1) // B) * B}):
        nb = min(B, hi - f0)
        if nb != B:
            continue
        img, kp = frames_fn(f0, nb)
        pipes[0].launch(img, kp, chk, cfg)
        torch.cuda.synchronize()
        want = torch.cat([chk["theta"], chk["j_smpl"].reshape(nb, 66)], 1)
        ok = ok and bool(torch.equal(gathered[f0:f0 + nb], want))
    return {"workload": "C5: %d-frame synthetic stream sharded over %d GPU(s) (%d frames on this rank), batches of %d "
                        "on %d in-flight pipelines, one all-gather of the SMPL outputs (theta + joints)"
                        % (total, world, n, B, S),
            "ms": ms, "frames_per_s": total / (ms / 1e3), "scaling": "strong",
            "gathered_rows": int(gathered.shape[0]), "gathered_bytes_per_rank": int(n * 142 * 4),
            "outputs_verified": ok}


def verify_streams(torch, pipes, outs_s, images, kps, cfg, B, steps, nslot, S):
    """Re-run the last step's batch of every lane alone on pipeline 0 and
    compare bit for bit with what the concurrent run produced."""
    torch.cuda.synchronize()
    ref = pipes[0].allocate_outputs(B, tail=True)
    ok = True
    for j in range(S):
        s = ((steps - 1) * S + j) % nslot
        got = {k: outs_s[j][k].clone() for k in ("merged", "theta", "j_smpl")}
        pipes[0].launch(images[s * B:(s + 1) * B], kps[s * B:(s + 1) * B], ref, cfg)
        torch.cuda.synchronize()
        ok = ok and all(torch.equal(got[k], ref[k]) for k in got)
    return bool(ok)


E2E_STREAMS = int(os.environ.get("FSB_E2E_STREAMS", "16"))


def pinned_h2d_gbs(torch, dev, nbytes=256 << 20):
    """Measured pinned host -> HBM copy bandwidth (the e2e roofline's
    denominator): one 256 MB cudaMemcpyAsync, best of 3."""
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def host_read_gbs(torch, dev, nbytes=256 << 20):
    """Measured SM-driven read rate of pinned host memory (cp.async.bulk from
    the mapped host pointer, as K1 reads host frames): 256 MB, best of 3 over
    a few CTA counts."""
    import ctypes

    from paper_2603_15603_b200 import runtime as rt

    lib = rt.lib()
    fn = lib.fsb_debug_host_read
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    best = 0.0
    for ctas in (148, 296, 592):
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if fn(h.data_ptr(), nbytes, d.data_ptr(), ctas, st.cuda_stream) != 0:
                raise RuntimeError("fsb_debug_host_read failed")
            e1.record(st)
            torch.cuda.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    if not torch.equal(h[: 1 << 16], d[: 1 << 16].cpu()):
        raise RuntimeError("fsb_debug_host_read copied wrong bytes")
    return best


def end_to_end(torch, pipes, images, kps, cfg, B, steps, warmup, dist, world):
    """Pipeline.run_batch on frames that live in pinned host memory (the
    reference's images are host float32 arrays).  K1 reads each frame in
    place over PCIe -- only the crop footprints (the rows and x-spans the
    three crops tap) cross the bus -- so there is no separate whole-frame
    H2D copy; steps rotate over E2E_STREAMS streams so one batch's gather
    overlaps the others' compute.  Every step ends with a D2H read of
    merged/theta/j_smpl into pinned host buffers; after the timed region every
    context's non-finite flag is read (NumericError contract).  The host bank
    (every frame of the HBM bank) is several times the 126 MB L2, so the crop
    footprints cannot be served from L2.  h2d_bytes_per_step is counted on
    the device by K1 (fsb_input_bytes) plus the keypoints."""
    NS = E2E_STREAMS
    pipes = list(pipes[:NS])
    while len(pipes) < NS:
        pipes.append(pipes[0].fork())
    ctxs = [p_.context() for p_ in pipes]
    dev = images.device
    nhost = min(images.shape[0], 256)
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

    for i in range(max(warmup, NS * nslot // math.gcd(NS, nslot))):
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
    n_e2e = max(steps, 2 * nslot)  # every host frame at least twice
    for i in range(n_e2e):
        run(i)
    for j in range(NS):
        tail[j].record(streams[j])
        streams[0].wait_event(tail[j])
    e1.record(streams[0])
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    for c in ctxs:  # the reference raises NumericError on non-finite results
        c.check_finite("e2e")
    frame_bytes = sum(c.input_bytes(reset=True) for c in ctxs)
    # the host-side results of the last step of each stream equal a fresh
    # device-frame run of the same frames
    ok = True
    ref = pipes[0].allocate_outputs(B, tail=True)
    for j in range(min(NS, n_e2e)):
        last = max(i for i in range(n_e2e) if i % NS == j)
        s = last % nslot
        pipes[0].launch(images[s * B:(s + 1) * B], kps[s * B:(s + 1) * B], ref, cfg)
        torch.cuda.synchronize()
        ok = ok and all(torch.equal(h_out[j][k], ref[k].cpu()) for k in ("merged", "theta", "j_smpl"))
    ms = max_over_ranks(dist, torch, ms, dev)
    h2d_b = frame_bytes // n_e2e + B * 44 * 4
    d2h_b = B * (76 + 76 + 66) * 4
    full = B * (images[0].numel() + 44) * 4
    peak_copy = pinned_h2d_gbs(torch, dev)
    peak_read = host_read_gbs(torch, dev)
    peak = max(peak_copy, peak_read)
    achieved = h2d_b / (ms / n_e2e / 1e3) / 1e9
    return {"value": world * B * n_e2e / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d_b,
            "d2h_bytes_per_step": d2h_b, "ms_per_step": ms / n_e2e, "steps": n_e2e, "batch": B,
            "api": "Pipeline.run_batch on pinned host frames (K1 gathers the crop footprints over PCIe in "
                   "place; %d streams; %d-frame host bank, %.0f MB)" % (NS, nhost, nhost * 512 * 512 * 12 / 1e6),
            "h2d_fraction_of_frames": h2d_b / full, "outputs_verified": bool(ok), "nonfinite_checked": True,
            "roofline": {"bound": "pcie", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_copy_engine_gbs": peak_copy, "peak_sm_bulk_read_gbs": peak_read,
                         "peak_source": "max of measured pinned H2D cudaMemcpyAsync and SM cp.async.bulk reads of "
                                        "mapped pinned host memory (fsb_debug_host_read), 256 MB each"}}


if __name__ == "__main__":
    main()
