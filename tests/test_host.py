"""CPU: the C-ABI library loads and exports the header's entry points, and
the host-side logic (plans, selection masks, operand packing, frame
sharding across ranks) behaves like the reference."""

import ctypes
import os
import re
from dataclasses import replace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "fsb_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsb_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_15603_b200 import _build, runtime

    if not os.path.exists(runtime.LIB_PATH):
        _build.build()
    return ctypes.CDLL(runtime.LIB_PATH)


def test_library_exports_every_header_symbol(lib):
    names = _header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), "libfsb_b200.so does not export %s" % n


def test_runtime_binds_every_header_symbol():
    from paper_2603_15603_b200 import runtime

    assert set(_header_functions()) == set(runtime.exported_symbols())


@pytest.mark.parametrize("n", [0, 7, 1 << 16, 512 * 512 * 3, 1000003])
def test_stage_frame_copies_and_flags_non_finite(lib, n):
    """fsb_stage_frame (host-only): the single-frame path's check_finite +
    pinned staging copy in one pass over a thread pool
    (numkit.py:136-140 semantics: any NaN / inf raises)."""
    fn = lib.fsb_stage_frame
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]
    rng = np.random.default_rng(n)
    src = rng.standard_normal(n).astype(np.float32)
    dst = np.full(n, 7.0, np.float32)
    bad = ctypes.c_int(-1)
    assert fn(src.ctypes.data, dst.ctypes.data, n, ctypes.byref(bad)) == 0
    assert bad.value == 0 and np.array_equal(src, dst)
    for v in (np.nan, np.inf, -np.inf):
        for pos in {0, n // 2, n - 1} if n else set():
            s2 = src.copy()
            s2[pos] = v
            assert fn(s2.ctypes.data, dst.ctypes.data, n, ctypes.byref(bad)) == 0
            assert bad.value == 1
            assert np.array_equal(s2, dst, equal_nan=True)
    big = np.full(n, np.finfo(np.float32).max, np.float32)  # large but finite
    assert fn(big.ctypes.data, dst.ctypes.data, n, ctypes.byref(bad)) == 0 and bad.value == 0


def test_build_info_without_gpu(lib):
    lib.fsb_build_info.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.fsb_build_info()


def test_library_is_sm100a_only():
    import subprocess

    from paper_2603_15603_b200 import runtime

    out = subprocess.run(["cuobjdump", "--list-elf", runtime.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_tcgen05_and_bulk_copy_in_sass():
    import subprocess

    from paper_2603_15603_b200 import runtime

    sass = subprocess.run(["cuobjdump", "-sass", runtime.LIB_PATH], capture_output=True, text=True).stdout
    for op in ("UTCHMMA", "LDTM", "UBLKCP", "UTCBAR"):
        assert op in sass, op
    # the CTA-pair GEMM: M = 256 MMAs across two SMs, pair TMA loads and
    # multicast commits
    for op in ("UTCHMMA.2CTA", "UTMALDG.2D.2CTA", "UTCBAR.2CTA.MULTICAST", "UTMASTG.2D"):
        assert op in sass, op


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2603_15603_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2603_15603_b200 import runtime

    monkeypatch.setattr(runtime, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(runtime, "_LIB", None)
    with pytest.raises(RuntimeError, match="not built"):
        runtime.lib()


# ---------------------------------------------------------------------------
# operand packing (host side of the tcgen05 kernels)


def test_pack_kmajor_matches_layout_formula():
    from paper_2603_15603_b200 import runtime

    r, k = 24, 48
    m = np.arange(r * k, dtype=np.uint16).reshape(r, k)
    img = runtime.pack_kmajor(m)
    for rr in range(r):
        for kk in range(k):
            off = (rr // 8) * k * 16 + (kk // 8) * 128 + (rr % 8) * 16 + (kk % 8) * 2
            assert img[off // 2] == m[rr, kk]


def test_bf16_rounding():
    from paper_2603_15603_b200 import runtime

    x = np.array([1.0, -2.5, 3.14159, 1e-3, 65504.0], np.float32)
    back = runtime.bf16_bits_to_f32(runtime.to_bf16_bits(x))
    assert np.all(np.abs(back - x) <= np.abs(x) * 2.0 ** -8)
    assert back[0] == 1.0 and back[1] == -2.5


# ---------------------------------------------------------------------------
# plans and configuration (reference test_pipeline.py:38-107)


def test_plan_topology_and_buffers():
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200.numkit import UsageError

    for cfg in (pl.serial_config(), pl.fast_config(), pl.limit_config(),
                replace(pl.fast_config(), hands=False), replace(pl.fast_config(), batch_encode=False)):
        plan = pl.build_plan(cfg)
        assert plan.stages[0].name == "detect" and plan.stages[-1].name == "merge"
    stages = pl._stage_graph(pl.fast_config())
    with pytest.raises(UsageError):
        pl.PipelinePlan((stages[-1],) + stages[1:-1] + (stages[0],), pl.FAST_STATIC)
    with pytest.raises(UsageError):
        pl.PipelinePlan(stages + (stages[0],), pl.FAST_STATIC)
    with pytest.raises(UsageError):
        pl.PipelinePlan(stages, "jit_compiled")
    plan = pl.build_plan(pl.fast_config())
    a = plan.buffer("scratch", (4, 4))
    assert plan.buffer("scratch", (4, 4)) is a and plan.allocations == 1
    with pytest.raises(UsageError):
        with plan.stage("refine_pass"):
            pass


def test_accelerated_path_rejects_serial_configs():
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200.numkit import UsageError

    for cfg in (pl.serial_config(), pl.limit_config(), replace(pl.fast_config(), refine=True)):
        with pytest.raises(UsageError):
            pl._check_fast(cfg)
    pl._check_fast(pl.fast_config())


def test_selection_masks():
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200.numkit import UsageError

    assert dc.selection_mask((0, 1, 2), 5) == (0b111, 3)
    assert dc.selection_mask((), 5) == (0, 0)
    assert dc.selection_mask((4, 4, 0), 5) == (0b10001, 2)
    with pytest.raises(UsageError):
        dc.selection_mask((5,), 5)


def test_equivalence_report():
    from paper_2603_15603_b200 import pipeline as pl

    a = np.zeros(76, np.float32)
    b = a.copy()
    b[52] = 1e-3
    assert pl.check_equivalence(a, a).passed
    r = pl.check_equivalence(a, b, {"tier": "bounded", "max_abs": 1e-2})
    assert r.passed and r.deltas["left_hand"] == pytest.approx(1e-3)


def test_fsb1_round_trip(tmp_path):
    from paper_2603_15603_b200 import numkit as nk

    a = np.arange(24, dtype=np.float32).reshape(2, 3, 4)
    nk.write_fsb1(tmp_path / "a.fsb1", a)
    assert np.array_equal(nk.read_fsb1(tmp_path / "a.fsb1"), a)
    raw = (tmp_path / "a.fsb1").read_bytes()
    assert raw[:4] == b"FSB1" and len(raw) == 8 + 12 + 96
    (tmp_path / "b.fsb1").write_bytes(b"NOPE")
    with pytest.raises(nk.UsageError):
        nk.read_fsb1(tmp_path / "b.fsb1")


def test_render_records_layout(full_models):
    from paper_2603_15603_b200 import priors as pr
    from paper_2603_15603_b200 import synth

    _, smpl, _ = full_models
    sc = synth.random_scene(np.random.default_rng(5000), smpl, (512, 512))
    rec = pr.render_records([sc])
    assert rec.shape == (1, 116) and rec.nbytes == 464
    assert np.array_equal(rec[0, :44].reshape(22, 2), sc.keypoints2d)
    gdir = rec[0, 112:116].view(np.float64)
    rng = np.random.default_rng(sc.seed)
    rng.uniform(0.4, 1.0, size=(22, 3))
    assert np.array_equal(gdir, rng.uniform(-1.0, 1.0, size=2))


# ---------------------------------------------------------------------------
# multi-GPU sharding logic: frames shard across ranks with no exchange until
# the final gather of SMPL outputs (exercised here with gloo, world size 2)


def test_shard_bounds_cover_stream():
    import bench

    for world in (1, 2, 4, 8):
        spans = [bench.shard_bounds(8192, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 8192
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        assert len({b - a for a, b in spans}) == 1
    seeds = [set(bench.frame_seeds(r, 256)) for r in range(8)]
    assert all(not (seeds[i] & seeds[j]) for i in range(8) for j in range(i + 1, 8))


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = bench.shard_bounds(64, rank, world)
    # stand-in per-frame SMPL outputs: a deterministic function of the frame id
    frames = torch.arange(lo, hi, dtype=torch.float32)
    packed = torch.stack([frames * 1.5, frames + 0.25], dim=1)
    out = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(out, packed)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((torch.cat(out).numpy(), float(t.item())))
    dist.destroy_process_group()


def test_gloo_two_rank_gather_of_sharded_frames():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = np.arange(64, dtype=np.float32)
    assert np.array_equal(gathered, np.stack([ids * 1.5, ids + 0.25], axis=1))
    assert tmax == 2.0


def _bench_shard_worker(rank, world, port, q):
    """Runs bench.stream_shard -- the C5 code path bench.py drives on the GPU
    (lanes, ragged last batch, per-rank result rows, ONE gather) -- on CPU
    over gloo, with a stand-in pipeline whose SMPL outputs are a
    deterministic function of the frame."""
    import torch
    import torch.distributed as dist

    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total, B, bank = 200, 32, 48
    frames = torch.arange(bank, dtype=torch.float32)[:, None, None, None].expand(bank, 2, 2, 3).contiguous()
    kps = torch.arange(bank, dtype=torch.float32)[:, None, None].expand(bank, 22, 2).contiguous()

    def frames_fn(f0, nb):
        idx = torch.arange(f0, f0 + nb) % bank
        return frames[idx], kps[idx]

    calls = []

    def launch(j, img, kp, nb, res, r):  # stand-in for Pipeline.launch on lane j + result placement
        calls.append((j, nb))
        fid = img[:, 0, 0, 0]
        res[r:r + nb, :76] = fid[:, None] * 0.5 + torch.arange(76, dtype=torch.float32)[None]
        res[r:r + nb, 76:] = (kp[:, :, :1].expand(nb, 22, 3) + 0.25).reshape(nb, 66)

    lanes = bench.Lanes(torch, 3, torch.device("cpu"))
    gathered, ms = bench.stream_shard(lanes, launch, frames_fn, B, dist, world, rank, total)
    if rank == 0:
        q.put((gathered.numpy(), ms, calls))
    dist.destroy_process_group()


def test_bench_stream_shard_gloo_two_ranks():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bench_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, ms, calls = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fid = (np.arange(200) % 48).astype(np.float32)
    want = np.concatenate([fid[:, None] * 0.5 + np.arange(76, dtype=np.float32)[None],
                           np.repeat(fid[:, None] + 0.25, 66, axis=1)], axis=1)
    assert gathered.shape == (200, 142)
    assert np.array_equal(gathered, want)
    # rank 0 owns frames [0, 100): batches of 32, 32, 32, 4 round-robin over 3 lanes
    assert calls == [(0, 32), (1, 32), (2, 32), (0, 4)]
    assert ms >= 0.0


def test_bench_self_spawns_torchrun():
    """`bench.py --gpus N` outside torchrun re-executes itself under
    torch.distributed.run with N ranks on 127.0.0.1."""
    import bench

    argv = bench.torchrun_argv(["--gpus", "4", "--steps", "20"], 4, 29555)
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert argv[argv.index("--nproc-per-node") + 1] == "4"
    assert argv[argv.index("--master-addr") + 1] == "127.0.0.1"
    assert argv[-4:] == ["--gpus", "4", "--steps", "20"] and argv[-5].endswith("bench.py")
    a = bench.parse(["--gpus", "4"])
    assert a.gpus == 4 and a.steps >= 20 and a.warmup >= 3
