#!/usr/bin/env python
"""Benchmark of the B200 fusion + property-query path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

A step = one full pass of the hot path over one object: voxel-domain bbox, the per-object
G = fmap @ text^T table, the fused project / depth-test / gather / normalise / similarity /
softmax / regression / voxel + integrate partials kernel, (N>1: partial all-reduce), voxel-mass
finalisation. Default workload: BASELINE config 5 (16M points, 64 views, 37x37x1024 bf16 maps,
K=128, 512^3 grid) — the config BASELINE quotes at 1/2/4/8 GPUs; it fits one B200. Points are
range-sharded across ranks (strong scaling); views are replicated.

`value` = point-view samples/s over the whole job with inputs resident in HBM; `e2e` = the same
through the public API with inputs uploaded from pinned host memory and per-point properties +
mass read back inside the timed region. `--impl reference` times the CPU oracle port of the
reference (rank 0 only) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
SIMT_FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # nominal at max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=None, help="points in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-simt", action="store_true")
    ap.add_argument("--feature-kernel", action="store_true", help="bf16: the feature-product tile kernel (A/B)")
    ap.add_argument("--serial-prepare", action="store_true",
                    help="A/B: build the per-object G table on the step's stream before fuse_query")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def device_and_backend(local):
    """cuda:LOCAL_RANK over NCCL. PF_BENCH_DEVICE / PF_BENCH_BACKEND override both for the
    single-GPU smoke test of the multi-rank code path (gloo: every collective is a host-side step,
    so ranks sharing one GPU never have kernels waiting on each other); never used for timing."""
    dev_index = int(os.environ.get("PF_BENCH_DEVICE", local))
    return dev_index, os.environ.get("PF_BENCH_BACKEND", "nccl")


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------------------------
def algorithmic_bytes(cfg, n, nv, k, p, d, fmap_bytes, cells, kpad):
    """Compulsory HBM bytes of one fused-kernel launch (SURVEY §8d formula + the bitset/counts the
    kernel writes + the G table it reads): points 12N; depth V*H*W*4; maps V*Hf*Wf*D*b; text K*D*4
    and table K*P*4 (read by prepare / the kernel); G cells*Kpad*4; outputs N*(4P + 4 code +
    4 count + 4*ceil(V/32) mask)."""
    h = w = cfg.image
    hf, wf, _ = cfg.fmap
    nwords = (nv + 31) // 32
    return (12 * n + nv * h * w * 4 + nv * hf * wf * d * fmap_bytes + k * d * 4 + k * p * 4
            + cells * kpad * 4 + n * (4 * p + 4 + 4 + 4 * nwords))


def cpu_oracle_run(wl, sample: int):
    """Time the oracle port of the reference on the first `sample` points (all views)."""
    from oracle import propfield_oracle as O

    views = wl.views(f32_maps=True)
    pts = wl.points[:sample]
    # JIT warm-up of the numba kernels on a tiny slice (excluded, like kernels.warmup())
    O.fuse_and_query(pts[:64], views, wl.text, wl.values, wl.cfg.temperature, wl.cfg.eps, 8)
    t0 = time.perf_counter()
    out = O.fuse_and_query(pts, views, wl.text, wl.values, wl.cfg.temperature, wl.cfg.eps, wl.cfg.grid)
    dt = time.perf_counter() - t0
    return dt, out


_PAR = {}


def _par_init():
    """Pool worker: one BLAS thread (the processes are the parallelism), numba JIT warm-up."""
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass
    from oracle import propfield_oracle as O

    d = _PAR
    O.fuse_and_query(d["pts"][:64], d["views"], d["text"], d["values"], d["T"], d["eps"], 8)


def _par_chunk(idx):
    from oracle import propfield_oracle as O

    d = _PAR
    O.fuse_and_query(d["pts"][idx], d["views"], d["text"], d["values"], d["T"], d["eps"], d["grid"])
    return len(idx)


def cpu_oracle_parallel(wl, sample: int, procs: int, reps: int = 1) -> list:
    """The oracle port of the reference over `sample` points split across `procs` forked processes
    (the reference's algorithm is independent per point; its numba kernels are single-threaded, so
    the host's cores are used through processes). Returns the wall time of the parallel pass (JIT
    warm-up excluded) of each of `reps` passes."""
    import multiprocessing as mp

    _PAR.update(views=wl.views(f32_maps=True), pts=wl.points[:sample], text=wl.text, values=wl.values,
                T=wl.cfg.temperature, eps=wl.cfg.eps, grid=wl.cfg.grid)
    chunks = [c for c in np.array_split(np.arange(sample), procs * 4) if len(c)]
    times = []
    with mp.get_context("fork").Pool(procs, initializer=_par_init) as pool:
        pool.map(abs, range(procs))  # workers up (their initializers have run)
        for _ in range(reps):
            t0 = time.perf_counter()
            pool.map(_par_chunk, chunks, chunksize=1)
            times.append(time.perf_counter() - t0)
    return times


def _rows_chunk(idx):
    from oracle import propfield_oracle as O

    d = _PAR
    p = d["pts"][idx].astype(np.float64)
    vis = O.visibility_mask(p, d["views"], d["eps"])
    feats, counts = O.aggregate_geometric_features(p, d["views"], vis)
    fhat = O.normalize_rows(feats)
    featured = counts > 0
    weights = np.zeros((p.shape[0], d["text"].shape[0]))
    if featured.any():
        weights[featured] = O.softmax_weights(O.material_similarity(fhat[featured], d["text"]), d["T"])
    props = O.regress_with_weights(weights, d["values"])
    codes, _ = O.voxel_codes(d["pts"][idx], d["grid"], d["lo"], d["hi"])
    return idx, counts, props, codes


def cpu_oracle_rows(wl, idx, procs: int) -> dict:
    """Per-point oracle outputs (counts, props, voxel codes over the full object's domain) for the
    points `idx`, over `procs` forked processes (parity check only; never timed)."""
    import multiprocessing as mp

    p64 = wl.points.astype(np.float64)
    _PAR.update(views=wl.views(f32_maps=True), pts=wl.points, text=wl.text, values=wl.values, T=wl.cfg.temperature,
                eps=wl.cfg.eps, grid=wl.cfg.grid, lo=p64.min(axis=0), hi=p64.max(axis=0))
    chunks = [c for c in np.array_split(np.asarray(idx), procs * 4) if len(c)]
    with mp.get_context("fork").Pool(procs, initializer=_par_init) as pool:
        parts = pool.map(_rows_chunk, chunks, chunksize=1)
    order = np.argsort(np.concatenate([q[0] for q in parts]), kind="stable")
    return {k: np.concatenate([q[j] for q in parts])[order] for j, k in ((1, "counts"), (2, "props"), (3, "codes"))}


def default_cpu_sample(cfg) -> int:
    # ~10-20 s of CPU work at the reference's ~1 M samples/s
    return int(min(cfg.n, max(2000, 12_000_000 // max(1, cfg.nviews) // max(1, cfg.d // 512))))


def cores_used() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------------------------
def run_reference(args, cfg):
    """`--impl reference`: the reference algorithm (CPU oracle port) on the host cores, rank 0."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2511_03126_b200 import workloads

    procs = cores_used()
    sample = min(cfg.n, args.cpu_sample or max(2000, default_cpu_sample(cfg) // 4) * procs)
    wl = workloads.generate(cfg, device_splat=cfg.n > 500_000)
    wl.points = wl.points[:sample] if wl.points.shape[0] > sample else wl.points
    times = cpu_oracle_parallel(wl, sample, procs, reps=args.warmup + args.steps)[args.warmup:]
    t = statistics.mean(times)
    value = sample * cfg.nviews / t
    line = {
        "impl": "reference", "metric": "point-view samples/sec", "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {**config_desc(cfg), "parallelism": (f"cell-range x{world} (points routed to voxel owners)"
                                                       if world > 1 else "single GPU"),
                   "l2": "inputs larger than L2"},
        "rate_note": (f"samples/s of {sample} of the {cfg.n} points x {cfg.nviews} views per step; the "
                      "reference's algorithm is independent per point, so the rate carries to the whole object"),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": procs, "kind": "port",
                         "sample": f"first {sample} of {cfg.n} points x {cfg.nviews} views per step, "
                                   f"point chunks over {procs} processes (numba kernels single-threaded "
                                   "per process, as the reference's backend)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_desc(cfg):
    hf, wf, d = cfg.fmap
    return {"workload": f"{cfg.name}: N={cfg.n} points, V={cfg.nviews} views, {cfg.image}^2 depth, "
                        f"{hf}x{wf}x{d} {'bf16' if cfg.bf16 else 'f32'} maps, K={cfg.k}, {cfg.grid}^3 grid",
            "points": cfg.n, "views": cfg.nviews, "image": cfg.image, "fmap": list(cfg.fmap),
            "feature_storage": "bf16" if cfg.bf16 else "f32", "materials": cfg.k, "grid": cfg.grid,
            "temperature": cfg.temperature, "eps": cfg.eps}


# ---------------------------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch

    rank, world, local = env_rank()
    dev_index, backend = device_and_backend(local)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_2511_03126_b200 as pf
    from paper_2511_03126_b200 import _lib, workloads
    from paper_2511_03126_b200.dist import shard_range

    wl = workloads.generate(cfg, device_splat=True)
    n_total = cfg.n
    lo, hi = shard_range(n_total, rank, world)
    nv = cfg.nviews
    R = np.stack([p.rotation for p in wl.poses])
    tv = np.stack([p.translation for p in wl.poses])
    intr = np.tile([wl.intrinsics.fx, wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy], (nv, 1))
    if cfg.bf16:
        fmap_dev = torch.from_numpy(wl.fmaps.view(np.int16)).to(dev).view(torch.bfloat16)
    else:
        fmap_dev = torch.from_numpy(wl.fmaps).to(dev)
    depth_dev = wl.depth.to(dev)
    views = pf.ViewSet.from_tensors(R, tv, intr, depth_dev, fmap_dev, device=dev)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, density_col=0, device=dev)
    pts_host = np.ascontiguousarray(wl.points[lo:hi])
    pts = torch.from_numpy(pts_host).to(dev)
    n = pts.shape[0]
    stream = torch.cuda.current_stream()
    if world > 1:
        # cell-range sharding (dist.cell_sharded_steps): points routed to the rank owning their
        # voxel, so only a 1 MB histogram and K + 8 doubles are all-reduced (no dense voxel grid)
        from paper_2511_03126_b200.dist import DeviceShardOps, cell_sharded_steps, run_dist

        bufs = None
        shard_ops = DeviceShardOps(views, tables, temperature=cfg.temperature, epsilon=cfg.eps, grid=cfg.grid)
        nwords = (nv + 31) // 32

        def step(ev=None):
            if ev:
                ev[0].record(stream)
                ev[1].record(stream)
            res = run_dist(cell_sharded_steps(pts, rank, world, shard_ops, k=tables.k, p=tables.p, nwords=nwords))
            if ev:
                ev[2].record(stream)
            return res
    else:
        bufs = pf.FuseBuffers(n, views, tables, cfg.grid, device=dev)

        def step(ev=None):
            bufs.reset()
            if ev:
                ev[0].record(stream)
            if args.serial_prepare:  # A/B knob: the per-object tables on the step's stream first
                pf.fuse_prepare(views, tables, bufs)
            if ev:
                ev[1].record(stream)
            # default: pf_fuse_query builds the tables itself on a forked stream, concurrently with
            # the point sort and the tile prep
            res = pf.fuse_and_query(pts, views, tables, temperature=cfg.temperature, epsilon=cfg.eps,
                                    grid=cfg.grid, buffers=bufs, reduce=False,
                                    prepared=args.serial_prepare, force_simt=args.force_simt, reset=False,
                                    feature_kernel=args.feature_kernel)
            if ev:
                ev[2].record(stream)
            res.finalize()
            return res

    inputs_bytes = (pts.numel() * 4 + depth_dev.numel() * 4 + fmap_dev.numel() * fmap_dev.element_size())
    flush = inputs_bytes < 2 * L2_BYTES
    scratch = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if flush else None

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    evs = [[mk() for _ in range(4)] for _ in range(args.steps)]
    starts = [mk() for _ in range(args.steps)]
    clk = ClockSampler(dev_index)
    clk.start()
    # soak: untimed steps for >= 0.8 s so the clock samples (200 ms period) see the GPU under load
    t_soak = time.time()
    while time.time() - t_soak < 0.8:
        step()
        torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    _lib.stage_timing(True)  # CUDA events at the tile path's stage boundaries (same stream)
    for i in range(args.steps):
        if flush:
            scratch.fill_(float(i))  # L2 flush between steps (outside the step's events)
        starts[i].record(stream)
        res = step(evs[i])
        evs[i][3].record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    launches = _lib.launch_count() - launches0
    st_calls, st_ms = _lib.stage_times()
    _lib.stage_timing(False)
    stage_avg = {k: v / st_calls for k, v in st_ms.items()} if st_calls else {}
    step_ms = [starts[i].elapsed_time(evs[i][3]) for i in range(args.steps)]
    kern_ms = [evs[i][1].elapsed_time(evs[i][2]) for i in range(args.steps)]
    prep_ms = [evs[i][0].elapsed_time(evs[i][1]) for i in range(args.steps)]
    t_step = sum(step_ms) / args.steps
    t_kern = sum(kern_ms) / args.steps
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([t_step, t_kern], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_kern = (float(x) for x in tt.cpu())
    mass = res.mass_kg()
    part = res.host_partials()
    executed_flop = 0.0
    if bufs is not None:  # tcgen05 FLOPs the tile kernel issued in the last step (diagnostic read-back)
        import ctypes as C

        from paper_2511_03126_b200.fused import _make_args

        fa = _make_args(pts, n, views, tables, cfg.temperature, cfg.eps, cfg.grid, bufs,
                        _lib.PF_FUSE_FEATURE_KERNEL if args.feature_kernel else 0)
        ex = C.c_double(0.0)
        _lib.call("pf_tile_executed_flops", C.byref(fa), C.addressof(ex), stream.cuda_stream)
        executed_flop = ex.value

    # ---- end to end through the public API, host buffers ---------------------------------------
    # paper_2511_03126_b200.stream.FusePipeline: every object's inputs are uploaded from pinned host
    # memory and its per-point properties + mass are read back, with the copies of neighbouring
    # objects overlapped with the compute (two device slots, H2D / compute / D2H streams).
    e2e = None
    if not args.no_e2e:
        from paper_2511_03126_b200.stream import FusePipeline, HostObject

        del bufs  # the pipeline holds its own two slots
        if world > 1:
            del shard_ops
        torch.cuda.empty_cache()
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        obj = HostObject(
            points=pin(pts_host), rotation=R, translation=tv, intrinsics=intr,
            depth=wl.depth.cpu().reshape(nv, cfg.image, cfg.image).pin_memory(),
            fmap=(torch.from_numpy(wl.fmaps.view(np.int16)).reshape(nv, *cfg.fmap).pin_memory() if cfg.bf16
                  else pin(wl.fmaps).reshape(nv, *cfg.fmap)),
            text=pin(wl.text), values=pin(wl.values.astype(np.float32)),
            mid_theta=pin(wl.mid_theta.astype(np.float32)))
        pipe = FusePipeline(n, nv, (cfg.image, cfg.image), cfg.fmap, bf16=cfg.bf16, k=cfg.k, p=tables.p,
                            grid=cfg.grid, temperature=cfg.temperature, epsilon=cfg.eps, device=dev,
                            sharded=world > 1)
        for _ in pipe.run([obj] * max(3, args.warmup)):
            pass
        torch.cuda.synchronize()
        barrier()
        ea, eb = mk(), mk()
        masses = [r.mass[0].item() for r in pipe.run([obj] * args.steps, events=(ea, eb))]
        torch.cuda.synchronize()
        t_e2e = ea.elapsed_time(eb) / args.steps
        if world > 1:
            import torch.distributed as dist

            tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        # one cold object: its upload, compute and download with nothing to overlap them (the
        # reference's per-run latency, pipeline.py:78-97); median of a few single-object runs
        cold = []
        for _ in range(3):
            ca, cb = mk(), mk()
            list(pipe.run([obj], events=(ca, cb)))
            torch.cuda.synchronize()
            cold.append(ca.elapsed_time(cb))
        t_cold = statistics.median(cold)
        if world > 1:
            import torch.distributed as dist

            tt = torch.tensor([t_cold], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_cold = float(tt.item())
        e2e = {"value": n_total * nv / (t_e2e * 1e-3), "unit": "samples/s", "ms_per_step": t_e2e,
               "h2d_bytes_per_step": int(pipe.h2d_bytes), "d2h_bytes_per_step": int(pipe.d2h_bytes),
               "api": "paper_2511_03126_b200.stream.FusePipeline: per-object throughput, the copies of "
                      "neighbouring objects overlap the compute",
               "latency_ms_per_object_cold": t_cold,
               "latency_note": "one object alone: H2D of its inputs + compute + D2H of its properties and mass, "
                               "nothing overlapped (median of 3, CUDA events on the copy streams)",
               "mass_kg_last": masses[-1]}

    if rank != 0:
        return
    # ---- roofline of the dominant kernel --------------------------------------------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_src = "measured"
    except Exception:
        peak_src = "fallback"
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # the tile kernel runs ~4 ms inside a ~7 ms step, not seconds back to back: the burst GEMM figure
    tc_peak = float(peaks.get("bf16_tflops", 1600.0))
    cells = nv * cfg.fmap[0] * cfg.fmap[1]
    kpad = 32 * ((cfg.k + 31) // 32)
    algo = algorithmic_bytes(cfg, n, nv, cfg.k, tables.p, cfg.d, 2 if cfg.bf16 else 4, cells, kpad)
    from paper_2511_03126_b200.build import source_hash

    build = source_hash()
    tile_path = bool(stage_avg) and stage_avg.get("tile_kernel", 0.0) > 0.0
    kname = ("k_tile_gram" if cfg.bf16 and not args.feature_kernel else "k_tile_ws") if tile_path else "k_fuse_simt"
    ncu = {}
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        ent = json.load(open(tf)).get(cfg.name, {})
        if ent.get("source_hash") == build and ent.get("kernel", "").startswith(kname):
            ncu = ent  # an ncu capture of this very build (profiles/summarize_ncu.py traffic)
    traffic = ncu.get("dram_bytes_per_launch")
    vis_pairs = part["visible_pairs"]
    # SURVEY §8d algorithmic FLOPs: bilinear gather 8*D per visible sample + similarity 2*N*D*K
    algo_flop = 8.0 * cfg.d * vis_pairs / max(1, world) + 2.0 * n * cfg.d * cfg.k
    if tile_path:
        t_dom = stage_avg["tile_kernel"]
        # frac: the tcgen05 FLOPs the kernel actually issued (Gram T T^T, W M~, W G per work item;
        # pf_tile_executed_flops) over its CUDA-event time, against the burst bf16 peak
        ach = executed_flop / (t_dom * 1e-3) / 1e12
        eff = algo_flop / (t_dom * 1e-3) / 1e12
        roofline = {"bound": "tensor", "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s",
                    "frac": ach / tc_peak, "traffic": traffic,
                    "peak_source": f"{peak_src} bf16_tflops (burst: the kernel is {t_dom:.2f} ms of a {t_step:.2f} ms step)",
                    "kernel": kname, "kernel_ms": t_dom, "executed_flop_per_launch": executed_flop,
                    # the SURVEY §8d algorithmic count (8 D per visible sample + 2 N D K) the formulation
                    # avoids most of (similarity through the G table, |F| through the Gram matrix)
                    "effective_frac": eff / tc_peak, "algorithmic_flop_per_launch": algo_flop,
                    "effective_note": "SURVEY 8d FLOPs / kernel time / peak: may exceed 1, the Gram formulation "
                                      "executes fewer FLOPs than the reference algorithm",
                    "kernel_scope": "the tile stage on its stream: work-list build + sort, the tcgen05 kernel, and "
                                    "(Gram path) the feature-product kernel over the split items",
                    "hbm": {"algorithmic_bytes_per_launch": algo,
                            "achieved_gbs": algo / (t_dom * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                            "frac": algo / (t_dom * 1e-3) / 1e9 / hbm_peak,
                            "step_frac": algo / (t_step * 1e-3) / 1e9 / hbm_peak},
                    "build": build}
        if ncu:
            roofline["tensor_pipe_active_ncu"] = ncu.get("tensor_pipe_active")
            roofline["ncu_source"] = ncu.get("source")
        else:
            roofline["traffic_note"] = "no ncu capture of this build in profiles/ncu_traffic.json"
    else:
        ach = algo / (t_kern * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ach / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                    "kernel": "k_fuse_simt", "kernel_ms": t_kern, "algorithmic_bytes_per_launch": algo,
                    "simt": {"fma_tflops": algo_flop / (t_kern * 1e-3) / 1e12,
                             "peak_tflops_nominal": SIMT_FP32_PEAK_TFLOPS}, "build": build}
    line = {
        "metric": "point-view samples/sec",
        "value": n_total * nv / (t_step * 1e-3),
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step,
        "latency_ms_per_object": t_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16" if tile_path else "f32",
        "data": "synthetic",
        "config": {**config_desc(cfg), "parallelism": (f"cell-range x{world} (points routed to voxel owners)"
                                                       if world > 1 else "single GPU"),
                   "l2": ("inputs larger than L2" if not flush else "L2 flushed between steps")},
        "stages_ms": {"fuse_query": t_kern, **{k: v for k, v in stage_avg.items()},
                      **({"prepare_G": sum(prep_ms) / args.steps} if args.serial_prepare or world > 1 else {}),
                      "rest(bbox,zero,voxel-mass,allreduce)": t_step - t_kern - sum(prep_ms) / args.steps},
        **({} if args.serial_prepare or world > 1 else
           {"prepare_G_note": "the per-object G table is built on a forked stream inside fuse_query, "
                              "concurrently with the sort and prep stages (no serial stage)"}),
        "roofline": roofline,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "result": {"mass_kg": mass, "featured": part["featured"], "visible_pairs": vis_pairs,
                   "visible_fraction": vis_pairs / (n_total * nv)},
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        sample = args.cpu_sample or default_cpu_sample(cfg)
        procs = cores_used()
        psample = min(cfg.n, sample * procs)
        dtp = cpu_oracle_parallel(wl, psample, procs)[0]
        line["cpu_baseline"] = {"value": psample * nv / dtp, "unit": "samples/s", "cores": procs,
                                "kind": "port",
                                "sample": f"first {psample} of {cfg.n} points x {nv} views, full path, point "
                                          f"chunks over {procs} processes (numba single-threaded per process)"}
        # parity of the measured full-object run (the last timed step's outputs, caller order) on a
        # stratified slice of its points, against the oracle with the full object's voxel domain
        stride = max(1, cfg.n // 250_000)
        idx = np.arange(0, n, stride)
        ref = cpu_oracle_rows(wl, idx, procs)
        cnt = res.counts.cpu().numpy()[idx]
        codes = res.codes.cpu().numpy()[idx]
        props = res.props.cpu().numpy()[idx].astype(np.float64)
        featured = ref["counts"] > 0
        rel = np.abs(props[featured, 0] - ref["props"][featured, 0]) / np.abs(ref["props"][featured, 0])
        line["parity_sample"] = {"points": int(idx.size), "of": int(n), "stride": int(stride),
                                 "counts_equal": bool(np.array_equal(cnt, ref["counts"])),
                                 "codes_equal": bool(np.array_equal(codes, ref["codes"])),
                                 "density_max_rel_err": float(rel.max()) if rel.size else 0.0,
                                 "density_mean_rel_err": float(rel.mean()) if rel.size else 0.0,
                                 "source": "the timed full-object step vs the CPU oracle on every "
                                           f"{stride}-th point (full-object voxel domain)"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def run_batch(args, cfg):
    """Config 4: B independent objects per step, sharded object-wise across ranks (no collective
    beyond the timing max). A step = batch.fuse_batch over this rank's objects (bbox, G table,
    fused pass, voxel mass per object; 2 streams)."""
    import torch

    rank, world, local = env_rank()
    dev_index, backend = device_and_backend(local)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_2511_03126_b200 as pf
    from paper_2511_03126_b200 import _lib, workloads
    from paper_2511_03126_b200.dist import shard_range

    b_total = cfg.objects
    o0, o1 = shard_range(b_total, rank, world)
    wls = [workloads.generate(cfg, seed=cfg.seed + 1000 + i, device_splat=True) for i in range(o0, o1)]
    nv = cfg.nviews
    views, tables, pts, hosts = [], [], [], []
    for wl in wls:
        R = np.stack([p.rotation for p in wl.poses])
        tv = np.stack([p.translation for p in wl.poses])
        intr = np.tile([wl.intrinsics.fx, wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy], (nv, 1))
        fm = torch.from_numpy(wl.fmaps).to(dev)
        views.append(pf.ViewSet.from_tensors(R, tv, intr, wl.depth.to(dev), fm, device=dev))
        tables.append(pf.QueryTables.build(wl.text, wl.values, wl.mid_theta, device=dev))
        pts.append(torch.from_numpy(wl.points).to(dev))
        hosts.append((R, tv, intr))
    kw = dict(temperature=cfg.temperature, epsilon=cfg.eps, grid=cfg.grid, streams=2)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    res, ws = pf.fuse_batch(pts, views, tables, **kw)
    for _ in range(args.warmup):
        res, ws = pf.fuse_batch(pts, views, tables, workspace=ws, **kw)
    torch.cuda.synchronize()
    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    clk = ClockSampler(dev_index)
    clk.start()
    t_soak = time.time()
    while time.time() - t_soak < 0.8:
        pf.fuse_batch(pts, views, tables, workspace=ws, **kw)
        torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    ev = [(mk(), mk()) for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record(stream)
        res, ws = pf.fuse_batch(pts, views, tables, workspace=ws, **kw)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    launches = _lib.launch_count() - launches0
    t_step = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([t_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    samples = b_total * cfg.n * nv
    masses = res.mass[:, 0].cpu().numpy()
    vis_pairs = float(res.partials[:, cfg.k + 5].sum().item())

    e2e = None
    if not args.no_e2e:
        from paper_2511_03126_b200.stream import FusePipeline, HostObject

        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        objs = [HostObject(points=pin(wl.points), rotation=R, translation=tv, intrinsics=intr,
                           depth=wl.depth.cpu().reshape(nv, cfg.image, cfg.image).pin_memory(),
                           fmap=pin(wl.fmaps).reshape(nv, *cfg.fmap), text=pin(wl.text),
                           values=pin(wl.values.astype(np.float32)), mid_theta=pin(wl.mid_theta.astype(np.float32)))
                for wl, (R, tv, intr) in zip(wls, hosts)]
        del ws
        torch.cuda.empty_cache()
        pipe = FusePipeline(cfg.n, nv, (cfg.image, cfg.image), cfg.fmap, bf16=cfg.bf16, k=cfg.k, p=2,
                            grid=cfg.grid, temperature=cfg.temperature, epsilon=cfg.eps, device=dev)
        for _ in pipe.run(objs[: max(3, min(len(objs), args.warmup))]):
            pass
        torch.cuda.synchronize()
        barrier()
        ea, eb = mk(), mk()
        reps = max(1, args.steps // 3)
        for _ in range(reps):
            list(pipe.run(objs, events=(ea, eb)))
        torch.cuda.synchronize()
        t_e2e = ea.elapsed_time(eb)  # the last repetition: one batch through the pipeline
        if world > 1:
            import torch.distributed as dist

            tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": samples / (t_e2e * 1e-3), "unit": "samples/s", "ms_per_step": t_e2e,
               "h2d_bytes_per_step": int(pipe.h2d_bytes) * len(objs), "d2h_bytes_per_step": int(pipe.d2h_bytes) * len(objs),
               "api": "paper_2511_03126_b200.stream.FusePipeline over this rank's objects"}
    if rank != 0:
        return
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_src = "measured"
    except Exception:
        peak_src = "fallback"
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    cells = nv * cfg.fmap[0] * cfg.fmap[1]
    kpad = 32 * ((cfg.k + 31) // 32)
    nloc = len(wls)
    algo = nloc * algorithmic_bytes(cfg, cfg.n, nv, cfg.k, 2, cfg.d, 4, cells, kpad)
    algo_flop = 8.0 * cfg.d * vis_pairs + 2.0 * nloc * cfg.n * cfg.d * cfg.k
    ach = algo / (t_step * 1e-3) / 1e9
    line = {
        "metric": "point-view samples/sec", "value": samples / (t_step * 1e-3), "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "latency_ms_per_object": t_step / max(1, nloc), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {**config_desc(cfg), "workload": f"c4: {b_total} objects x " + config_desc(cfg)["workload"][4:],
                   "objects": b_total, "parallelism": f"object-wise x{world} ({nloc} objects on rank 0)",
                   "l2": "inputs larger than L2 (64 objects, 3.2 GB of maps)"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                     "traffic": None, "peak_source": peak_src, "kernel": "batch step (k_fuse_simt dominant)",
                     "kernel_ms": t_step, "algorithmic_bytes_per_launch": algo,
                     "simt": {"fma_tflops": algo_flop / (t_step * 1e-3) / 1e12,
                              "peak_tflops_nominal": SIMT_FP32_PEAK_TFLOPS}},
        "gpu_launches": int(launches), "clocks": clocks,
        "result": {"mass_kg_first": float(masses[0]), "mass_kg_mean": float(masses.mean()),
                   "visible_fraction": vis_pairs / (nloc * cfg.n * nv)},
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        procs = cores_used()
        sample = min(cfg.n, (args.cpu_sample or default_cpu_sample(cfg)) * procs)
        dt = cpu_oracle_parallel(wls[0], sample, procs)[0]
        line["cpu_baseline"] = {"value": sample * nv / dt, "unit": "samples/s", "cores": procs, "kind": "port",
                                "sample": f"first {sample} points x {nv} views of object 0, point chunks over "
                                          f"{procs} processes"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_2511_03126_b200 import workloads

    cfg = workloads.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.objects > 1:
        run_batch(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
