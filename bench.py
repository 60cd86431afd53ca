#!/usr/bin/env python
"""bench.py — J^T W J p matvecs/s (and LM iterations/s) at 1M Gaussians on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
1M Gaussians (random_init state, SH-0: the reference supports only SH-0,
SURVEY §7 hard part 8), 200 ring cameras at 1280x720 (50 deg FOV, radius 3.2),
LM batch of 8 views drawn by the k-means view sampler, 32 stratified samples
per 16x16 tile.  One "step" = one J^T W J p + lambda p product over the 8-view
batch (SampledJacobian::gn_apply, jacobian.cpp:339-344) — the unit the
north-star roofline target is stated for.  At N ranks each rank owns 8 views
(weak scaling) and the product includes the per-CG-iteration NCCL allreduce.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line on rank 0.  The working set (records, tile lists,
tangents, ~1.5 GB) is far larger than the 126 MB L2, so no flush is needed
between timed iterations.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


METRIC = "JTWJp matvecs/s (8-view LM batch, 1M Gaussians)"
UNIT = "matvec/s"
KMEANS_SALT = 0x9E3779B97F4A7C15  # run.cpp:144


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--width", type=int, default=1280)
    ap.add_argument("--height", type=int, default=720)
    ap.add_argument("--batch", type=int, default=8, help="views per rank per LM batch (weak scaling)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: this many views per LM batch in total, split over the ranks")
    ap.add_argument("--spt", type=int, default=32, help="samples per tile")
    ap.add_argument("--lm-steps", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-psnr", action="store_true", help="skip the configs[0] time-to-PSNR run")
    ap.add_argument("--accumulate", default="ordered", choices=["ordered", "atomic"],
                    help="J^T / diag accumulation: fixed per-plan order (bitwise reproducible, default) "
                         "or float red.global.add")
    return ap.parse_args()


def parse_args_for(gaussians: int):
    """Default bench arguments (for tools/ drivers)."""
    saved = sys.argv
    sys.argv = [saved[0], "--gaussians", str(gaussians)]
    try:
        return parse()
    finally:
        sys.argv = saved


T0 = time.perf_counter()
DATA_TEXT = "synthetic (random_init state, ring cameras; BASELINE configs[2] shape)"
CFG0_TEXT = ("configs[0]: toy scene 5000 GT / 10k random_init Gaussians, 8 train + 4 test views 256x256, "
             "full pixels (N=256), PCG 8, 10 LM iterations")


def workload_config(args) -> dict:
    """The workload both arms run (identical dict for --impl b200 and reference)."""
    return {"workload": "configs[2]: 1M Gaussians (SH-0), 200 views 1280x720, 8-view LM batch per rank, "
                        "N=32 samples/tile, lambda=0.1",
            "gaussians": args.gaussians, "views": args.views, "width": args.width, "height": args.height,
            "batch_views_per_rank": args.batch, "samples_per_tile": args.spt,
            **({"global_batch_views": args.global_batch} if args.global_batch else {}),
            "l2": "working set > 126 MB L2 (no flush needed)"}


def lm_step_bytes(st: dict) -> int:
    """SURVEY 8(d) algorithmic bytes of one lm_step from its own counters
    (Lib.step_stats): k * B_matvec + B_diag + B_rhs + two full-image renders, with
    B_matvec = 4 (88 G + 19 E + 4 S), B_diag = 4 (68 G + 64 E + 4 S),
    B_rhs = 4 (51 G + 10 E + 4 S) (B_matvec without the Jv half) and a render
    4 (10 E + 8 W H)."""
    G, E, S, k, pix = st["valid"], st["entries"], st["samples"], st["pcg_iterations"], st["pixels"]
    matvec = 4 * (88 * G + 19 * E + 4 * S)
    diag = 4 * (68 * G + 64 * E + 4 * S)
    rhs = 4 * (51 * G + 10 * E + 4 * S)
    renders = 4 * (10 * E + 8 * pix) + 4 * (10 * st["entries_after"] + 8 * pix)
    return k * matvec + diag + rhs + renders


def log(msg: str) -> None:
    print(f"[bench {time.perf_counter() - T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def cameras(args):
    from paper_2504_12905_b200.types import ring_camera
    return [ring_camera(2.0 * math.pi * i / args.views, 3.2, 1.1, args.width, args.height)
            for i in range(args.views)]


def LmConfig(**kw):
    from paper_2504_12905_b200.types import LmConfig as _L
    return _L(**kw)


def rank_views(args, world) -> int:
    """Views per rank: --batch (weak scaling) or --global-batch / world (strong)."""
    if args.global_batch:
        if args.global_batch % world:
            raise SystemExit("--global-batch must be a multiple of the rank count")
        return args.global_batch // world
    return args.batch


def host_inputs(H, args, world):
    """Seeded exactly like train_run (run.cpp:126-167): random_init consumes the
    run RNG first, then the view batch and the sample plan draw from it."""
    rng = H.rng(1)
    state = H.random_init(args.gaussians, [-1, -1, -1], [1, 1, 1], rng)
    cams = cameras(args)
    clusters = H.kmeans_cameras(cams, rank_views(args, world) * world, 1 ^ KMEANS_SALT)
    batch = H.sample_view_batch(clusters, rng)
    plan = H.build_sample_plan([cams[i] for i in batch], args.spt, 0, rng, 32)
    return state, cams, clusters, batch, plan


def sub_plan(plan, lo: int, hi: int):
    from paper_2504_12905_b200.types import SamplePlan
    a, b = int(plan.view_offset[lo]), int(plan.view_offset[hi])
    return SamplePlan(np.arange(hi - lo, dtype=np.int32), plan.view_offset[lo:hi + 1] - a,
                      plan.px[a:b], plan.py[a:b], plan.tile[a:b], plan.weight[a:b], plan.samples_per_tile)


def gt_scene(count: int, seed: int = 20214, H=None):
    """Ground truth of the LM-step workload: io::generate_toy_scene's Gaussians
    (scene_gen.cpp:38-71, mt19937_64(seed), bit-exact) with the log-scales shifted
    by log(20/count)/3, i.e. scales x (20/count)^(1/3), so the scene keeps the toy
    scene's density (20 Gaussians) -- the toy scales at 500k Gaussians would cover
    every pixel with ~10^4 splats.  oracle/ref_bench.cpp builds the identical set
    with the reference's own generator for the CPU arm."""
    if H is None:
        from paper_2504_12905_b200 import splatlm
        H = splatlm.HostSampler()
    g = H.toy_gaussians(count, seed)
    shift = math.log(20.0 / count) / 3.0
    g.log_scales = g.log_scales + shift
    return g


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling during the timed region (NVML)."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k): k for k in dir(nv) if k.startswith("nvmlClocksThrottleReason") and
                 isinstance(getattr(nv, k), int)}
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if bit and mask & bit and name not in ("nvmlClocksThrottleReasonGpuIdle",
                                                           "nvmlClocksThrottleReasonAll",
                                                           "nvmlClocksThrottleReasonNone"):
                        self.reasons.add(name.replace("nvmlClocksThrottleReason", ""))
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the
    last committed `ncu --set full` capture (profiles/traffic.json, written by
    tools/summarize_profiles.py), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            return json.load(f)[kernel]["bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(stats: dict) -> dict:
    """B_matvec = 4 * sum_v (88 G_v + 19 E_v + 4 S_v) bytes; the fused
    raster's share is 4 * (19 E_v + 4 S_v) (index + value + tangent record per
    tile-list entry, packed pixel + weight + forward state per sample)."""
    G, E, S = stats["valid"], stats["entries"], stats["samples"]
    return {"matvec": 4 * (88 * G + 19 * E + 4 * S), "raster": 4 * (19 * E + 4 * S),
            "G_v_sum": G, "E_v_sum": E, "S_v_sum": S}


# ---------------------------------------------------------------------------- CPU
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")


def ref_bench(args, steps: int, warmup: int, lm_steps: int, psnr: bool, timeout: float = 1700.0) -> dict:
    """The UNMODIFIED reference timed on this host (oracle/ref_bench.cpp linked to the
    reference objects only): its own random_init / ring cameras / k-means batch /
    build_sample_plan draw the workload, SampledJacobian::gn_apply is timed over
    the whole view batch, solver::lm_step at the same shape, and the configs[0]
    toy run for time-to-PSNR.  All host threads.  Nothing of libslm_b200 is loaded."""
    import subprocess
    if not os.path.exists(REF_BENCH):
        raise FileNotFoundError(f"{REF_BENCH} not built (make -C oracle refbench, needs /root/reference)")
    cmd = [REF_BENCH, "--gaussians", args.gaussians, "--views", args.views, "--width", args.width,
           "--height", args.height, "--batch", args.batch, "--spt", args.spt, "--steps", steps,
           "--warmup", warmup, "--lm-steps", lm_steps, "--psnr", int(psnr)]
    out = subprocess.run([str(c) for c in cmd], capture_output=True, text=True, timeout=timeout, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def ref_time_to_psnr(r: dict):
    """configs[0] time-to-PSNR of the reference run inside ref_bench (same target as the
    GPU arm: the reference's own final test PSNR after 10 iterations - 0.05 dB)."""
    if not r.get("psnr_curve_db"):
        return None
    target = json.load(open(PSNR_TARGET))["psnr"][-1] - 0.05
    t, reached = 0.0, None
    for p, w in zip(r["psnr_curve_db"], r["psnr_wall_s"]):
        t += w
        if reached is None and p >= target:
            reached = t
    return {"config": CFG0_TEXT, "target_db": round(target, 4), "time_to_psnr_s": reached,
            "iterations": len(r["psnr_curve_db"]), "psnr_curve_db": [round(x, 4) for x in r["psnr_curve_db"]],
            "wall_per_iteration_s": r["psnr_wall_s"]}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    r = ref_bench(args, args.steps, args.warmup, 1 if args.lm_steps > 0 else 0, not args.no_psnr)
    value = 1.0 / r["gn_apply_mean_s"]
    lm = None
    if r["lm_step_s"]:
        lm = {"lm_iters_per_s": 1.0 / float(np.mean(r["lm_step_s"])), "ms_per_lm_step": 1000 * float(np.mean(r["lm_step_s"])),
              "pcg_iters": 8, "steps_timed": len(r["lm_step_s"])}
    sample = (f"SampledJacobian::gn_apply over the whole {args.batch}-view batch ({args.width}x{args.height}, "
              f"N={args.spt}, {args.gaussians} Gaussians): {args.steps} timed after {args.warmup} warm-up, "
              f"median {r['gn_apply_median_s']:.3f} s; inputs drawn by the reference itself")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * r["gn_apply_mean_s"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA_TEXT,
            "impl": "reference", "config": workload_config(args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["threads"], "kind": "reference",
                             "sample": sample, "cpu_model": r["cpu_model"], "nproc": r["nproc"],
                             "smt_active": r["smt_active"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "lm": lm, "time_to_psnr": ref_time_to_psnr(r),
            "reference": {"batch": r["batch"], "samples": r["samples"], "ctor_s": r["ctor_s"],
                          "gn_apply_s": r["gn_apply_s"], "lm_gt_render_s": r["lm_gt_render_s"], "total_s": r["total_s"]}}
    print(json.dumps(line), flush=True)


PSNR_TARGET = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden", "psnr_cfg0.json")


def cfg0_scene(L, c):
    """configs[0] as io::train_run builds the toy scene (run.cpp:26-36, scene_gen.cpp:38-86):
    ground truth from the reference's generator (bit-exact), ring cameras, images rendered here."""
    gt = L.toy_gaussians(c["toy_gaussians"], c["scene_seed"])
    train = [L.ring_camera(2.0 * math.pi * i / c["train"], 3.2, 1.1, c["size"]) for i in range(c["train"])]
    test = [L.ring_camera(0.37 + 2.0 * math.pi * i / c["test"], 3.2, 1.6, c["size"]) for i in range(c["test"])]
    # make_split (scene_gen.cpp:73-86): narrow(render_full(gt)), the FP64 render narrowed to f32
    timgs = [L.render_full(gt, cam)[0].astype(np.float32) for cam in train]
    simgs = [L.render_full(gt, cam)[0].astype(np.float32) for cam in test]
    return train, timgs, test, simgs


def psnr(a, b) -> float:  # metrics::psnr (image_metrics.cpp:108-119)
    m = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return 100.0 if m < 1e-10 else 10.0 * math.log10(1.0 / m)


def time_to_psnr(L, stream):
    """configs[0]: wall time of lm_step iterations until the mean test PSNR reaches the
    reference's final PSNR - 0.05 dB (tests/golden/psnr_cfg0.json, the reference itself
    run on the same inputs); evaluation renders are outside the timed region."""
    import torch
    from paper_2504_12905_b200 import splatlm

    ref = json.load(open(PSNR_TARGET))
    c = ref["config"]
    train, timgs, test, simgs = cfg0_scene(L, c)
    td = L.train_data(train, timgs)
    td.set_clusters(L.kmeans_cameras(train, min(c["batch"], len(train)), c["seed"] ^ KMEANS_SALT))
    rng = L.rng(c["seed"])
    scene = splatlm.Scene(L, L.random_init(c["gaussians"], [-1, -1, -1], [1, 1, 1], rng))
    cfg = LmConfig(pcg_iters_initial=c["pcg"], pcg_iters_late=c["pcg"], batch_size_initial=c["batch"],
                   batch_size_late=c["batch"], samples_per_tile=c["spt"])
    target = ref["psnr"][-1] - 0.05
    sd = L.train_data(test, simgs)
    with torch.cuda.stream(stream):  # one untimed pass of the same run: buffers sized, caches warm
        wrng = L.rng(c["seed"])
        wscene = splatlm.Scene(L, L.random_init(c["gaussians"], [-1, -1, -1], [1, 1, 1], wrng))
        for it in range(len(ref["psnr"])):
            wscene.lm_step(td, cfg, it, wrng)
        torch.cuda.synchronize()
        del wscene
    elapsed, reached, curve, ssim_curve, nbytes, bytes_at = 0.0, None, [], [], 0, None
    with torch.cuda.stream(stream):
        for it in range(len(ref["psnr"])):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            scene.lm_step(td, cfg, it, rng)
            torch.cuda.synchronize()
            elapsed += time.perf_counter() - t0
            nbytes += lm_step_bytes(L.step_stats())
            ev = scene.evaluate_split(sd)  # io::evaluate_split on the device
            curve.append(ev.psnr)
            ssim_curve.append(ev.ssim)
            if reached is None and curve[-1] >= target:
                reached, bytes_at = elapsed, nbytes
    peak, _ = measured_peaks()
    roof = None
    if reached:  # algorithmic bytes of the steps until the target / the time they took
        ach = bytes_at / reached / 1e9
        roof = {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "bytes": bytes_at,
                "roofline_time_s": bytes_at / (peak * 1e9)}
    return {"config": CFG0_TEXT,
            "target_db": round(target, 4), "time_to_psnr_s": reached, "iterations": len(curve),
            "psnr_curve_db": [round(x, 4) for x in curve],
            "ssim_curve": [round(x, 5) for x in ssim_curve],
            "max_abs_psnr_diff_vs_reference_db": round(max(abs(a - b) for a, b in zip(curve, ref["psnr"])), 5),
            "roofline": roof}


# ---------------------------------------------------------------------------- B200
def run_b200(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        # NCCL's init lines (rank, nRanks, transport) stay on stderr for the driver's rank check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            import nvidia.nccl
            os.environ.setdefault("SLM_NCCL_LIB", os.path.join(os.path.dirname(nvidia.nccl.__file__), "lib",
                                                               "libnccl.so.2"))
        except Exception:
            pass
    from paper_2504_12905_b200 import splatlm
    L = splatlm.Lib(local)
    L.set_deterministic(args.accumulate == "ordered")
    stream = torch.cuda.Stream()
    L.set_stream(stream.cuda_stream)
    if world > 1:
        uid = splatlm.Lib.nccl_unique_id(L.dll) if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        L.init_comm(obj[0], rank, world)

    t_setup = time.perf_counter()
    state, cams, clusters, batch, plan = host_inputs(L, args, world)
    log(f"host inputs: G={args.gaussians}, batch={batch}, samples={plan.total_samples()}")
    nv = rank_views(args, world)
    lo, hi = rank * nv, (rank + 1) * nv
    scene = splatlm.Scene(L, state)
    # Global N_total weights, this rank's views: slice the plan but keep weights
    # relative to the whole batch (the solver's allreduce sums the slices).
    my_plan = sub_plan(plan, lo, hi)
    jac = scene.jacobian([cams[i] for i in batch[lo:hi]], my_plan)
    stats = jac.stats()
    log(f"jacobian ready: {stats}")
    P = 14 * scene.padded
    p = torch.empty(P, device="cuda", dtype=torch.float32).uniform_(-1, 1)
    u = torch.zeros(P, device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    def product():
        jac.gn_apply_dev(0.1, p.data_ptr(), u.data_ptr())

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            product()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = L.launch_count()
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            start.record(stream)
            for _ in range(args.steps):
                product()
            end.record(stream)
        torch.cuda.synchronize()
    launches = L.launch_count() - launches0
    ms = start.elapsed_time(end)
    log(f"timed {args.steps} products: {ms / args.steps:.3f} ms each")
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_per_step = ms / args.steps
    # in units of 8-view products: weak = one per rank per step, strong = global batch / 8
    units = world * nv / 8.0
    value = units * args.steps / (ms / 1000.0)

    # per-kernel breakdown of the product (CUDA events around each kernel)
    L.set_profiling(True)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            product()
    prof = L.profile_collect()
    L.set_profiling(False)
    log(f"profile: {prof}")
    n = max(prof["n"], 1)
    raster_ms = prof["raster_ms"] / n
    bytes_ = algorithmic_bytes(stats)
    peak, peak_src = measured_peaks()
    achieved = bytes_["raster"] / (raster_ms / 1000.0) / 1e9
    matvec_achieved = bytes_["matvec"] / (ms_per_step / 1000.0) / 1e9

    # e2e through the drop-in host API (SampledJacobian::gn_apply on host f64 vectors)
    host_jac = L.jacobian(state, [cams[i] for i in batch[lo:hi]], my_plan)
    # host ParamVectors in pinned memory (the e2e contract's host buffers)
    ph = torch.empty(host_jac.param_dim(), dtype=torch.float64, pin_memory=True).numpy()
    ph[:] = np.random.default_rng(0).uniform(-1, 1, host_jac.param_dim())
    oh = torch.empty(host_jac.param_dim(), dtype=torch.float64, pin_memory=True).numpy()
    host_jac.gn_apply(0.1, ph, out=oh)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        host_jac.gn_apply(0.1, ph, out=oh)
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    del host_jac
    e2e_value = units / e2e_s
    log(f"e2e host gn_apply: {e2e_s * 1000:.1f} ms")

    # LM iterations/s on the device-resident scene (lm_step, lm.cpp:56-157)
    lm = None
    if args.lm_steps > 0:
        gt = splatlm.Scene(L, gt_scene(args.gaussians // 2, H=L))
        imgs = [gt.render(c)[0] for c in cams]
        del gt
        log("ground truth rendered")
        td = L.train_data(cams, imgs)
        del imgs
        td.set_clusters(clusters)
        lm_scene = splatlm.Scene(L, state)
        cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, batch_size_initial=nv * world,
                       batch_size_late=nv * world, samples_per_tile=args.spt)
        rng = L.rng(1)
        L.random_init(args.gaussians, [-1, -1, -1], [1, 1, 1], rng)  # same stream position as train_run
        L.set_timing(True)
        with torch.cuda.stream(stream):
            # two untimed steps: the first fills the pinned host buffers and
            # starts the speculative plan of the next step (lm_step's steady state)
            rep = lm_scene.lm_step(td, cfg, 0, rng)
            lm_scene.lm_step(td, cfg, 1, rng)
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            reps, lm_bytes = [], 0
            for i in range(args.lm_steps):
                reps.append(lm_scene.lm_step(td, cfg, 2 + i, rng))
                lm_bytes += lm_step_bytes(L.step_stats())
            e1.record(stream)
        torch.cuda.synchronize()
        lm_ms = e0.elapsed_time(e1) / args.lm_steps
        if dist:
            t = torch.tensor([lm_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            lm_ms = float(t.item())
        log(f"lm_step: {lm_ms:.1f} ms/step, stages {L.timings()}")
        peak, _ = measured_peaks()
        step_bytes = lm_bytes / args.lm_steps  # this rank's views
        ach = step_bytes / (lm_ms / 1000.0) / 1e9
        lm = {"lm_iters_per_s": 1000.0 / lm_ms, "ms_per_lm_step": lm_ms, "pcg_iters": 8,
              "loss_before_first": rep.loss_before, "loss_after_last": reps[-1].loss_after,
              "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                           "bytes_per_step": step_bytes, "roofline_lm_iters_per_s": peak * 1e9 / step_bytes,
                           "formula": "k*B_matvec + B_diag + B_rhs + 2 renders (SURVEY 8d), counted per step"}}

    ttp = None
    if not args.no_psnr and os.path.exists(PSNR_TARGET):
        ttp = time_to_psnr(L, stream)
        log(f"time-to-PSNR: {ttp['time_to_psnr_s']} s (target {ttp['target_db']} dB, "
            f"max |dPSNR| vs reference {ttp['max_abs_psnr_diff_vs_reference_db']} dB)")

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline:
        try:
            log("cpu baseline (oracle/_ref/ref_bench)")
            r = ref_bench(args, 2, 1, 0, False, timeout=600)
            cval = 1.0 / r["gn_apply_mean_s"]
            log(f"cpu baseline: {cval:.4f} matvec/s (reference, {r['threads']} threads)")
            cpu = {"value": cval, "unit": UNIT, "cores": r["threads"], "kind": "reference",
                   "sample": f"SampledJacobian::gn_apply over the whole {args.batch}-view batch, 2 timed after "
                             f"1 warm-up ({r['gn_apply_s']} s), inputs drawn by the reference itself",
                   "cpu_model": r["cpu_model"], "nproc": r["nproc"], "smt_active": r["smt_active"]}
        except Exception as e:  # the checker is optional on a box without the build
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": f"{type(e).__name__}: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if args.global_batch else "weak", "vs_baseline": None,
        "dtype": "f32 (raster, linearisation, CG vectors; f64 projection, blend decisions and parameters)",
        "data": DATA_TEXT,
        "config": workload_config(args),
        "parallelism": f"view-sharded x{world}, NCCL allreduce per product" if world > 1 else "1 GPU",
        "accumulation": args.accumulate,
        "roofline": {"bound": "hbm", "kernel": "k_sample_raster<GN> (fused Jv -> W -> J^T)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic("k_sample_raster<2>"), "algorithmic_bytes_per_launch": bytes_["raster"],
                     "avg_launch_ms": raster_ms, "peak_source": peak_src},
        "matvec_roofline": {"achieved": matvec_achieved, "peak": peak, "unit": "GB/s",
                            "frac": matvec_achieved / peak, "bytes_per_matvec": bytes_["matvec"],
                            "roofline_matvecs_per_s": peak * 1e9 / bytes_["matvec"] * units,
                            **{k: bytes_[k] for k in ("G_v_sum", "E_v_sum", "S_v_sum")}},
        "breakdown_ms": {"tangents": prof["tangents_ms"] / n, "raster": raster_ms, "chain": prof["chain_ms"] / n},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * 14 * args.gaussians,
                "d2h_bytes_per_step": 8 * 14 * args.gaussians,
                "path": "slm_jacobian_gn_apply (host f64 ParamVector in/out, pinned host buffers)"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "lm": lm,
        "time_to_psnr": ttp,
        "setup_s": round(setup_s, 1),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
