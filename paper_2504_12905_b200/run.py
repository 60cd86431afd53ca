"""The run driver around the B200 path: io::train_run / io::eval_run
(io/run.hpp:14-54, io/run.cpp:16-230) for the toy scene.

The optimizer steps, renders and evaluations all run on the device through
libslm_b200.so; this module only orchestrates and writes the reference's wire
formats byte for byte:

* ``metrics.csv`` — header ``iter,wall_ms,train_loss,test_psnr,test_ssim,eta,
  pcg_iters,breakdown`` (run.hpp:33-37), doubles as ``%.17g``, wall time as
  ``%.3f``, empty fields where not applicable and ``wall_ms`` empty in
  deterministic mode (run.cpp:54-75);
* ``checkpoint.bin`` (+ ``.meta.txt``) — ``SPLMGS01`` (checkpoint.cpp:12-66),
  written by ``slm_save_checkpoint``;
* ``summary.json`` / ``eval.json`` — nlohmann ``dump(2)`` layout: keys sorted,
  two-space indent, shortest round-trip doubles (run.cpp:106-118,197-212).

Dataset directories (NeRF-synthetic PNG + JSON) and the PNG test renders are
out of scope (no libpng on the path); ``scene`` must be ``"toy"``.
"""
from __future__ import annotations

import json

import numpy as np
import math
import os
import time
from dataclasses import dataclass, field

from .types import (FO_ADAM, FO_RMSPROP, FO_SGD_MOMENTUM, LOSS_MSE_SSIM, FirstOrderConfig, LmConfig,
                    MetricReport)

METRICS_CSV_HEADER = "iter,wall_ms,train_loss,test_psnr,test_ssim,eta,pcg_iters,breakdown"
KMEANS_SALT = 0x9E3779B97F4A7C15
_DIST_NAMES = {0: "uniform", 1: "residual", 2: "gaussian"}  # sample_plan.cpp:10-17


@dataclass
class ToySceneConfig:
    """io::ToySceneConfig (scene_gen.hpp:18-23)."""
    gaussians: int = 20
    train_cameras: int = 8
    test_cameras: int = 4
    image_size: int = 64


@dataclass
class RunConfig:
    """io::RunConfig (run.hpp:14-31)."""
    scene: str = "toy"
    optimizer: str = "lm"  # lm | adam | rmsprop | sgd
    iterations: int = 200
    seed: int = 1
    out_dir: str = ""
    gaussians: int = 0  # 0 -> 2 x toy.gaussians
    lm: LmConfig = field(default_factory=LmConfig)
    first_order: FirstOrderConfig = field(default_factory=FirstOrderConfig)
    eval_every: int = 50
    deterministic: bool = False
    scene_seed: int = 20214
    toy: ToySceneConfig = field(default_factory=ToySceneConfig)


@dataclass
class TrainResult:
    """io::TrainResult (run.hpp:39-44)."""
    final_train_loss: float = 0.0
    final_test: MetricReport = field(default_factory=MetricReport)
    checkpoint: str = ""
    metrics_csv: str = ""


def _fmt(v: float, spec: str = "%.17g") -> str:  # run.cpp:54-58
    return spec % v


def _json_dump(obj: dict) -> str:
    """nlohmann::json::dump(2) of a flat object: sorted keys, shortest round-trip doubles."""
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


def toy_scene(L, cfg: RunConfig):
    """io::generate_toy_scene (scene_gen.cpp:38-86): ground truth drawn bit-exactly by the
    library (slm_toy_gaussians), ring cameras, images rendered on the device."""
    from .splatlm import Scene

    t = cfg.toy
    gt = L.toy_gaussians(t.gaussians, cfg.scene_seed)
    train = [L.ring_camera(0.0 + 2.0 * math.pi * i / t.train_cameras, 3.2, 1.1, t.image_size)
             for i in range(t.train_cameras)]
    test = [L.ring_camera(0.37 + 2.0 * math.pi * i / t.test_cameras, 3.2, 1.6, t.image_size)
            for i in range(t.test_cameras)]
    # make_split (scene_gen.cpp:73-86): narrow(render_full(gt)) -- the FP64 drop-in render narrowed to f32
    return (train, [L.render_full(gt, c)[0].astype(np.float32) for c in train], test,
            [L.render_full(gt, c)[0].astype(np.float32) for c in test])


def _config_json(cfg: RunConfig) -> dict:  # run.cpp:106-118
    return {"scene": cfg.scene, "optimizer": cfg.optimizer, "iterations": cfg.iterations, "seed": cfg.seed,
            "gaussians": cfg.gaussians, "samples_per_tile": cfg.lm.samples_per_tile, "damping": cfg.lm.damping,
            "residual_dist": _DIST_NAMES.get(cfg.lm.dist, "unknown"),
            "loss": "mse+ssim" if cfg.lm.loss == LOSS_MSE_SSIM else "mse", "deterministic": cfg.deterministic}


def train_run(L, cfg: RunConfig) -> TrainResult:
    """io::train_run (run.cpp:120-212) with every step on the device."""
    from dataclasses import replace

    from .splatlm import FirstOrder, Scene

    if cfg.iterations < 1:
        raise ValueError("iteration budget must be at least 1")
    if cfg.scene != "toy":
        raise ValueError("only the toy scene is supported (dataset I/O is out of scope)")
    os.makedirs(cfg.out_dir, exist_ok=True)
    train, timgs, test, simgs = toy_scene(L, cfg)
    rng = L.rng(cfg.seed)
    count = cfg.gaussians if cfg.gaussians > 0 else 2 * cfg.toy.gaussians
    state = Scene(L, L.random_init(count, [-1.0, -1.0, -1.0], [1.0, 1.0, 1.0], rng))
    data = L.train_data(train, timgs)
    split = L.train_data(test, simgs) if test else None

    is_lm = cfg.optimizer == "lm"
    kinds = {"adam": FO_ADAM, "rmsprop": FO_RMSPROP, "sgd": FO_SGD_MOMENTUM}
    if not is_lm and cfg.optimizer not in kinds:
        raise ValueError(f"unknown optimizer: {cfg.optimizer}")
    fo_cfg = replace(cfg.first_order, kind=kinds.get(cfg.optimizer, cfg.first_order.kind))
    if fo_cfg.decay_iterations == 0:
        fo_cfg.decay_iterations = cfg.iterations
    fo = None if is_lm else FirstOrder(L, state)
    cluster_k, cluster_seed = 0, cfg.seed ^ KMEANS_SALT

    result = TrainResult(metrics_csv=os.path.join(cfg.out_dir, "metrics.csv"))
    train_loss = 0.0
    with open(result.metrics_csv, "w", newline="") as csv:
        csv.write(METRICS_CSV_HEADER + "\n")
        for it in range(cfg.iterations):
            t0 = time.perf_counter()
            eta = pcg = brk = ""
            if is_lm:
                k = min(cfg.lm.batch_size_at(it), len(train))
                if k != cluster_k:  # run.cpp:145-153
                    data.rebuild_clusters(k, cluster_seed)
                    cluster_k = k
                rep = state.lm_step(data, cfg.lm, it, rng)
                train_loss = rep.loss_after
                eta, pcg, brk = _fmt(rep.eta), str(rep.pcg_iterations), "1" if rep.breakdown else "0"
            else:
                train_loss = fo.step(data, fo_cfg)
            wall_ms = (time.perf_counter() - t0) * 1000.0
            psnr = ssim = ""
            if split is not None and (it == cfg.iterations - 1 or
                                      (cfg.eval_every > 0 and (it + 1) % cfg.eval_every == 0)):
                rep_t = state.evaluate_split(split)
                psnr, ssim = _fmt(rep_t.psnr), _fmt(rep_t.ssim)
                result.final_test = rep_t
            wall = "" if cfg.deterministic else _fmt(wall_ms, "%.3f")
            csv.write(f"{it},{wall},{_fmt(train_loss)},{psnr},{ssim},{eta},{pcg},{brk}\n")
    result.final_train_loss = train_loss
    result.checkpoint = os.path.join(cfg.out_dir, "checkpoint.bin")
    L.save_checkpoint(result.checkpoint, state.download())
    summary = _config_json(cfg)
    summary["final_train_loss"] = result.final_train_loss
    if split is not None:
        summary["test_mse"] = result.final_test.mse
        summary["test_psnr"] = result.final_test.psnr
        summary["test_ssim"] = result.final_test.ssim
    with open(os.path.join(cfg.out_dir, "summary.json"), "w") as f:
        f.write(_json_dump(summary))
    return result


def eval_run(L, cfg: RunConfig, checkpoint: str) -> MetricReport:
    """io::eval_run (run.cpp:212-230): evaluate a checkpoint on the test split (train if none)."""
    from .splatlm import Scene

    train, timgs, test, simgs = toy_scene(L, cfg)
    name, cams, imgs = ("test", test, simgs) if test else ("train", train, timgs)
    report = Scene(L, L.load_checkpoint(checkpoint)).evaluate_split(L.train_data(cams, imgs))
    if cfg.out_dir:
        os.makedirs(cfg.out_dir, exist_ok=True)
        with open(os.path.join(cfg.out_dir, "eval.json"), "w") as f:
            f.write(_json_dump({"checkpoint": checkpoint, "split": name, "mse": report.mse,
                                "psnr": report.psnr, "ssim": report.ssim}))
    return report
