"""ctypes binding shared by the two CPU checkers — TEST INFRASTRUCTURE ONLY.

``oracle/_ref/libsplatlm_ref.so`` (prefix ``ref_``, the real reference behind
``oracle/ref_capi.cpp``) and ``oracle/liboracle.so`` (prefix ``orc_``, the C
restatement ``oracle/splat_oracle.c``) export the same entry points, so one
Python class drives either.  The method names follow the reference API
(render::bin_and_sort, SampledJacobian::gn_apply, solver::lm_step, ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2504_12905_b200.types import (CCamera, CFirstOrderConfig, CGaussians, CLmConfig, CPcgResult, CPlan,
                                         CStepReport, Camera, GaussianSet, LmConfig,
                                         PcgResult, SamplePlan, StepReport, cameras_to_c,
                                         f32ptr, f64ptr, i32ptr, i64ptr)

from . import PORT_SO, REF_SO

_vp = C.c_void_p
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)


class CpuError(RuntimeError):
    pass


class CpuLib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.p = prefix
        self.kind = "reference" if prefix == "ref_" else "port"
        sig = {
            "last_error": (C.c_char_p, []),
            "set_threads": (None, [C.c_int]),
            "threads": (C.c_int, []),
            "rng_new": (_vp, [C.c_uint64]),
            "rng_free": (None, [_vp]),
            "rng_next": (C.c_uint64, [_vp]),
            "random_init": (C.c_int, [C.c_int, _f64p, _f64p, _vp, C.POINTER(CGaussians)]),
            "ring_camera": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int,
                                      C.POINTER(CCamera)]),
            "toy_scene": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                    C.POINTER(CGaussians), C.POINTER(CCamera),
                                    C.POINTER(C.c_float)]),
            "prepare": (C.c_int, [C.POINTER(CGaussians), C.POINTER(CCamera), _f64p, _f64p, _f64p,
                                  _f64p, _f64p, _f64p, _i32p]),
            "bin_and_sort": (C.c_int, [C.POINTER(CGaussians), C.POINTER(CCamera), _i32p, _i32p,
                                       C.c_int64, C.POINTER(C.c_int64)]),
            "render_full": (C.c_int, [C.POINTER(CGaussians), C.POINTER(CCamera), _f64p, _f64p,
                                      _i32p]),
            "build_sample_plan": (_vp, [C.POINTER(CCamera), C.c_int, C.c_int, C.c_int, C.c_int,
                                        _vp, C.POINTER(_f64p), C.POINTER(_i32p),
                                        C.POINTER(_f64p)]),
            "exhaustive_plan": (_vp, [C.POINTER(CCamera), C.c_int]),
            "plan_free": (None, [_vp]),
            "plan_views": (C.c_int, [_vp]),
            "plan_total": (C.c_int64, [_vp]),
            "plan_export": (None, [_vp, _i32p, C.POINTER(C.c_int64), _i32p, _i32p, _i32p,
                                   _f64p]),
            "estimate_loss": (C.c_int, [C.POINTER(CCamera), C.POINTER(CPlan), C.POINTER(_f64p),
                                        _f64p]),
            "kmeans_cameras": (C.c_int, [C.POINTER(CCamera), C.c_int, C.c_int, C.c_uint64,
                                         _i32p]),
            "camera_features": (C.c_int, [C.POINTER(CCamera), C.c_int, _f64p]),
            "jac_new": (_vp, [C.POINTER(CGaussians), C.POINTER(CCamera), C.c_int,
                              C.POINTER(CPlan)]),
            "jac_free": (None, [_vp]),
            "jac_residual_dim": (C.c_int64, [_vp]),
            "jac_param_dim": (C.c_int64, [_vp]),
            "jac_jvp": (C.c_int, [_vp, _f64p, _f64p]),
            "jac_vjp": (C.c_int, [_vp, _f64p, _f64p]),
            "jac_jtj_diag": (C.c_int, [_vp, _f64p]),
            "jac_gn_apply": (C.c_int, [_vp, C.c_double, _f64p, _f64p]),
            "jac_weights": (C.c_int, [_vp, _f64p]),
            "jac_set_weights": (C.c_int, [_vp, _f64p]),
            "jac_pcg": (C.c_int, [_vp, C.c_double, _f64p, _f64p, C.c_int, _f64p,
                                  C.POINTER(CPcgResult)]),
            "pcg_dense": (C.c_int, [_f64p, C.c_int, _f64p, _f64p, C.c_int, _f64p,
                                    C.POINTER(CPcgResult)]),
            "learning_rate": (C.c_double, [_f64p, C.c_int64, C.c_int, C.POINTER(CLmConfig)]),
            "apply_update": (C.c_int, [C.POINTER(CGaussians), _f64p, C.c_double]),
            "train_new": (_vp, [C.POINTER(CCamera), C.c_int, C.POINTER(C.c_float)]),
            "train_new_f64": (_vp, [C.POINTER(CCamera), C.c_int, _f64p]),
            "train_free": (None, [_vp]),
            "train_rebuild_clusters": (C.c_int, [_vp, C.c_int, C.c_uint64]),
            "train_set_clusters": (C.c_int, [_vp, _i32p, C.c_int, C.c_int]),
            "lm_step": (C.c_int, [C.POINTER(CGaussians), _vp, C.POINTER(CLmConfig), C.c_int, _vp,
                                  C.POINTER(CStepReport)]),
            "batch_loss": (C.c_int, [C.POINTER(CGaussians), C.POINTER(CCamera), C.c_int,
                                     C.POINTER(C.c_float), C.c_int, C.c_double, _f64p]),
            "mse": (C.c_double, [_f64p, _f64p, C.c_int, C.c_int]),
            "psnr": (C.c_double, [_f64p, _f64p, C.c_int, C.c_int]),
            "ssim": (C.c_double, [_f64p, _f64p, C.c_int, C.c_int]),
            "full_gradient": (C.c_int, [C.POINTER(CGaussians), C.POINTER(CCamera), C.c_int,
                                        C.POINTER(C.c_float), C.c_int, C.c_double, _f64p]),
            "first_order_step": (C.c_int, [C.POINTER(CGaussians), _f64p, _f64p, C.POINTER(C.c_int64),
                                           _f64p, C.POINTER(CFirstOrderConfig)]),
            "ssim_diag_residuals": (None, [_f64p, _f64p, C.c_int, C.c_int, _f64p, _f64p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, "_" + name, fn)
        if hasattr(self.lib, prefix + "sample_view_batch"):  # the reference library only
            fn = getattr(self.lib, prefix + "sample_view_batch")
            fn.restype = C.c_int
            fn.argtypes = [_i32p, C.c_int, C.c_int, _vp, _i32p]
            self._sample_view_batch = fn

    # ---- helpers ----
    def _check(self, rc: int):
        if rc != 0:
            msg = self._last_error().decode()
            exc = {1: ValueError, 2: ArithmeticError, 3: RuntimeError}.get(rc, CpuError)
            raise exc(msg)

    def set_threads(self, n: int) -> None:
        self._set_threads(int(n))

    # ---- RNG ----
    def rng(self, seed: int) -> "Rng":
        return Rng(self, seed)

    # ---- io helpers (harness) ----
    def random_init(self, count: int, cube_min, cube_max, rng: "Rng") -> GaussianSet:
        g = GaussianSet(count)
        lo = np.asarray(cube_min, np.float64)
        hi = np.asarray(cube_max, np.float64)
        cg = g.to_c()
        self._check(self._random_init(count, f64ptr(lo), f64ptr(hi), rng.h, C.byref(cg)))
        return g

    def ring_camera(self, angle, radius, height, size) -> Camera:
        c = CCamera()
        self._check(self._ring_camera(angle, radius, height, size, C.byref(c)))
        return Camera.from_c(c)

    def toy_scene(self, gaussians=20, train_cameras=8, test_cameras=4, image_size=64, seed=20214):
        """io::generate_toy_scene -> (gt, train_cams, train_imgs f32, test_cams, test_imgs)."""
        g = GaussianSet(gaussians)
        n = train_cameras + test_cameras
        cams = (CCamera * n)()
        imgs = np.zeros((n, image_size, image_size, 3), np.float32)
        cg = g.to_c()
        self._check(self._toy_scene(gaussians, train_cameras, test_cameras, image_size, seed,
                                    C.byref(cg), cams, f32ptr(imgs)))
        cl = [Camera.from_c(cams[i]) for i in range(n)]
        return g, cl[:train_cameras], imgs[:train_cameras], cl[train_cameras:], imgs[train_cameras:]

    # ---- render ----
    def prepare(self, g: GaussianSet, cam: Camera) -> dict:
        n = g.count
        out = dict(mean2d=np.zeros(2 * n), conic=np.zeros(3 * n), opacity=np.zeros(n),
                   color=np.zeros(3 * n), depth=np.zeros(n), radius=np.zeros(n),
                   valid=np.zeros(n, np.int32))
        cg, cc = g.to_c(), cam.to_c()
        self._check(self._prepare(C.byref(cg), C.byref(cc), *(f64ptr(out[k]) for k in
                                  ("mean2d", "conic", "opacity", "color", "depth", "radius")),
                                  i32ptr(out["valid"])))
        return out

    def bin_and_sort(self, g: GaussianSet, cam: Camera):
        """render::bin_and_sort -> (offsets[T+1], indices[E]) (CSR tile lists)."""
        tiles = cam.tiles_x * cam.tiles_y
        offsets = np.zeros(tiles + 1, np.int32)
        cap = max(16, 4 * g.count)
        cg, cc = g.to_c(), cam.to_c()
        while True:
            idx = np.zeros(cap, np.int32)
            n = C.c_int64()
            self._check(self._bin_and_sort(C.byref(cg), C.byref(cc), i32ptr(offsets), i32ptr(idx),
                                           cap, C.byref(n)))
            if n.value <= cap:
                return offsets, idx[:n.value].copy()
            cap = n.value

    def render_full(self, g: GaussianSet, cam: Camera):
        """render::render_full -> (image[H,W,3], transmittance[H,W], contrib[H,W])."""
        img = np.zeros((cam.height, cam.width, 3))
        tr = np.zeros((cam.height, cam.width))
        cn = np.zeros((cam.height, cam.width), np.int32)
        cg, cc = g.to_c(), cam.to_c()
        self._check(self._render_full(C.byref(cg), C.byref(cc), f64ptr(img), f64ptr(tr), i32ptr(cn)))
        return img, tr, cn

    # ---- sampling ----
    def _export_plan(self, h) -> SamplePlan:
        if not h:
            raise ValueError(self._last_error().decode())
        try:
            nv = self._plan_views(h)
            tot = self._plan_total(h)
            vc = np.zeros(nv, np.int32)
            vo = np.zeros(nv + 1, np.int64)
            px, py, tl = (np.zeros(tot, np.int32) for _ in range(3))
            w = np.zeros(tot)
            self._plan_export(h, i32ptr(vc), vo.ctypes.data_as(C.POINTER(C.c_int64)), i32ptr(px),
                              i32ptr(py), i32ptr(tl), f64ptr(w))
            return SamplePlan(vc, vo, px, py, tl, w)
        finally:
            self._plan_free(h)

    def build_sample_plan(self, cams, samples_per_tile, dist, rng: "Rng", lane_width=32,
                          aux=None) -> SamplePlan:
        """sampling::build_sample_plan; aux = [(image[H,W,3], contrib[H,W], gt[H,W,3] | None)]."""
        cc = cameras_to_c(cams)
        ai = ac = ag = None
        keep = []
        if aux is not None:
            ai = (_f64p * len(aux))()
            ac = (_i32p * len(aux))()
            ag = (_f64p * len(aux))()
            for i, (im, cn, gt) in enumerate(aux):
                im = np.ascontiguousarray(im, np.float64)
                cn = np.ascontiguousarray(cn, np.int32)
                gt = np.ascontiguousarray(gt if gt is not None else np.zeros_like(im), np.float64)
                keep += [im, cn, gt]
                ai[i], ac[i], ag[i] = f64ptr(im), i32ptr(cn), f64ptr(gt)
        h = self._build_sample_plan(cc, len(cams), samples_per_tile, dist, lane_width, rng.h,
                                    ai, ac, ag)
        plan = self._export_plan(h)
        plan.samples_per_tile, plan.dist = samples_per_tile, dist
        return plan

    def exhaustive_plan(self, cams) -> SamplePlan:
        plan = self._export_plan(self._exhaustive_plan(cameras_to_c(cams), len(cams)))
        plan.samples_per_tile = 256
        return plan

    def estimate_loss(self, cams, plan: SamplePlan, residual_fields) -> float:
        arr = (_f64p * plan.n_views)()
        keep = [np.ascontiguousarray(f, np.float64) for f in residual_fields]
        for i, f in enumerate(keep):
            arr[i] = f64ptr(f)
        out = C.c_double()
        cp = plan.to_c()
        self._check(self._estimate_loss(cameras_to_c(cams), C.byref(cp), arr, C.byref(out)))
        return out.value

    def kmeans_cameras(self, cams, k, seed) -> list:
        assign = np.zeros(len(cams), np.int32)
        self._check(self._kmeans_cameras(cameras_to_c(cams), len(cams), k, seed, i32ptr(assign)))
        return [list(np.nonzero(assign == c)[0]) for c in range(k)]

    def sample_view_batch(self, clusters, rng: "Rng") -> list:
        """sampling::sample_view_batch (view_sampler.cpp:173-184)."""
        n = sum(len(c) for c in clusters)
        assign = np.zeros(n, np.int32)
        for c, m in enumerate(clusters):
            assign[list(m)] = c
        out = np.zeros(len(clusters), np.int32)
        self._check(self._sample_view_batch(i32ptr(assign), n, len(clusters), rng.h, i32ptr(out)))
        return [int(x) for x in out]

    def camera_features(self, cams) -> np.ndarray:
        f = np.zeros((len(cams), 6))
        self._check(self._camera_features(cameras_to_c(cams), len(cams), f64ptr(f)))
        return f

    # ---- Jacobian ----
    def jacobian(self, g: GaussianSet, cams, plan: SamplePlan) -> "CpuJacobian":
        return CpuJacobian(self, g, cams, plan)

    def pcg_dense(self, a: np.ndarray, b: np.ndarray, minv: np.ndarray, iters: int) -> PcgResult:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        minv = np.ascontiguousarray(minv, np.float64)
        x = np.zeros_like(b)
        r = CPcgResult()
        self._check(self._pcg_dense(f64ptr(a), b.size, f64ptr(b), f64ptr(minv), iters, f64ptr(x),
                                    C.byref(r)))
        return PcgResult(x, r.iterations, bool(r.breakdown), r.rel_residual)

    def learning_rate(self, delta: np.ndarray, iteration: int, cfg: LmConfig) -> float:
        d = np.ascontiguousarray(delta, np.float64)
        c = cfg.to_c()
        return self._learning_rate(f64ptr(d), d.size, iteration, C.byref(c))

    def apply_update(self, g: GaussianSet, delta: np.ndarray, eta: float) -> None:
        d = np.ascontiguousarray(delta, np.float64)
        cg = g.to_c()
        self._check(self._apply_update(C.byref(cg), f64ptr(d), eta))

    # ---- training ----
    def train_data(self, cams, images) -> "CpuTrainData":
        return CpuTrainData(self, cams, images)

    def lm_step(self, state: GaussianSet, data: "CpuTrainData", cfg: LmConfig, iteration: int,
                rng: "Rng") -> StepReport:
        batch = np.zeros(1024, np.int32)
        rep = CStepReport()
        rep.batch = i32ptr(batch)
        rep.batch_capacity = batch.size
        cg = state.to_c()
        cc = cfg.to_c()
        self._check(self._lm_step(C.byref(cg), data.h, C.byref(cc), iteration, rng.h, C.byref(rep)))
        return StepReport(rep.iteration, rep.loss_before, rep.loss_after, rep.eta,
                          rep.pcg_iterations, bool(rep.breakdown), list(batch[:rep.batch_size]))

    def batch_loss(self, g: GaussianSet, cams, gts_f32, loss: int = 0, ssim_weight: float = 0.0) -> float:
        gts = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float32).reshape(-1) for x in gts_f32]))
        out = C.c_double()
        cg = g.to_c()
        self._check(self._batch_loss(C.byref(cg), cameras_to_c(cams), len(cams), f32ptr(gts),
                                     loss, ssim_weight, C.byref(out)))
        return out.value

    def mse(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self._mse(f64ptr(a), f64ptr(b), a.shape[1], a.shape[0])

    def psnr(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self._psnr(f64ptr(a), f64ptr(b), a.shape[1], a.shape[0])

    def ssim(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self._ssim(f64ptr(a), f64ptr(b), a.shape[1], a.shape[0])

    def full_gradient(self, g: GaussianSet, cams, gts_f32, loss: int = 0, ssim_weight: float = 0.2) -> np.ndarray:
        """baselines::full_gradient (first_order.cpp:11-44) -> ParamVector (AoS, 14 per Gaussian)."""
        gts = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float32).reshape(-1) for x in gts_f32]))
        out = np.zeros(14 * g.count)
        cg = g.to_c()
        self._check(self._full_gradient(C.byref(cg), cameras_to_c(cams), len(cams), f32ptr(gts), loss,
                                        ssim_weight, f64ptr(out)))
        return out

    def first_order_step(self, g: GaussianSet, m1: np.ndarray, m2: np.ndarray, step: int, grad: np.ndarray,
                         cfg) -> int:
        """baselines::first_order_step on caller-held moments (updated in place); returns the new step."""
        st = C.c_int64(step)
        grad = np.ascontiguousarray(grad, np.float64)
        cg, cc = g.to_c(), cfg.to_c()
        self._check(self._first_order_step(C.byref(cg), f64ptr(m1), f64ptr(m2), C.byref(st), f64ptr(grad),
                                           C.byref(cc)))
        return st.value

    # ---- reference-only entry points (oracle/_ref): run driver and checkpoints
    def train_run_toy(self, out_dir: str, optimizer: str, iterations: int, lm, fo, seed: int = 1,
                      gaussians: int = 0, eval_every: int = 50, deterministic: bool = True,
                      scene_seed: int = 20214, toy=(20, 8, 4, 64)):
        """io::train_run (run.cpp:120-212) on the toy scene; returns (final_train_loss, [mse, psnr, ssim])."""
        fn = self.lib.ref_train_run_toy
        fn.restype = C.c_int
        fn.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_uint64,
                       C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(CLmConfig), C.POINTER(CFirstOrderConfig),
                       _f64p, _f64p]
        loss, test = C.c_double(), np.zeros(3)
        lc, fc = lm.to_c(), fo.to_c()
        self._check(fn(os.fsencode(out_dir), optimizer.encode(), iterations, seed, gaussians, eval_every,
                       int(deterministic), scene_seed, *toy, C.byref(lc), C.byref(fc), C.byref(loss), f64ptr(test)))
        return loss.value, test

    def save_checkpoint(self, path: str, g: GaussianSet) -> None:
        fn = self.lib.ref_save_checkpoint
        fn.restype, fn.argtypes = C.c_int, [C.c_char_p, _f64p, C.c_int64]
        p = np.ascontiguousarray(g.pack())
        self._check(fn(os.fsencode(path), f64ptr(p), g.count))

    def load_checkpoint(self, path: str) -> GaussianSet:
        fn = self.lib.ref_load_checkpoint
        fn.restype, fn.argtypes = C.c_int, [C.c_char_p, _f64p, C.c_int64, C.POINTER(C.c_int64)]
        n = C.c_int64()
        empty = np.zeros(1)
        self._check(fn(os.fsencode(path), f64ptr(empty), 0, C.byref(n)))
        p = np.zeros(14 * n.value)
        self._check(fn(os.fsencode(path), f64ptr(p), p.size, C.byref(n)))
        return GaussianSet.unpack(p)

    def ssim_diag_residuals(self, a, b):
        """metrics::ssim_diag_residuals -> (residual, d_center), both H x W x 3."""
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        r, d = np.zeros_like(a), np.zeros_like(a)
        self._ssim_diag_residuals(f64ptr(a), f64ptr(b), a.shape[1], a.shape[0], f64ptr(r), f64ptr(d))
        return r, d


class Rng:
    """std::mt19937_64 living inside the checker library."""

    def __init__(self, lib: CpuLib, seed: int):
        self.lib = lib
        self.h = lib._rng_new(seed)

    def __call__(self) -> int:
        return self.lib._rng_next(self.h)

    def __del__(self):
        try:
            self.lib._rng_free(self.h)
        except Exception:
            pass


class CpuJacobian:
    """autodiff::SampledJacobian (jacobian.hpp:25-76) inside the checker library."""

    def __init__(self, lib: CpuLib, g: GaussianSet, cams, plan: SamplePlan):
        self.lib = lib
        cg = g.to_c()
        cp = plan.to_c()
        self._plan = plan
        self.h = lib._jac_new(C.byref(cg), cameras_to_c(cams), len(cams), C.byref(cp))
        if not self.h:
            raise ValueError(lib._last_error().decode())
        self.rdim = lib._jac_residual_dim(self.h)
        self.pdim = lib._jac_param_dim(self.h)

    def __del__(self):
        try:
            self.lib._jac_free(self.h)
        except Exception:
            pass

    def residual_dim(self) -> int:
        return self.rdim

    def param_dim(self) -> int:
        return self.pdim

    def jvp(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float64)
        if v.size != self.pdim:
            raise ValueError("jvp: probe vector length mismatch")
        out = np.zeros(self.rdim)
        self.lib._check(self.lib._jac_jvp(self.h, f64ptr(v), f64ptr(out)))
        return out

    def vjp(self, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, np.float64)
        if u.size != self.rdim:
            raise ValueError("vjp: input length mismatch")
        out = np.zeros(self.pdim)
        self.lib._check(self.lib._jac_vjp(self.h, f64ptr(u), f64ptr(out)))
        return out

    def jtj_diag(self) -> np.ndarray:
        out = np.zeros(self.pdim)
        self.lib._check(self.lib._jac_jtj_diag(self.h, f64ptr(out)))
        return out

    def gn_apply(self, lam: float, p: np.ndarray) -> np.ndarray:
        p = np.ascontiguousarray(p, np.float64)
        out = np.zeros(self.pdim)
        self.lib._check(self.lib._jac_gn_apply(self.h, lam, f64ptr(p), f64ptr(out)))
        return out

    def residual_weights(self) -> np.ndarray:
        out = np.zeros(self.rdim)
        self.lib._check(self.lib._jac_weights(self.h, f64ptr(out)))
        return out

    def set_residual_weights(self, w: np.ndarray) -> None:
        w = np.ascontiguousarray(w, np.float64)
        if w.size != self.rdim:
            raise ValueError("residual weight vector has wrong length")
        self.lib._check(self.lib._jac_set_weights(self.h, f64ptr(w)))

    def pcg(self, lam: float, b: np.ndarray, minv: np.ndarray, iters: int) -> PcgResult:
        b = np.ascontiguousarray(b, np.float64)
        minv = np.ascontiguousarray(minv, np.float64)
        x = np.zeros(self.pdim)
        r = CPcgResult()
        self.lib._check(self.lib._jac_pcg(self.h, lam, f64ptr(b), f64ptr(minv), iters, f64ptr(x),
                                          C.byref(r)))
        return PcgResult(x, r.iterations, bool(r.breakdown), r.rel_residual)


class CpuTrainData:
    """solver::TrainData (lm.hpp:53-60); images as float32 dataset buffers (or float64)."""

    def __init__(self, lib: CpuLib, cams, images):
        self.lib = lib
        self.cameras = list(cams)
        cc = cameras_to_c(cams)
        if all(np.asarray(im).dtype == np.float64 for im in images):
            buf = np.ascontiguousarray(np.concatenate([np.asarray(im).reshape(-1) for im in images]))
            self.h = lib._train_new_f64(cc, len(cams), f64ptr(buf))
        else:
            buf = np.ascontiguousarray(np.concatenate([np.asarray(im, np.float32).reshape(-1)
                                                       for im in images]))
            self.h = lib._train_new(cc, len(cams), f32ptr(buf))

    def rebuild_clusters(self, k: int, seed: int) -> None:
        self.lib._check(self.lib._train_rebuild_clusters(self.h, k, seed))

    def set_clusters(self, clusters) -> None:
        assign = np.zeros(len(self.cameras), np.int32)
        for c, members in enumerate(clusters):
            for i in members:
                assign[i] = c
        self.lib._check(self.lib._train_set_clusters(self.h, i32ptr(assign), len(self.cameras),
                                                     len(clusters)))

    def __del__(self):
        try:
            self.lib._train_free(self.h)
        except Exception:
            pass


_cache: dict = {}


def ref() -> CpuLib:
    """The real reference (oracle/_ref)."""
    if "ref" not in _cache:
        _cache["ref"] = CpuLib(REF_SO, "ref_")
    return _cache["ref"]


def port() -> CpuLib:
    """The C restatement (oracle/liboracle.so)."""
    if "port" not in _cache:
        _cache["port"] = CpuLib(PORT_SO, "orc_")
    return _cache["port"]
