"""Python mirror of the reference's C++ solver API over libslm_b200.so.

Method names and argument meaning follow the reference
(render::bin_and_sort, sampling::build_sample_plan, SampledJacobian::gn_apply,
solver::pcg_solve, solver::lm_step, ...), and errors map like the reference's
exceptions: std::invalid_argument -> ValueError, std::domain_error ->
ArithmeticError, std::runtime_error -> RuntimeError.  Every compute call runs
the sm_100a kernels; there is no CPU fallback — without the built library or
a CUDA device, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .types import (CCamera, CFirstOrderConfig, CGaussians, CLmConfig, CMetricReport, CPcgResult, CPlan, CStepReport, Camera,
                    GaussianSet, LmConfig, MetricReport, PcgResult, SamplePlan, StepReport, cameras_to_c, f32ptr,
                    f64ptr, i32ptr, i64ptr)

LIB_PATH = os.environ.get("SLM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libslm_b200.so")

_vp = C.c_void_p
_f64p = C.POINTER(C.c_double)
_f32p = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_APPLY = C.CFUNCTYPE(None, C.c_void_p, _f64p, _f64p)


class SlmError(RuntimeError):
    pass


class CudaUnavailable(SlmError):
    pass


_SIGS = {
    "slm_last_error": (C.c_char_p, []),
    "slm_version": (C.c_int, []),
    "slm_device_count": (C.c_int, [_i32p]),
    "slm_context_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "slm_context_destroy": (C.c_int, [_vp]),
    "slm_context_synchronize": (C.c_int, [_vp]),
    "slm_context_set_stream": (C.c_int, [_vp, _vp]),
    "slm_context_set_timing": (C.c_int, [_vp, C.c_int]),
    "slm_context_set_deterministic": (C.c_int, [_vp, C.c_int]),
    "slm_render_pixel": (C.c_int, [_vp, C.c_int, _f64p, C.c_double, C.c_double, _f64p, _i32p]),
    "slm_render_splats": (C.c_int, [_vp, C.c_void_p, C.c_int, _f64p, _i32p, _i32p, _f64p, _f64p, _i32p]),
    "slm_residuals": (C.c_int, [_f64p, _f64p, C.c_int64, _f64p]),
    "slm_context_step_stats": (C.c_int, [_vp, _i64p]),
    "slm_context_last_samples": (C.c_int, [_vp, C.c_int64, _i64p, _i32p, _i32p, _f32p]),
    "slm_context_timings": (C.c_int, [_vp, _f64p, C.c_int, _i32p]),
    "slm_context_timing_names": (C.c_char_p, [_vp]),
    "slm_launch_count": (C.c_longlong, []),
    "slm_context_set_profiling": (C.c_int, [_vp, C.c_int]),
    "slm_context_profile_collect": (C.c_int, [_vp, _f64p, _i32p]),
    "slm_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "slm_debug_nccl_selftest": (C.c_int, [_vp, _f64p]),
    "slm_context_init_comm": (C.c_int, [_vp, C.POINTER(C.c_uint8), C.c_int, C.c_int]),
    "slm_local_group_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "slm_local_group_destroy": (None, [_vp]),
    "slm_context_init_local": (C.c_int, [_vp, _vp, C.c_int]),
    "slm_context_set_comm_chunks": (C.c_int, [_vp, C.c_int]),
    "slm_context_rank": (C.c_int, [_vp, _i32p, _i32p]),
    "slm_rng_create": (C.c_int, [C.c_uint64, C.POINTER(_vp)]),
    "slm_rng_destroy": (None, [_vp]),
    "slm_rng_next": (C.c_uint64, [_vp]),
    "slm_scene_create": (C.c_int, [_vp, C.POINTER(CGaussians), C.POINTER(_vp)]),
    "slm_scene_destroy": (None, [_vp]),
    "slm_scene_upload": (C.c_int, [_vp, C.POINTER(CGaussians)]),
    "slm_scene_download": (C.c_int, [_vp, C.POINTER(CGaussians)]),
    "slm_scene_count": (C.c_int, [_vp, _i32p, _i32p]),
    "slm_scene_apply_update": (C.c_int, [_vp, _f64p, C.c_double]),
    "slm_scene_beta_ptrs": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp)]),
    "slm_bin_and_sort": (C.c_int, [_vp, C.POINTER(CGaussians), C.POINTER(CCamera), _i32p, _i32p,
                                   C.c_int64, _i64p]),
    "slm_prepare": (C.c_int, [_vp, C.POINTER(CGaussians), C.POINTER(CCamera), _f64p, _f64p, _f64p,
                              _f64p, _f64p, _f64p, _i32p]),
    "slm_render_full": (C.c_int, [_vp, C.POINTER(CGaussians), C.POINTER(CCamera), _f64p, _f64p,
                                  _i32p]),
    "slm_scene_render": (C.c_int, [_vp, C.POINTER(CCamera), _f32p, _f32p, _i32p]),
    "slm_build_sample_plan": (C.c_int, [C.POINTER(CCamera), C.c_int, C.c_int, C.c_int, C.c_int, _vp,
                                        C.POINTER(_f64p), C.POINTER(_i32p), C.POINTER(_f64p),
                                        C.POINTER(_vp)]),
    "slm_exhaustive_plan": (C.c_int, [C.POINTER(CCamera), C.c_int, C.POINTER(_vp)]),
    "slm_plan_destroy": (None, [_vp]),
    "slm_plan_size": (C.c_int, [_vp, _i32p, _i64p]),
    "slm_plan_export": (C.c_int, [_vp, _i32p, _i64p, _i32p, _i32p, _i32p, _f64p]),
    "slm_estimate_loss": (C.c_int, [C.POINTER(CCamera), C.POINTER(CPlan), C.POINTER(_f64p), _f64p]),
    "slm_camera_features": (C.c_int, [C.POINTER(CCamera), C.c_int, _f64p]),
    "slm_kmeans_cameras": (C.c_int, [C.POINTER(CCamera), C.c_int, C.c_int, C.c_uint64, _i32p]),
    "slm_sample_view_batch": (C.c_int, [_i32p, C.c_int, C.c_int, _vp, _i32p]),
    "slm_jacobian_create": (C.c_int, [_vp, C.POINTER(CGaussians), C.POINTER(CCamera), C.c_int,
                                      C.POINTER(CPlan), C.POINTER(_vp)]),
    "slm_jacobian_create_scene": (C.c_int, [_vp, C.POINTER(CCamera), C.c_int, C.POINTER(CPlan),
                                            C.POINTER(_vp)]),
    "slm_jacobian_destroy": (None, [_vp]),
    "slm_jacobian_dims": (C.c_int, [_vp, _i64p, _i64p]),
    "slm_jacobian_jvp": (C.c_int, [_vp, _f64p, _f64p]),
    "slm_jacobian_vjp": (C.c_int, [_vp, _f64p, _f64p]),
    "slm_jacobian_jtj_diag": (C.c_int, [_vp, _f64p]),
    "slm_jacobian_gn_apply": (C.c_int, [_vp, C.c_double, _f64p, _f64p]),
    "slm_jacobian_weights": (C.c_int, [_vp, _f64p]),
    "slm_jacobian_set_weights": (C.c_int, [_vp, _f64p]),
    "slm_jacobian_gn_apply_dev": (C.c_int, [_vp, C.c_float, _vp, _vp]),
    "slm_jacobian_pcg": (C.c_int, [_vp, C.c_double, _f64p, _f64p, C.c_int, _f64p,
                                   C.POINTER(CPcgResult)]),
    "slm_jacobian_stats": (C.c_int, [_vp, _i64p]),
    "slm_toy_gaussians": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(CGaussians)]),
    "slm_jacobian_mask_stats": (C.c_int, [_vp, _i64p]),
    "slm_pcg_solve": (C.c_int, [_vp, _APPLY, _vp, _f64p, _f64p, C.c_int64, C.c_int, _f64p,
                                C.POINTER(CPcgResult)]),
    "slm_learning_rate": (C.c_int, [_vp, _f64p, C.c_int64, C.c_int, C.POINTER(CLmConfig), _f64p]),
    "slm_default_lm_config": (None, [C.POINTER(CLmConfig)]),
    "slm_train_create": (C.c_int, [_vp, C.POINTER(CCamera), C.c_int, _f32p, C.POINTER(_vp)]),
    "slm_train_destroy": (None, [_vp]),
    "slm_train_rebuild_clusters": (C.c_int, [_vp, C.c_int, C.c_uint64]),
    "slm_train_set_clusters": (C.c_int, [_vp, _i32p, C.c_int]),
    "slm_train_clusters": (C.c_int, [_vp, _i32p, _i32p]),
    "slm_lm_step": (C.c_int, [_vp, _vp, C.POINTER(CLmConfig), C.c_int, _vp,
                              C.POINTER(CStepReport)]),
    "slm_lm_step_host": (C.c_int, [_vp, C.POINTER(CGaussians), _vp, C.POINTER(CLmConfig), C.c_int,
                                   _vp, C.POINTER(CStepReport)]),
    "slm_batch_loss": (C.c_int, [_vp, _vp, _i32p, C.c_int, _f64p]),
    "slm_save_checkpoint": (C.c_int, [C.c_char_p, C.POINTER(CGaussians)]),
    "slm_checkpoint_count": (C.c_int, [C.c_char_p, _i32p]),
    "slm_load_checkpoint": (C.c_int, [C.c_char_p, C.POINTER(CGaussians)]),
    "slm_default_first_order_config": (None, [C.POINTER(CFirstOrderConfig)]),
    "slm_full_gradient": (C.c_int, [_vp, _vp, C.c_int, C.c_double, _f64p]),
    "slm_first_order_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "slm_first_order_destroy": (None, [_vp]),
    "slm_first_order_moments": (C.c_int, [_vp, _f64p, _f64p, _i64p]),
    "slm_first_order_set_moments": (C.c_int, [_vp, _f64p, _f64p, C.c_int64]),
    "slm_first_order_apply": (C.c_int, [_vp, _f64p, C.POINTER(CFirstOrderConfig)]),
    "slm_first_order_step": (C.c_int, [_vp, _vp, C.POINTER(CFirstOrderConfig), _f64p]),
    "slm_batch_loss_kind": (C.c_int, [_vp, _vp, _i32p, C.c_int, C.c_int, C.c_double, _f64p]),
    "slm_ssim_diag_residuals": (C.c_int, [_vp, _f64p, _f64p, C.c_int, C.c_int, _f64p, _f64p]),
    "slm_evaluate": (C.c_int, [_vp, _f64p, _f64p, C.c_int, C.c_int, C.POINTER(CMetricReport)]),
    "slm_evaluate_split": (C.c_int, [_vp, _vp, C.POINTER(CMetricReport)]),
    "slm_random_init": (C.c_int, [C.c_int, _f64p, _f64p, _vp, C.POINTER(CGaussians)]),
    "slm_ring_camera": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                  C.POINTER(CCamera)]),
}


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libslm_b200.so and bind every C-ABI entry point (no GPU needed)."""
    if not os.path.exists(path):
        raise SlmError(f"{path} is not built; run `python -m paper_2504_12905_b200.build`")
    dll = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(dll, name)
        fn.restype = res
        fn.argtypes = args
    return dll


_dll_cache: dict = {}


def dll() -> C.CDLL:
    if "dll" not in _dll_cache:
        _dll_cache["dll"] = load_library()
    return _dll_cache["dll"]


def _check(rc: int):
    if rc != 0:
        msg = dll().slm_last_error().decode()
        exc = {1: ValueError, 2: ArithmeticError, 3: RuntimeError}.get(rc, SlmError)
        raise exc(msg)


class Rng:
    """std::mt19937_64 inside the library (run.cpp:126-127); host-only."""

    def __init__(self, seed: int):
        h = _vp()
        _check(dll().slm_rng_create(seed, C.byref(h)))
        self.h = h

    def __call__(self) -> int:
        return dll().slm_rng_next(self.h)

    def __del__(self):
        try:
            dll().slm_rng_destroy(self.h)
        except Exception:
            pass


class HostSampler:
    """The host half of the path: samplers that must replay the reference's
    libstdc++ RNG stream (build_sample_plan, k-means batching, random_init).
    Needs the built library but no GPU."""

    kind = "b200-host"

    def __init__(self):
        self.dll = dll()

    def _check(self, rc: int):
        _check(rc)

    def rng(self, seed: int) -> Rng:
        return Rng(seed)

    # ---- io helpers

    def random_init(self, count, cube_min, cube_max, rng: Rng) -> GaussianSet:
        g = GaussianSet(count)
        lo = np.asarray(cube_min, np.float64)
        hi = np.asarray(cube_max, np.float64)
        cg = g.to_c()
        self._check(self.dll.slm_random_init(count, f64ptr(lo), f64ptr(hi), rng.h, C.byref(cg)))
        return g

    def toy_gaussians(self, count: int, seed: int = 20214) -> GaussianSet:
        """io::generate_toy_scene's ground truth (scene_gen.cpp:38-71)."""
        g = GaussianSet(count)
        cg = g.to_c()
        self._check(self.dll.slm_toy_gaussians(count, seed, C.byref(cg)))
        return g

    def ring_camera(self, angle, radius, height, width, height_px=0) -> Camera:
        c = CCamera()
        self._check(self.dll.slm_ring_camera(angle, radius, height, width, height_px, C.byref(c)))
        return Camera.from_c(c)

    # ---- sampling
    def _export_plan(self, h) -> SamplePlan:
        try:
            nv = C.c_int32()
            tot = C.c_int64()
            self._check(self.dll.slm_plan_size(h, C.byref(nv), C.byref(tot)))
            vc = np.zeros(nv.value, np.int32)
            vo = np.zeros(nv.value + 1, np.int64)
            px, py, tl = (np.zeros(tot.value, np.int32) for _ in range(3))
            w = np.zeros(tot.value)
            self._check(self.dll.slm_plan_export(h, i32ptr(vc), i64ptr(vo), i32ptr(px), i32ptr(py),
                                                 i32ptr(tl), f64ptr(w)))
            return SamplePlan(vc, vo, px, py, tl, w)
        finally:
            self.dll.slm_plan_destroy(h)

    def build_sample_plan(self, cams, samples_per_tile, dist, rng: Rng, lane_width=32,
                          aux=None) -> SamplePlan:
        cc = cameras_to_c(cams)
        ai = ac = ag = None
        keep = []
        if aux is not None:
            ai, ac, ag = (_f64p * len(aux))(), (_i32p * len(aux))(), (_f64p * len(aux))()
            for i, (im, cn, gt) in enumerate(aux):
                im = np.ascontiguousarray(im, np.float64)
                cn = np.ascontiguousarray(cn, np.int32)
                gt = np.ascontiguousarray(gt if gt is not None else np.zeros_like(im), np.float64)
                keep += [im, cn, gt]
                ai[i], ac[i], ag[i] = f64ptr(im), i32ptr(cn), f64ptr(gt)
        h = _vp()
        self._check(self.dll.slm_build_sample_plan(cc, len(cams), samples_per_tile, dist, lane_width,
                                                   rng.h, ai, ac, ag, C.byref(h)))
        plan = self._export_plan(h)
        plan.samples_per_tile, plan.dist = samples_per_tile, dist
        return plan

    def exhaustive_plan(self, cams) -> SamplePlan:
        h = _vp()
        self._check(self.dll.slm_exhaustive_plan(cameras_to_c(cams), len(cams), C.byref(h)))
        plan = self._export_plan(h)
        plan.samples_per_tile = 256
        return plan

    def estimate_loss(self, cams, plan: SamplePlan, residual_fields) -> float:
        """sampling::estimate_loss (sample_plan.cpp:199-222): residual_fields[v] is the
        H x W x 3 residual image of plan view v."""
        if len(residual_fields) != plan.n_views:
            raise ValueError("one residual field per plan view required")
        arr = (_f64p * plan.n_views)()
        keep = [np.ascontiguousarray(f, np.float64) for f in residual_fields]
        for i, f in enumerate(keep):
            arr[i] = f64ptr(f)
        out = C.c_double()
        cp = plan.to_c()
        self._check(self.dll.slm_estimate_loss(cameras_to_c(cams), C.byref(cp), arr, C.byref(out)))
        return out.value

    def kmeans_cameras(self, cams, k, seed) -> list:
        assign = np.zeros(len(cams), np.int32)
        self._check(self.dll.slm_kmeans_cameras(cameras_to_c(cams), len(cams), k, seed, i32ptr(assign)))
        return [list(np.nonzero(assign == c)[0]) for c in range(k)]

    def camera_features(self, cams) -> np.ndarray:
        f = np.zeros((len(cams), 6))
        self._check(self.dll.slm_camera_features(cameras_to_c(cams), len(cams), f64ptr(f)))
        return f

    def sample_view_batch(self, clusters, rng: Rng) -> list:
        n = sum(len(c) for c in clusters)
        assign = np.zeros(n, np.int32)
        for c, m in enumerate(clusters):
            assign[list(m)] = c
        out = np.zeros(len(clusters), np.int32)
        self._check(self.dll.slm_sample_view_batch(i32ptr(assign), n, len(clusters), rng.h, i32ptr(out)))
        return [int(x) for x in out]



class LocalGroup:
    """slm_local_group: `world` contexts of this process acting as ranks."""

    def __init__(self, world: int):
        self.dll = dll()
        h = _vp()
        _check(self.dll.slm_local_group_create(world, C.byref(h)))
        self.h = h
        self.world = world

    def __del__(self):
        try:
            self.dll.slm_local_group_destroy(self.h)
        except Exception:
            pass


class Lib(HostSampler):
    """One CUDA context (device + stream) driving the B200 kernels."""

    kind = "b200"

    def __init__(self, device: int = 0):
        self.dll = dll()
        n = C.c_int32(0)
        if self.dll.slm_device_count(C.byref(n)) != 0 or n.value == 0:
            raise CudaUnavailable("no CUDA device: the B200 path has no CPU fallback")
        h = _vp()
        self._check(self.dll.slm_context_create(device, C.byref(h)))
        self.ctx = h

    def __del__(self):
        try:
            self.dll.slm_context_destroy(self.ctx)
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != 0:
            msg = self.dll.slm_last_error().decode()
            exc = {1: ValueError, 2: ArithmeticError, 3: RuntimeError}.get(rc, SlmError)
            raise exc(msg)

    def synchronize(self):
        self._check(self.dll.slm_context_synchronize(self.ctx))

    def set_stream(self, stream_handle: int):
        self._check(self.dll.slm_context_set_stream(self.ctx, _vp(stream_handle)))

    def set_deterministic(self, on: bool):
        """Fixed-order J^T / diag accumulation (default on): bitwise reproducible
        products, PCG solutions and LM trajectories.  Off: float atomics."""
        self._check(self.dll.slm_context_set_deterministic(self.ctx, 1 if on else 0))

    def last_samples(self):
        """(px, py, weight) of the last lm_step's sampled pixels in plan order."""
        n = C.c_int64()
        self._check(self.dll.slm_context_last_samples(self.ctx, 0, C.byref(n), None, None, None))
        px, py = np.zeros(n.value, np.int32), np.zeros(n.value, np.int32)
        w = np.zeros(n.value, np.float32)
        self._check(self.dll.slm_context_last_samples(self.ctx, n.value, C.byref(n), i32ptr(px), i32ptr(py),
                                                      f32ptr(w)))
        return px, py, w

    def step_stats(self) -> dict:
        """Counters of the last lm_step on this context (views, sum G_v, entries,
        samples, pixels, PCG iterations; G_v / entries after the update)."""
        out = np.zeros(8, np.int64)
        self._check(self.dll.slm_context_step_stats(self.ctx, i64ptr(out)))
        return dict(views=int(out[0]), valid=int(out[1]), entries=int(out[2]), samples=int(out[3]),
                    pixels=int(out[4]), pcg_iterations=int(out[5]), valid_after=int(out[6]),
                    entries_after=int(out[7]))

    def set_timing(self, on: bool):
        self._check(self.dll.slm_context_set_timing(self.ctx, 1 if on else 0))

    def timings(self) -> dict:
        """CUDA-event stage timings (ms) of the last lm_step with timing enabled."""
        buf = np.zeros(256)
        n = C.c_int32()
        self._check(self.dll.slm_context_timings(self.ctx, f64ptr(buf), 256, C.byref(n)))
        names = self.dll.slm_context_timing_names(self.ctx).decode().split(",")
        out: dict = {}
        for name, ms in zip(names, buf[:n.value]):
            out[name] = round(out.get(name, 0.0) + float(ms), 3)
        return out

    def launch_count(self) -> int:
        return self.dll.slm_launch_count()

    def set_profiling(self, on: bool):
        self._check(self.dll.slm_context_set_profiling(self.ctx, 1 if on else 0))

    def profile_collect(self) -> dict:
        """Summed ms of {tangents, raster, chain} over the profiled products."""
        out = np.zeros(3)
        n = C.c_int32()
        self._check(self.dll.slm_context_profile_collect(self.ctx, f64ptr(out), C.byref(n)))
        return dict(n=n.value, tangents_ms=out[0], raster_ms=out[1], chain_ms=out[2])

    # ---- multi-GPU
    @staticmethod
    def nccl_unique_id(dll) -> bytes:
        buf = (C.c_uint8 * 128)()
        rc = dll.slm_nccl_unique_id(buf)
        if rc != 0:
            raise SlmError(dll.slm_last_error().decode())
        return bytes(buf)

    def init_local(self, group: "LocalGroup", rank: int):
        """Join an in-process rank group (slm_context_init_local): the view-sharded
        lm_step / products with the group's rank-order sums as the collectives."""
        self._check(self.dll.slm_context_init_local(self.ctx, group.h, rank))
        self._group = group  # keep the group alive while this context uses it

    def set_comm_chunks(self, chunks: int):
        """Gaussian chunks of the pipelined chain + allreduce (world > 1)."""
        self._check(self.dll.slm_context_set_comm_chunks(self.ctx, chunks))

    def nccl_selftest(self):
        """One-rank NCCL communicator on this device: (max |error|, elements checked)."""
        out = np.zeros(2)
        self._check(self.dll.slm_debug_nccl_selftest(self.ctx, f64ptr(out)))
        return float(out[0]), int(out[1])

    def init_comm(self, uid: bytes, rank: int, world: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self.dll.slm_context_init_comm(self.ctx, buf, rank, world))

    # ---- render
    def bin_and_sort(self, g: GaussianSet, cam: Camera):
        tiles = cam.tiles_x * cam.tiles_y
        offsets = np.zeros(tiles + 1, np.int32)
        cap = max(16, 8 * g.count)
        cg, cc = g.to_c(), cam.to_c()
        while True:
            idx = np.zeros(cap, np.int32)
            n = C.c_int64()
            self._check(self.dll.slm_bin_and_sort(self.ctx, C.byref(cg), C.byref(cc), i32ptr(offsets),
                                                  i32ptr(idx), cap, C.byref(n)))
            if n.value <= cap:
                return offsets, idx[:n.value].copy()
            cap = n.value

    def prepare(self, g: GaussianSet, cam: Camera) -> dict:
        n = g.count
        out = dict(mean2d=np.zeros(2 * n), conic=np.zeros(3 * n), opacity=np.zeros(n),
                   color=np.zeros(3 * n), depth=np.zeros(n), radius=np.zeros(n),
                   valid=np.zeros(n, np.int32))
        cg, cc = g.to_c(), cam.to_c()
        self._check(self.dll.slm_prepare(self.ctx, C.byref(cg), C.byref(cc),
                                         *(f64ptr(out[k]) for k in ("mean2d", "conic", "opacity",
                                                                    "color", "depth", "radius")),
                                         i32ptr(out["valid"])))
        return out

    @staticmethod
    def pack_splats(prep: dict) -> np.ndarray:
        """render::SplatD fields of a prepare() dict as the [n, 10] f64 layout of
        render_pixel / render_with_context (mean2d, conic, opacity, colour, unused)."""
        n = prep["opacity"].size
        d = np.zeros((n, 10))
        d[:, 0:2] = prep["mean2d"].reshape(n, 2)
        d[:, 2:5] = prep["conic"].reshape(n, 3)
        d[:, 5] = prep["opacity"]
        d[:, 6:9] = prep["color"].reshape(n, 3)
        return d

    def render_pixel(self, splats, px: float, py: float):
        """render::render_pixel (rasterizer.cpp:52-60) over an ordered [n, 10] splat array
        -> (rgb[3], transmittance, contrib)."""
        d = np.ascontiguousarray(splats, np.float64).reshape(-1, 10)
        out = np.zeros(4)
        cnt = C.c_int32()
        self._check(self.dll.slm_render_pixel(self.ctx, d.shape[0], f64ptr(d), px, py, f64ptr(out), C.byref(cnt)))
        return out[:3], float(out[3]), cnt.value

    def render_with_context(self, cam: Camera, splats, offsets, indices):
        """render::render_with_context (rasterizer.cpp:62-91) of prepared splats ([n, 10])
        and their CSR tile grid -> (image, transmittance, contrib)."""
        d = np.ascontiguousarray(splats, np.float64).reshape(-1, 10)
        off = np.ascontiguousarray(offsets, np.int32)
        idx = np.ascontiguousarray(indices, np.int32)
        if off.size != cam.tiles_x * cam.tiles_y + 1:
            raise ValueError("render_with_context: offsets must have tiles + 1 entries")
        img = np.zeros((cam.height, cam.width, 3))
        tr = np.zeros((cam.height, cam.width))
        cn = np.zeros((cam.height, cam.width), np.int32)
        cc = cam.to_c()
        self._check(self.dll.slm_render_splats(self.ctx, C.byref(cc), d.shape[0], f64ptr(d), i32ptr(off),
                                               i32ptr(idx if idx.size else np.zeros(1, np.int32)), f64ptr(img),
                                               f64ptr(tr), i32ptr(cn)))
        return img, tr, cn

    def residuals(self, rendered, truth) -> np.ndarray:
        """render::residuals (rasterizer.cpp:97-104)."""
        a = np.ascontiguousarray(rendered, np.float64)
        b = np.ascontiguousarray(truth, np.float64)
        if a.shape != b.shape:
            raise ValueError("residuals: image shapes differ")
        out = np.empty_like(a)
        self._check(self.dll.slm_residuals(f64ptr(a), f64ptr(b), a.size, f64ptr(out)))
        return out

    def render_full(self, g: GaussianSet, cam: Camera):
        img = np.zeros((cam.height, cam.width, 3))
        tr = np.zeros((cam.height, cam.width))
        cn = np.zeros((cam.height, cam.width), np.int32)
        cg, cc = g.to_c(), cam.to_c()
        self._check(self.dll.slm_render_full(self.ctx, C.byref(cg), C.byref(cc), f64ptr(img),
                                             f64ptr(tr), i32ptr(cn)))
        return img, tr, cn

    # ---- Jacobian / solver
    def jacobian(self, g, cams, plan: SamplePlan) -> "Jacobian":
        return Jacobian(self, g, cams, plan)

    def pcg_dense(self, a, b, minv, iters) -> PcgResult:
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]

        def apply(_user, p, out):
            pv = np.ctypeslib.as_array(p, shape=(n,))
            ov = np.ctypeslib.as_array(out, shape=(n,))
            ov[:] = a @ pv

        return self.pcg_solve(apply, b, minv, iters)

    def pcg_solve(self, apply, b, minv, iters) -> PcgResult:
        """solver::pcg_solve(ApplyFn, b, minv, max_iters) (pcg.hpp:22-23)."""
        b = np.ascontiguousarray(b, np.float64)
        minv = np.ascontiguousarray(minv, np.float64)
        if minv.size != b.size:
            raise ValueError("pcg: preconditioner length mismatch")
        x = np.zeros_like(b)
        r = CPcgResult()
        cb = _APPLY(apply)
        self._check(self.dll.slm_pcg_solve(self.ctx, cb, None, f64ptr(b), f64ptr(minv), b.size, iters,
                                           f64ptr(x), C.byref(r)))
        return PcgResult(x, r.iterations, bool(r.breakdown), r.rel_residual)

    def learning_rate(self, delta, iteration, cfg: LmConfig) -> float:
        d = np.ascontiguousarray(delta, np.float64)
        out = C.c_double()
        c = cfg.to_c()
        self._check(self.dll.slm_learning_rate(self.ctx, f64ptr(d), d.size, iteration, C.byref(c),
                                               C.byref(out)))
        return out.value

    def apply_update(self, g: GaussianSet, delta, eta) -> None:
        s = Scene(self, g)
        s.apply_update(delta, eta)
        s.download(g)

    # ---- training
    def train_data(self, cams, images) -> "TrainData":
        return TrainData(self, cams, images)

    def lm_step(self, state: GaussianSet, data: "TrainData", cfg: LmConfig, iteration: int,
                rng: Rng) -> StepReport:
        """solver::lm_step on a host GaussianSet (drop-in form, lm.hpp:70-71)."""
        batch = np.zeros(4096, np.int32)
        rep = CStepReport()
        rep.batch, rep.batch_capacity = i32ptr(batch), batch.size
        cg, cc = state.to_c(), cfg.to_c()
        self._check(self.dll.slm_lm_step_host(self.ctx, C.byref(cg), data.h, C.byref(cc), iteration,
                                              rng.h, C.byref(rep)))
        return _report(rep, batch)

    def batch_loss(self, g: GaussianSet, data: "TrainData", cam_ids, loss: int = 0,
                   ssim_weight: float = 0.0) -> float:
        return Scene(self, g).batch_loss(data, cam_ids, loss, ssim_weight)

    def evaluate(self, rendered, ground_truth) -> MetricReport:
        """metrics::evaluate (image_metrics.cpp:180-186): mse, psnr, ssim of two H x W x 3
        images, computed on the device in f64."""
        a = np.ascontiguousarray(rendered, np.float64)
        b = np.ascontiguousarray(ground_truth, np.float64)
        if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
            raise ValueError("metrics: image shapes differ")
        r = CMetricReport()
        self._check(self.dll.slm_evaluate(self.ctx, f64ptr(a), f64ptr(b), a.shape[1], a.shape[0],
                                          C.byref(r)))
        return MetricReport(r.mse, r.psnr, r.ssim)

    def evaluate_split(self, g: GaussianSet, split: "TrainData") -> MetricReport:
        return Scene(self, g).evaluate_split(split)

    def save_checkpoint(self, path: str, g: GaussianSet) -> None:
        """io::save_checkpoint (checkpoint.cpp:45-66): SPLMGS01 file + .meta.txt sidecar."""
        cg = g.to_c()
        self._check(self.dll.slm_save_checkpoint(os.fsencode(path), C.byref(cg)))

    def load_checkpoint(self, path: str) -> GaussianSet:
        """io::load_checkpoint (checkpoint.cpp:68-82)."""
        n = C.c_int32()
        self._check(self.dll.slm_checkpoint_count(os.fsencode(path), C.byref(n)))
        g = GaussianSet(n.value)
        cg = g.to_c()
        self._check(self.dll.slm_load_checkpoint(os.fsencode(path), C.byref(cg)))
        return g

    def full_gradient(self, g: GaussianSet, data: "TrainData", loss: int = 0, ssim_weight: float = 0.2) -> np.ndarray:
        """baselines::full_gradient (first_order.cpp:11-44) -> ParamVector (AoS, 14 per Gaussian)."""
        return Scene(self, g).full_gradient(data, loss, ssim_weight)

    def first_order_step(self, g: GaussianSet, m1: np.ndarray, m2: np.ndarray, step: int, grad: np.ndarray,
                         cfg) -> int:
        """baselines::first_order_step (first_order.cpp:115-122), drop-in host form: the state
        and the caller's moments (AoS, updated in place) go through the device; returns the step."""
        scene = Scene(self, g)
        fo = FirstOrder(self, scene)
        fo.set_moments(m1, m2, step)
        fo.apply(grad, cfg)
        a, b, st = fo.moments()
        m1[:], m2[:] = a, b
        scene.download(g)
        return st

    def ssim_diag_residuals(self, a, b):
        """metrics::ssim_diag_residuals (image_metrics.cpp:141-178) on the device:
        (residual, d_center), each H x W x 3 f64."""
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
            raise ValueError("metrics: image shapes differ")
        r, d = np.zeros_like(a), np.zeros_like(a)
        self._check(self.dll.slm_ssim_diag_residuals(self.ctx, f64ptr(a), f64ptr(b), a.shape[1], a.shape[0],
                                                     f64ptr(r), f64ptr(d)))
        return r, d


def _report(rep: CStepReport, batch) -> StepReport:
    return StepReport(rep.iteration, rep.loss_before, rep.loss_after, rep.eta, rep.pcg_iterations,
                      bool(rep.breakdown), [int(b) for b in batch[:rep.batch_size]])


class Scene:
    """Device-resident GaussianSet (f64 SoA [14][Gp] in HBM)."""

    def __init__(self, L: Lib, g: GaussianSet):
        self.L = L
        h = _vp()
        cg = g.to_c()
        L._check(L.dll.slm_scene_create(L.ctx, C.byref(cg), C.byref(h)))
        self.h = h
        self.count = g.count
        n, gp = C.c_int32(), C.c_int32()
        L.dll.slm_scene_count(h, C.byref(n), C.byref(gp))
        self.padded = gp.value

    def __del__(self):
        try:
            self.L.dll.slm_scene_destroy(self.h)
        except Exception:
            pass

    def upload(self, g: GaussianSet):
        cg = g.to_c()
        self.L._check(self.L.dll.slm_scene_upload(self.h, C.byref(cg)))

    def download(self, g: GaussianSet | None = None) -> GaussianSet:
        g = g if g is not None else GaussianSet(self.count)
        cg = g.to_c()
        self.L._check(self.L.dll.slm_scene_download(self.h, C.byref(cg)))
        return g

    def apply_update(self, delta, eta: float):
        d = np.ascontiguousarray(delta, np.float64)
        if d.size != 14 * self.count:
            raise ValueError("update length does not match parameter count")
        self.L._check(self.L.dll.slm_scene_apply_update(self.h, f64ptr(d), eta))

    def render(self, cam: Camera):
        img = np.zeros((cam.height, cam.width, 3), np.float32)
        tr = np.zeros((cam.height, cam.width), np.float32)
        cn = np.zeros((cam.height, cam.width), np.int32)
        cc = cam.to_c()
        self.L._check(self.L.dll.slm_scene_render(self.h, C.byref(cc), f32ptr(img), f32ptr(tr), i32ptr(cn)))
        return img, tr, cn

    def lm_step(self, data: "TrainData", cfg: LmConfig, iteration: int, rng: Rng) -> StepReport:
        batch = np.zeros(4096, np.int32)
        rep = CStepReport()
        rep.batch, rep.batch_capacity = i32ptr(batch), batch.size
        cc = cfg.to_c()
        self.L._check(self.L.dll.slm_lm_step(self.h, data.h, C.byref(cc), iteration, rng.h, C.byref(rep)))
        return _report(rep, batch)

    def batch_loss(self, data: "TrainData", cam_ids, loss: int = 0, ssim_weight: float = 0.0) -> float:
        """solver::batch_loss (lm.cpp:39-54); loss 1 = mse+ssim (diagonal SSIM residuals)."""
        ids = np.ascontiguousarray(cam_ids, np.int32)
        out = C.c_double()
        self.L._check(self.L.dll.slm_batch_loss_kind(self.h, data.h, i32ptr(ids), ids.size, loss, ssim_weight,
                                                     C.byref(out)))
        return out.value

    def jacobian(self, cams, plan: SamplePlan) -> "Jacobian":
        return Jacobian(self.L, None, cams, plan, scene=self)

    def full_gradient(self, data: "TrainData", loss: int = 0, ssim_weight: float = 0.2) -> np.ndarray:
        out = np.zeros(14 * self.count)
        self.L._check(self.L.dll.slm_full_gradient(self.h, data.h, loss, ssim_weight, f64ptr(out)))
        return out

    def evaluate_split(self, split: "TrainData") -> MetricReport:
        """io::evaluate_split (run.cpp:77-92): mean mse / psnr / ssim over the split's cameras,
        rendered and scored on the device."""
        r = CMetricReport()
        self.L._check(self.L.dll.slm_evaluate_split(self.h, split.h, C.byref(r)))
        return MetricReport(r.mse, r.psnr, r.ssim)


class FirstOrder:
    """baselines::FirstOrderState (first_order.hpp:39-51) in HBM, bound to a device scene."""

    def __init__(self, L: Lib, scene: Scene):
        self.L, self.scene = L, scene
        h = _vp()
        L._check(L.dll.slm_first_order_create(scene.h, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.L.dll.slm_first_order_destroy(self.h)
        except Exception:
            pass

    def step(self, data: "TrainData", cfg) -> float:
        """full_gradient + first_order_step + batch_loss (run.cpp:176-182); returns the train loss."""
        out = C.c_double()
        cc = cfg.to_c()
        self.L._check(self.L.dll.slm_first_order_step(self.h, data.h, C.byref(cc), C.byref(out)))
        return out.value

    def apply(self, grad, cfg) -> None:
        g = np.ascontiguousarray(grad, np.float64)
        cc = cfg.to_c()
        self.L._check(self.L.dll.slm_first_order_apply(self.h, f64ptr(g), C.byref(cc)))

    def moments(self):
        n = 14 * self.scene.count
        m1, m2, st = np.zeros(n), np.zeros(n), C.c_int64()
        self.L._check(self.L.dll.slm_first_order_moments(self.h, f64ptr(m1), f64ptr(m2), C.byref(st)))
        return m1, m2, st.value

    def set_moments(self, m1, m2, step: int) -> None:
        a = np.ascontiguousarray(m1, np.float64)
        b = np.ascontiguousarray(m2, np.float64)
        self.L._check(self.L.dll.slm_first_order_set_moments(self.h, f64ptr(a), f64ptr(b), step))


class Jacobian:
    """autodiff::SampledJacobian (jacobian.hpp:25-76) on the B200."""

    def __init__(self, L: Lib, g: GaussianSet | None, cams, plan: SamplePlan, scene: Scene | None = None):
        self.L = L
        cp = plan.to_c()
        self._plan = plan
        h = _vp()
        if scene is None:
            cg = g.to_c()
            L._check(L.dll.slm_jacobian_create(L.ctx, C.byref(cg), cameras_to_c(cams), len(cams),
                                               C.byref(cp), C.byref(h)))
        else:
            self._scene = scene
            L._check(L.dll.slm_jacobian_create_scene(scene.h, cameras_to_c(cams), len(cams),
                                                     C.byref(cp), C.byref(h)))
        self.h = h
        r, p = C.c_int64(), C.c_int64()
        L.dll.slm_jacobian_dims(h, C.byref(r), C.byref(p))
        self.rdim, self.pdim = r.value, p.value

    def __del__(self):
        try:
            self.L.dll.slm_jacobian_destroy(self.h)
        except Exception:
            pass

    def residual_dim(self) -> int:
        return self.rdim

    def param_dim(self) -> int:
        return self.pdim

    def jvp(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float64)
        if v.size != self.pdim:
            raise ValueError("jvp: probe vector length mismatch")
        out = np.zeros(self.rdim)
        self.L._check(self.L.dll.slm_jacobian_jvp(self.h, f64ptr(v), f64ptr(out)))
        return out

    def vjp(self, u) -> np.ndarray:
        u = np.ascontiguousarray(u, np.float64)
        if u.size != self.rdim:
            raise ValueError("vjp: input length mismatch")
        out = np.zeros(self.pdim)
        self.L._check(self.L.dll.slm_jacobian_vjp(self.h, f64ptr(u), f64ptr(out)))
        return out

    def jtj_diag(self) -> np.ndarray:
        out = np.zeros(self.pdim)
        self.L._check(self.L.dll.slm_jacobian_jtj_diag(self.h, f64ptr(out)))
        return out

    def gn_apply(self, lam: float, p, out=None) -> np.ndarray:
        """J^T W J p + lam p on host f64 ParamVectors; `out` (optional, f64
        contiguous, e.g. a pinned buffer) receives the result in place."""
        p = np.ascontiguousarray(p, np.float64)
        if p.size != self.pdim:
            raise ValueError("gn_apply: probe vector length mismatch")
        if out is None:
            out = np.zeros(self.pdim)
        elif out.dtype != np.float64 or out.size != self.pdim or not out.flags.c_contiguous:
            raise ValueError("gn_apply: out must be a contiguous f64 vector of param_dim")
        self.L._check(self.L.dll.slm_jacobian_gn_apply(self.h, lam, f64ptr(p), f64ptr(out)))
        return out

    def gn_apply_dev(self, lam: float, d_p: int, d_out: int):
        """Device-resident product on f32 SoA [14][Gp] vectors (device pointers)."""
        self.L._check(self.L.dll.slm_jacobian_gn_apply_dev(self.h, lam, _vp(d_p), _vp(d_out)))

    def residual_weights(self) -> np.ndarray:
        out = np.zeros(self.rdim)
        self.L._check(self.L.dll.slm_jacobian_weights(self.h, f64ptr(out)))
        return out

    def set_residual_weights(self, w) -> None:
        w = np.ascontiguousarray(w, np.float64)
        if w.size != self.rdim:
            raise ValueError("residual weight vector has wrong length")
        self.L._check(self.L.dll.slm_jacobian_set_weights(self.h, f64ptr(w)))

    def pcg(self, lam, b, minv, iters) -> PcgResult:
        b = np.ascontiguousarray(b, np.float64)
        minv = np.ascontiguousarray(minv, np.float64)
        x = np.zeros(self.pdim)
        r = CPcgResult()
        self.L._check(self.L.dll.slm_jacobian_pcg(self.h, lam, f64ptr(b), f64ptr(minv), iters, f64ptr(x),
                                                  C.byref(r)))
        return PcgResult(x, r.iterations, bool(r.breakdown), r.rel_residual)

    def stats(self) -> dict:
        out = np.zeros(6, np.int64)
        self.L.dll.slm_jacobian_stats(self.h, i64ptr(out))
        return dict(views=int(out[0]), valid=int(out[1]), entries=int(out[2]), samples=int(out[3]), groups=int(out[4]),
                    tiles=int(out[5]))

    def mask_stats(self) -> dict:
        """Diagnostic counters of the blend masks (raster.cu k_mask_stats)."""
        out = np.zeros(18, np.int64)
        self.L._check(self.L.dll.slm_jacobian_mask_stats(self.h, i64ptr(out)))
        keys = ["groups", "windows", "pairs", "it_walk", "entries", "it_walk64", "it_col",
                "rows_le8", "rows_le16", "rows_le20", "rows_le24", "rows_le28", "rows_le32",
                "it_win64", "it_ahead1", "it_ahead3", "it_ahead_inf", "it_pair_iters"]
        return dict(zip(keys, (int(x) for x in out)))


class TrainData:
    """solver::TrainData: cameras + f32 dataset images resident in HBM + clusters."""

    def __init__(self, L: Lib, cams, images):
        self.L = L
        self.cameras = list(cams)
        buf = np.ascontiguousarray(np.concatenate([np.asarray(im, np.float32).reshape(-1) for im in images]))
        h = _vp()
        L._check(L.dll.slm_train_create(L.ctx, cameras_to_c(cams), len(cams), f32ptr(buf), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.L.dll.slm_train_destroy(self.h)
        except Exception:
            pass

    def rebuild_clusters(self, k: int, seed: int) -> None:
        self.L._check(self.L.dll.slm_train_rebuild_clusters(self.h, k, seed))

    def set_clusters(self, clusters) -> None:
        assign = np.zeros(len(self.cameras), np.int32)
        for c, m in enumerate(clusters):
            assign[list(m)] = c
        self.L._check(self.L.dll.slm_train_set_clusters(self.h, i32ptr(assign), len(clusters)))

    def clusters(self) -> list:
        assign = np.zeros(len(self.cameras), np.int32)
        k = C.c_int32()
        self.L._check(self.L.dll.slm_train_clusters(self.h, i32ptr(assign), C.byref(k)))
        return [list(np.nonzero(assign == c)[0]) for c in range(k.value)]


_default: dict = {}


def lib(device: int = 0) -> Lib:
    """The process-wide context on `device` (fails loudly without a GPU)."""
    if device not in _default:
        _default[device] = Lib(device)
    return _default[device]
