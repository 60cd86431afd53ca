"""ctypes mirrors of include/slm_types.h plus small numpy-backed value types.

The Python classes follow the reference C++ structs field for field so host
code and tests read like the reference's own:

* :class:`Camera`       <- ``splatlm::Camera``       (proj/include/splatlm/core/types.hpp:61-75)
* :class:`GaussianSet`  <- ``splatlm::GaussianSet``  (types.hpp:31-57, pack/unpack types.cpp:20-46)
* :class:`SamplePlan`   <- ``sampling::SamplePlan``  (sample_plan.hpp:22-37)
* :class:`LmConfig`     <- ``solver::LmConfig``      (lm.hpp:14-40)
* :class:`StepReport`   <- ``solver::StepReport``    (lm.hpp:42-50)
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

PARAMS_PER_GAUSSIAN = 14
MEAN_OFFSET, LOG_SCALE_OFFSET, ROTATION_OFFSET, OPACITY_OFFSET, COLOR_OFFSET = 0, 3, 6, 10, 11
COLOR_C0 = 0.28209479177387814  # types.hpp:24
TILE = 16                        # rasterizer.hpp:14

DIST_UNIFORM, DIST_RESIDUAL, DIST_GAUSSIAN_COUNT = 0, 1, 2
LOSS_MSE, LOSS_MSE_SSIM = 0, 1

_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class CCamera(C.Structure):
    _fields_ = [("world_to_cam", C.c_double * 9), ("translation", C.c_double * 3),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("near_clip", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class CGaussians(C.Structure):
    _fields_ = [("count", C.c_int32), ("means", _f64p), ("log_scales", _f64p),
                ("rotations", _f64p), ("opacity_logits", _f64p), ("colors", _f64p)]


class CPlan(C.Structure):
    _fields_ = [("n_views", C.c_int32), ("samples_per_tile", C.c_int32), ("dist", C.c_int32),
                ("view_camera", _i32p), ("view_offset", _i64p), ("px", _i32p), ("py", _i32p),
                ("tile", _i32p), ("weight", _f64p)]


class CLmConfig(C.Structure):
    _fields_ = [("damping", C.c_double), ("pcg_iters_initial", C.c_int32),
                ("pcg_iters_late", C.c_int32), ("pcg_switch_iteration", C.c_int32),
                ("batch_size_initial", C.c_int32), ("batch_size_late", C.c_int32),
                ("batch_switch_iteration", C.c_int32), ("samples_per_tile", C.c_int32),
                ("sample_lane_width", C.c_int32), ("lr_cap", C.c_double),
                ("warmup_lr", C.c_double), ("warmup_iterations", C.c_int32),
                ("dist", C.c_int32), ("loss", C.c_int32), ("ssim_weight", C.c_double)]


class CFirstOrderConfig(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lr_mean", C.c_double), ("lr_color", C.c_double),
                ("lr_opacity", C.c_double), ("lr_scale", C.c_double), ("lr_rotation", C.c_double),
                ("adam_beta1", C.c_double), ("adam_beta2", C.c_double), ("adam_eps", C.c_double),
                ("rms_decay", C.c_double), ("rms_eps", C.c_double), ("momentum", C.c_double),
                ("mean_lr_final_factor", C.c_double), ("decay_iterations", C.c_int32),
                ("loss", C.c_int32), ("ssim_weight", C.c_double)]


class CStepReport(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("loss_before", C.c_double),
                ("loss_after", C.c_double), ("eta", C.c_double), ("pcg_iterations", C.c_int32),
                ("breakdown", C.c_int32), ("batch_size", C.c_int32), ("batch", _i32p),
                ("batch_capacity", C.c_int32)]


class CMetricReport(C.Structure):
    _fields_ = [("mse", C.c_double), ("psnr", C.c_double), ("ssim", C.c_double)]


class CPcgResult(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("breakdown", C.c_int32),
                ("rel_residual", C.c_double)]


def f64ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_f64p)


def i32ptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_i32p)


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def f32ptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_float))


@dataclass
class Camera:
    """Pinhole camera; world_to_cam maps world points to x right, y down, z forward."""
    world_to_cam: np.ndarray = field(default_factory=lambda: np.eye(3).reshape(9))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    near_clip: float = 0.2

    def to_c(self) -> CCamera:
        c = CCamera()
        for i in range(9):
            c.world_to_cam[i] = float(self.world_to_cam[i])
        for i in range(3):
            c.translation[i] = float(self.translation[i])
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.near_clip = float(self.near_clip)
        c.width, c.height = int(self.width), int(self.height)
        return c

    @staticmethod
    def from_c(c: CCamera) -> "Camera":
        return Camera(np.array(c.world_to_cam[:]), np.array(c.translation[:]), c.fx, c.fy, c.cx,
                      c.cy, c.width, c.height, c.near_clip)

    @property
    def tiles_x(self) -> int:
        return (self.width + TILE - 1) // TILE

    @property
    def tiles_y(self) -> int:
        return (self.height + TILE - 1) // TILE

    def position(self) -> np.ndarray:
        r = np.asarray(self.world_to_cam).reshape(3, 3)
        return -(r.T @ np.asarray(self.translation))

    def validate(self) -> None:
        """Camera::validate (types.cpp:89-101)."""
        if self.width <= 0 or self.height <= 0:
            raise ValueError("camera size must be positive")
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("camera focal must be positive")
        r = np.asarray(self.world_to_cam).reshape(3, 3)
        if np.max(np.abs(r @ r.T - np.eye(3))) > 1e-6:
            raise ValueError("camera rotation is not orthonormal")


def cameras_to_c(cams) -> C.Array:
    arr = (CCamera * max(1, len(cams)))()
    for i, cam in enumerate(cams):
        arr[i] = cam.to_c()
    return arr


def ring_camera(angle: float, radius: float, height: float, width: int, height_px: int | None = None) -> Camera:
    """Camera on a ring looking at the origin, io::ring_camera (scene_gen.cpp:11-36).

    ``height_px`` allows the non-square shapes BASELINE.json names (the
    reference generator is square-only, scene_gen.cpp:30-33); with it unset the
    result is the reference camera bit for bit (same double operation order).
    """
    pos = np.array([radius * math.cos(angle), height, radius * math.sin(angle)])
    fwd = np.array([0.0 - pos[0], 0.0 - pos[1], 0.0 - pos[2]])  # target - pos, signed zeros as C++
    fn =math.sqrt(fwd[0] * fwd[0] + fwd[1] * fwd[1] + fwd[2] * fwd[2])
    fwd = np.array([fwd[0] / fn, fwd[1] / fn, fwd[2] / fn])
    up = np.array([0.0, 1.0, 0.0])

    def cross(u, v):
        return np.array([u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2],
                         u[0] * v[1] - u[1] * v[0]])

    right = cross(fwd, up)
    rn = math.sqrt(right[0] * right[0] + right[1] * right[1] + right[2] * right[2])
    right = np.array([right[0] / rn, right[1] / rn, right[2] / rn])
    down = cross(fwd, right)
    r = np.array([right[0], right[1], right[2], down[0], down[1], down[2], fwd[0], fwd[1], fwd[2]])
    t = np.array([-(r[3 * k] * pos[0] + r[3 * k + 1] * pos[1] + r[3 * k + 2] * pos[2])
                  for k in range(3)])
    h = width if height_px is None else height_px
    fov_x = 50.0 * math.pi / 180.0
    f = 0.5 * width / math.tan(0.5 * fov_x)
    cam = Camera(r, t, f, f, 0.5 * width, 0.5 * h, width, h)
    cam.validate()
    return cam


class GaussianSet:
    """Raw (pre-activation) SoA parameters; mirrors splatlm::GaussianSet."""

    def __init__(self, count: int):
        self.count = int(count)
        self.means = np.zeros(3 * count)
        self.log_scales = np.zeros(3 * count)
        self.rotations = np.zeros(4 * count)
        self.rotations[0::4] = 1.0
        self.opacity_logits = np.zeros(count)
        self.colors = np.zeros(3 * count)

    @staticmethod
    def zeros(count: int) -> "GaussianSet":
        return GaussianSet(count)

    def copy(self) -> "GaussianSet":
        g = GaussianSet(self.count)
        for k in ("means", "log_scales", "rotations", "opacity_logits", "colors"):
            setattr(g, k, getattr(self, k).copy())
        return g

    def param_count(self) -> int:
        return PARAMS_PER_GAUSSIAN * self.count

    def pack(self) -> np.ndarray:
        """AoS 14-stride ParamVector (types.cpp:20-31)."""
        v = np.empty((self.count, PARAMS_PER_GAUSSIAN))
        v[:, 0:3] = self.means.reshape(-1, 3)
        v[:, 3:6] = self.log_scales.reshape(-1, 3)
        v[:, 6:10] = self.rotations.reshape(-1, 4)
        v[:, 10] = self.opacity_logits
        v[:, 11:14] = self.colors.reshape(-1, 3)
        return v.reshape(-1)

    @staticmethod
    def unpack(v: np.ndarray) -> "GaussianSet":
        if v.size % PARAMS_PER_GAUSSIAN != 0:
            raise ValueError("parameter vector length is not a multiple of 14")
        b = np.asarray(v, dtype=np.float64).reshape(-1, PARAMS_PER_GAUSSIAN)
        g = GaussianSet(b.shape[0])
        g.means = np.ascontiguousarray(b[:, 0:3]).reshape(-1)
        g.log_scales = np.ascontiguousarray(b[:, 3:6]).reshape(-1)
        g.rotations = np.ascontiguousarray(b[:, 6:10]).reshape(-1)
        g.opacity_logits = np.ascontiguousarray(b[:, 10])
        g.colors = np.ascontiguousarray(b[:, 11:14]).reshape(-1)
        return g

    def renormalize_rotations(self) -> None:
        """types.cpp:62-73."""
        q = self.rotations.reshape(-1, 4)
        for i in range(q.shape[0]):
            n = math.sqrt(q[i, 0] * q[i, 0] + q[i, 1] * q[i, 1] + q[i, 2] * q[i, 2] + q[i, 3] * q[i, 3])
            if n == 0.0:
                q[i] = (1.0, 0.0, 0.0, 0.0)
            else:
                q[i] /= n

    def to_c(self) -> CGaussians:
        for k in ("means", "log_scales", "rotations", "opacity_logits", "colors"):
            a = getattr(self, k)
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                setattr(self, k, np.ascontiguousarray(a, dtype=np.float64))
        return CGaussians(self.count, f64ptr(self.means), f64ptr(self.log_scales),
                          f64ptr(self.rotations), f64ptr(self.opacity_logits), f64ptr(self.colors))

    def __eq__(self, other) -> bool:  # bitwise, like comparing pack() vectors
        return isinstance(other, GaussianSet) and np.array_equal(self.pack(), other.pack())


@dataclass
class SamplePlan:
    """Flattened sampling::SamplePlan: view v owns samples view_offset[v]:view_offset[v+1]."""
    view_camera: np.ndarray
    view_offset: np.ndarray
    px: np.ndarray
    py: np.ndarray
    tile: np.ndarray
    weight: np.ndarray
    samples_per_tile: int = 0
    dist: int = DIST_UNIFORM

    @property
    def n_views(self) -> int:
        return int(self.view_camera.size)

    def total_samples(self) -> int:
        return int(self.view_offset[-1])

    def view(self, v: int):
        a, b = int(self.view_offset[v]), int(self.view_offset[v + 1])
        return self.px[a:b], self.py[a:b], self.tile[a:b], self.weight[a:b]

    def to_c(self) -> CPlan:
        self.view_camera = np.ascontiguousarray(self.view_camera, dtype=np.int32)
        self.view_offset = np.ascontiguousarray(self.view_offset, dtype=np.int64)
        for k in ("px", "py", "tile"):
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=np.int32))
        self.weight = np.ascontiguousarray(self.weight, dtype=np.float64)
        return CPlan(self.n_views, self.samples_per_tile, self.dist, i32ptr(self.view_camera),
                     i64ptr(self.view_offset), i32ptr(self.px), i32ptr(self.py), i32ptr(self.tile),
                     f64ptr(self.weight))

    @staticmethod
    def single(camera: int, px, py, tile, weight, samples_per_tile=1) -> "SamplePlan":
        n = len(px)
        return SamplePlan(np.array([camera], np.int32), np.array([0, n], np.int64),
                          np.asarray(px, np.int32), np.asarray(py, np.int32),
                          np.asarray(tile, np.int32), np.asarray(weight, np.float64),
                          samples_per_tile)


@dataclass
class LmConfig:
    damping: float = 0.1
    pcg_iters_initial: int = 3
    pcg_iters_late: int = 8
    pcg_switch_iteration: int = 50
    batch_size_initial: int = 8
    batch_size_late: int = 8
    batch_switch_iteration: int = 50
    samples_per_tile: int = 32
    sample_lane_width: int = 32
    lr_cap: float = 0.2
    warmup_lr: float = 0.05
    warmup_iterations: int = 10
    dist: int = DIST_UNIFORM
    loss: int = LOSS_MSE
    ssim_weight: float = 0.2

    def pcg_iters_at(self, iteration: int) -> int:
        return self.pcg_iters_late if iteration >= self.pcg_switch_iteration else self.pcg_iters_initial

    def batch_size_at(self, iteration: int) -> int:
        return self.batch_size_late if iteration >= self.batch_switch_iteration else self.batch_size_initial

    @staticmethod
    def real_world_preset() -> "LmConfig":
        """lm.cpp:13-19."""
        return LmConfig(pcg_iters_initial=5, batch_size_initial=16, batch_size_late=32)

    def to_c(self) -> CLmConfig:
        c = CLmConfig()
        for name, _ in CLmConfig._fields_:
            setattr(c, name, getattr(self, name))
        return c


@dataclass
class StepReport:
    iteration: int = 0
    loss_before: float = 0.0
    loss_after: float = 0.0
    eta: float = 0.0
    pcg_iterations: int = 0
    breakdown: bool = False
    batch: list = field(default_factory=list)


FO_ADAM, FO_RMSPROP, FO_SGD_MOMENTUM = 0, 1, 2


@dataclass
class FirstOrderConfig:
    """baselines::FirstOrderConfig (first_order.hpp:12-37)."""
    kind: int = FO_ADAM
    lr_mean: float = 1.6e-3
    lr_color: float = 2.5e-2
    lr_opacity: float = 5e-2
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-15
    rms_decay: float = 0.99
    rms_eps: float = 1e-15
    momentum: float = 0.99
    mean_lr_final_factor: float = 0.01
    decay_iterations: int = 0
    loss: int = LOSS_MSE
    ssim_weight: float = 0.2

    @staticmethod
    def sgd_paper_lrs() -> dict:
        """first_order.hpp:36 (mean, color, opacity, scale, rotation)."""
        return dict(lr_mean=0.16, lr_color=0.2, lr_opacity=0.1, lr_scale=0.1, lr_rotation=0.1)

    def to_c(self) -> CFirstOrderConfig:
        c = CFirstOrderConfig()
        for name, _ in CFirstOrderConfig._fields_:
            setattr(c, name, getattr(self, name))
        return c


@dataclass
class MetricReport:
    """metrics::MetricReport (image_metrics.hpp:7-11)."""
    mse: float = 0.0
    psnr: float = 0.0
    ssim: float = 0.0


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int = 0
    breakdown: bool = False
    rel_residual: float = 1.0
