"""paper_2205_02646_b200 -- B200-native RL-JSDE reconstruction (arXiv 2205.02646).

Python face of ``libtqsb.so`` (C ABI in ``include/tqsb/tqsb.h``), mirroring the
reference entry point ``tqs::reconstruct(frame, pattern, config, cache, reference)``
(/root/reference/proj/include/tqs/pipeline.hpp:45-47) and its types:

* ``ReconstructionConfig`` -- pipeline.hpp:17-26 (+ SolverOptions, WeightingConfig)
* ``ReconstructionReport`` -- pipeline.hpp:28-39
* ``Plan``                 -- the external KernelCache (rljsde.hpp:81-100): tables
                              resident on the GPU(s), reused across calls
* ``reconstruct``          -- pipeline.cpp:62-185, errors raised as the reference's
                              exception types (ValueError for std::invalid_argument)

The compute path is CUDA only: importing works without a GPU (host helpers such
as ``census`` and ``generate_pattern`` run anywhere), but every reconstruction
raises ``NoDeviceError`` when no CUDA device is present -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# TQSB_LIB selects an experiment variant built by build.py (default: the product library)
LIB_PATH = os.environ.get("TQSB_LIB") or os.path.join(HERE, "libtqsb.so")

TQSB_OK, TQSB_EINVAL, TQSB_ECUDA, TQSB_ENOMEM, TQSB_ELOGIC, TQSB_ENODEV, TQSB_EIO = range(7)


class TqsbError(RuntimeError):
    """CUDA / memory failures (std::runtime_error in the reference)."""


class NoDeviceError(TqsbError):
    """No CUDA device: the library has no CPU fallback."""


class LogicError(RuntimeError):
    """std::logic_error (pipeline.cpp:146-147)."""


class FormatError(RuntimeError):
    """File-format / I/O failure (std::runtime_error "<path>: <what>", io.cpp:15-31)."""


class _Config(C.Structure):
    _fields_ = [("window", C.c_int), ("block", C.c_int), ("max_iterations", C.c_int),
                ("step_width", C.c_double), ("spatial_decay", C.c_double),
                ("frequency_exponent", C.c_double), ("precision", C.c_int),
                ("clip_output", C.c_int), ("threads", C.c_int), ("compute", C.c_int),
                ("hot_columns", C.c_int), ("algorithm", C.c_int), ("early_stop", C.c_int),
                ("early_stop_scale", C.c_double)]


class _Report(C.Structure):
    _fields_ = [("seconds", C.c_double), ("warm_seconds", C.c_double),
                ("e2e_seconds", C.c_double), ("blocks_processed", C.c_longlong),
                ("classes_total", C.c_longlong), ("classes_interior", C.c_longlong),
                ("classes_created", C.c_longlong), ("cache_hits", C.c_longlong),
                ("cache_misses", C.c_longlong), ("psnr_db", C.c_double), ("has_psnr", C.c_int),
                ("gpu_launches", C.c_int), ("compute", C.c_int)]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)

EXPORTS = [
    "tqsb_last_error", "tqsb_version", "tqsb_config_default", "tqsb_validate_config",
    "tqsb_census", "tqsb_plan_create", "tqsb_plan_destroy", "tqsb_reconstruct",
    "tqsb_reconstruct_band", "tqsb_reconstruct_device", "tqsb_reconstruct_band_device",
    "tqsb_plan_warm", "tqsb_plan_stats", "tqsb_plan_export_tables", "tqsb_plan_block_trace",
    "tqsb_generate_pattern", "tqsb_simulate", "tqsb_synthetic_image", "tqsb_psnr",
    "tqsb_host_alloc", "tqsb_host_free", "tqsb_device_count", "tqsb_probe_peaks",
    "tqsb_reconstruct_batch",
    "tqsb_io_read", "tqsb_io_write_pgm", "tqsb_io_write_tqsm", "tqsb_io_read_pattern",
    "tqsb_io_write_pattern", "tqsb_plan_save_tables", "tqsb_plan_load_tables",
    "tqsb_pattern_digest", "tqsb_kernel_memory_report", "tqsb_synthetic_image_device",
    "tqsb_plan_simulate_device", "tqsb_reconstruct_with", "tqsb_reconstruct_batch_with",
    "tqsb_reconstruct_band_with", "tqsb_reconstruct_device_with",
]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2205_02646_b200/build.py` "
            "(the CUDA extension is required; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.tqsb_last_error.restype = C.c_char_p
    L.tqsb_version.restype = C.c_char_p
    L.tqsb_config_default.argtypes = [C.POINTER(_Config)]
    L.tqsb_config_default.restype = None
    L.tqsb_validate_config.argtypes = [C.POINTER(_Config), C.c_int]
    L.tqsb_census.argtypes = [C.c_int, C.c_int, C.POINTER(_Config), C.c_int,
                              C.POINTER(C.c_longlong)]
    L.tqsb_plan_create.argtypes = [_u8p, C.c_int, C.POINTER(_Config), _ip, C.c_int,
                                   C.POINTER(C.c_void_p)]
    L.tqsb_plan_destroy.argtypes = [C.c_void_p]
    L.tqsb_reconstruct.argtypes = [C.c_void_p, _dp, C.c_int, C.c_int, _dp, _dp,
                                   C.POINTER(_Report)]
    L.tqsb_reconstruct_band.argtypes = [C.c_void_p, _dp, C.c_int, C.c_int, C.c_int, C.c_int,
                                        _dp, C.POINTER(_Report)]
    L.tqsb_reconstruct_with.argtypes = [C.c_void_p, C.POINTER(_Config), _dp, C.c_int, C.c_int,
                                        _dp, _dp, C.POINTER(_Report)]
    L.tqsb_reconstruct_band_with.argtypes = [C.c_void_p, C.POINTER(_Config), _dp, C.c_int,
                                             C.c_int, C.c_int, C.c_int, _dp, C.POINTER(_Report)]
    L.tqsb_reconstruct_batch_with.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(_dp),
                                              C.c_int, C.c_int, C.c_int, C.POINTER(_dp),
                                              C.POINTER(_Report)]
    L.tqsb_reconstruct_device_with.argtypes = [C.c_void_p, C.POINTER(_Config), C.c_void_p,
                                               C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                               C.POINTER(_Report)]
    L.tqsb_reconstruct_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                          C.c_void_p, C.POINTER(_Report)]
    L.tqsb_reconstruct_band_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                               C.c_int, C.c_void_p, C.c_void_p,
                                               C.POINTER(_Report)]
    L.tqsb_plan_warm.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
    L.tqsb_plan_stats.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
    L.tqsb_plan_export_tables.argtypes = [C.c_void_p, C.c_int, C.c_int, _ip, _dp, _dp, _dp, _dp,
                                          _dp]
    L.tqsb_plan_block_trace.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _ip, _dp, _dp, _ip]
    L.tqsb_generate_pattern.argtypes = [C.c_uint64, C.c_int, C.c_int, _u8p]
    L.tqsb_simulate.argtypes = [_dp, C.c_int, C.c_int, _u8p, C.c_int, _dp]
    L.tqsb_synthetic_image.argtypes = [C.c_int, C.c_int, C.c_uint64, _dp]
    L.tqsb_psnr.argtypes = [_dp, _dp, C.c_longlong]
    L.tqsb_psnr.restype = C.c_double
    L.tqsb_host_alloc.argtypes = [C.c_size_t]
    L.tqsb_host_alloc.restype = C.c_void_p
    L.tqsb_host_free.argtypes = [C.c_void_p]
    L.tqsb_host_free.restype = None
    L.tqsb_probe_peaks.argtypes = [C.c_int, _dp, _dp]
    L.tqsb_reconstruct_batch.argtypes = [C.c_void_p, C.POINTER(_dp), C.c_int, C.c_int, C.c_int,
                                         C.POINTER(_dp), C.POINTER(_Report)]
    L.tqsb_io_read.argtypes = [C.c_char_p, C.c_int, _ip, _ip, _dp]
    L.tqsb_io_write_pgm.argtypes = [C.c_char_p, _dp, C.c_int, C.c_int, C.c_int]
    L.tqsb_io_write_tqsm.argtypes = [C.c_char_p, _dp, C.c_int, C.c_int]
    L.tqsb_io_read_pattern.argtypes = [C.c_char_p, _ip, C.POINTER(C.c_uint64), C.c_char_p,
                                       C.c_size_t, _u8p]
    L.tqsb_io_write_pattern.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_char_p, _u8p]
    L.tqsb_plan_save_tables.argtypes = [C.c_void_p, C.c_char_p, _ip]
    L.tqsb_plan_load_tables.argtypes = [C.c_void_p, C.c_char_p, _ip]
    L.tqsb_pattern_digest.argtypes = [_u8p, C.c_int]
    L.tqsb_pattern_digest.restype = C.c_uint64
    L.tqsb_kernel_memory_report.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.POINTER(C.c_uint64)]
    L.tqsb_synthetic_image_device.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p,
                                              C.c_void_p]
    L.tqsb_plan_simulate_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                            C.c_void_p]
    return L


lib = _load()


def _check(rc: int) -> None:
    if rc == TQSB_OK:
        return
    msg = lib.tqsb_last_error().decode()
    if rc == TQSB_EINVAL:
        raise ValueError(msg)
    if rc == TQSB_ELOGIC:
        raise LogicError(msg)
    if rc == TQSB_ENODEV:
        raise NoDeviceError(msg)
    if rc == TQSB_EIO:
        raise FormatError(msg)
    raise TqsbError(msg)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _out_array(out, shape, what="out"):
    """A caller-supplied output buffer: the kernels and staging copies store straight
    into it, so it must be exactly a C-contiguous float64 array of the output shape."""
    if out is None:
        return np.empty(shape)
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or \
            not out.flags.c_contiguous or not out.flags.writeable or tuple(out.shape) != tuple(shape):
        raise ValueError(f"{what} must be a writeable C-contiguous float64 array of shape "
                         f"{tuple(shape)}")
    return out


COMPUTE_FP32, COMPUTE_FP64 = 0, 1
PRECISION_SINGLE, PRECISION_DOUBLE = 0, 1
ALGO_LJSDE, ALGO_RLJSDE = 0, 1


@dataclasses.dataclass
class ReconstructionConfig:
    """pipeline.hpp:17-26 with SolverOptions / WeightingConfig flattened."""
    window: int = 32
    block: int = 4
    max_iterations: int = 200
    step_width: float = 0.5
    spatial_decay: float = 0.8
    frequency_exponent: float = 2.0
    precision: int = PRECISION_DOUBLE
    clip_output: bool = True
    threads: int = 1
    compute: int = COMPUTE_FP32
    hot_columns: int = -1
    algorithm: int = ALGO_RLJSDE
    early_stop: bool = False
    early_stop_scale: float = 1e-14

    def _c(self) -> _Config:
        return _Config(self.window, self.block, self.max_iterations, self.step_width,
                       self.spatial_decay, self.frequency_exponent, self.precision,
                       int(self.clip_output), self.threads, self.compute, self.hot_columns,
                       self.algorithm, int(self.early_stop), self.early_stop_scale)


@dataclasses.dataclass
class ReconstructionReport:
    """pipeline.hpp:28-39 (output image included, psnr None unless a reference is given)."""
    output: np.ndarray
    seconds: float
    warm_seconds: float
    e2e_seconds: float
    blocks_processed: int
    classes_total: int
    classes_interior: int
    classes_created: int
    cache_hits: int
    cache_misses: int
    psnr_db: float | None
    gpu_launches: int
    compute: int = 0  # COMPUTE_* the call actually ran in


def _report(out, r: _Report) -> ReconstructionReport:
    return ReconstructionReport(out, r.seconds, r.warm_seconds, r.e2e_seconds, r.blocks_processed,
                                r.classes_total, r.classes_interior, r.classes_created,
                                r.cache_hits, r.cache_misses,
                                r.psnr_db if r.has_psnr else None, r.gpu_launches, r.compute)


@dataclasses.dataclass
class QuadrantPattern:
    """grid.hpp:19-34: period in HR pixels, (period/2)^2 opaque quadrant indices."""
    period: int
    opaque: np.ndarray
    seed: int = 0
    rng: str = "mt19937_64"


def generate_pattern(seed: int, period: int, block: int = 4) -> QuadrantPattern:
    out = np.zeros((period // 2) ** 2, np.uint8)
    _check(lib.tqsb_generate_pattern(seed, period, block, out.ctypes.data_as(_u8p)))
    return QuadrantPattern(period, out, seed)


def simulate_measurement(image: np.ndarray, pattern: QuadrantPattern) -> np.ndarray:
    image = np.ascontiguousarray(image, np.float64)
    out = np.zeros((image.shape[0] // 2, image.shape[1] // 2))
    _check(lib.tqsb_simulate(_d(image), image.shape[0], image.shape[1],
                             pattern.opaque.ctypes.data_as(_u8p), pattern.period, _d(out)))
    return out


def synthetic_image(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.zeros((rows, cols))
    _check(lib.tqsb_synthetic_image(rows, cols, seed, _d(out)))
    return out


def synthetic_image_device(rows: int, cols: int, seed: int, d_out_ptr: int, device: int = 0,
                           stream: int = 0) -> None:
    """The synthetic scene evaluated on a device into d_out (rows x cols float64)."""
    _check(lib.tqsb_synthetic_image_device(device, rows, cols, seed, C.c_void_p(d_out_ptr),
                                           C.c_void_p(stream)))


def psnr(reference: np.ndarray, estimate: np.ndarray) -> float:
    reference = np.ascontiguousarray(reference, np.float64)
    estimate = np.ascontiguousarray(estimate, np.float64)
    if reference.shape != estimate.shape:
        raise ValueError("psnr: dimension mismatch")
    return lib.tqsb_psnr(_d(reference), _d(estimate), reference.size)


def validate_config(config: ReconstructionConfig, period: int) -> None:
    c = config._c()
    _check(lib.tqsb_validate_config(C.byref(c), period))


def census(frame_rows: int, frame_cols: int, config: ReconstructionConfig, period: int) -> dict:
    c = config._c()
    out = (C.c_longlong * 3)()
    _check(lib.tqsb_census(frame_rows, frame_cols, C.byref(c), period, out))
    return dict(blocks=out[0], classes_total=out[1], classes_interior=out[2])


def pattern_digest(pattern: QuadrantPattern) -> int:
    """FNV-1a content digest of a pattern (rljsde.cpp:322-333), pinned in TQSK headers."""
    opq = np.ascontiguousarray(pattern.opaque, np.uint8)
    return lib.tqsb_pattern_digest(opq.ctypes.data_as(_u8p), pattern.period)


def kernel_memory_report(classes: int, window: int, precision: int = PRECISION_DOUBLE,
                         local: int = -1) -> dict:
    """Byte accounting of `classes` table sets (kernel_memory_report, rljsde.cpp:322-335)."""
    out = (C.c_uint64 * 4)()
    _check(lib.tqsb_kernel_memory_report(classes, window, precision, local, out))
    return dict(b_bytes=out[0], c_bytes=out[1], d_bytes=out[2], total_bytes=out[3])


def device_count() -> int:
    return lib.tqsb_device_count()


def probe_peaks(device: int = 0) -> dict:
    """Measured FP32 (FFMA2) TFLOP/s and shared-memory TB/s of one device."""
    f, s = C.c_double(), C.c_double()
    _check(lib.tqsb_probe_peaks(device, C.byref(f), C.byref(s)))
    return dict(fp32_tflops=f.value, smem_tbps=s.value)


class Plan:
    """Device-resident table store bound to one pattern + config (KernelCache analogue)."""

    def __init__(self, pattern: QuadrantPattern, config: ReconstructionConfig,
                 devices: list[int] | None = None):
        self.pattern = pattern
        self.config = dataclasses.replace(config)
        c = self.config._c()
        h = C.c_void_p()
        devs = devices if devices is not None else [0]
        arr = (C.c_int * len(devs))(*devs)
        opq = np.ascontiguousarray(pattern.opaque, np.uint8)
        _check(lib.tqsb_plan_create(opq.ctypes.data_as(_u8p), pattern.period, C.byref(c), arr,
                                    len(devs), C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.tqsb_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def warm(self, frame_rows: int, frame_cols: int) -> float:
        s = C.c_double()
        _check(lib.tqsb_plan_warm(self._h, frame_rows, frame_cols, C.byref(s)))
        return s.value

    def stats(self) -> dict:
        n, b = C.c_longlong(), C.c_longlong()
        _check(lib.tqsb_plan_stats(self._h, C.byref(n), C.byref(b)))
        return dict(classes=n.value, device_bytes=b.value)

    def _call(self, config):
        """The per-call configuration (None = the plan's own): like the reference's
        shared KernelCache, the plan pins only the window and the tables."""
        return None if config is None else C.byref(config._c())

    def reconstruct(self, frame: np.ndarray, reference: np.ndarray | None = None,
                    out: np.ndarray | None = None,
                    config: ReconstructionConfig | None = None) -> ReconstructionReport:
        frame = np.ascontiguousarray(frame, np.float64)
        if frame.ndim != 2:
            raise ValueError("frame must be 2-D")
        rows, cols = frame.shape
        out = _out_array(out, (2 * rows, 2 * cols))
        refp = None
        if reference is not None:
            reference = np.ascontiguousarray(reference, np.float64)
            if reference.shape != (2 * rows, 2 * cols):
                raise ValueError("reference dimensions do not match the reconstruction")
            refp = _d(reference)
        r = _Report()
        _check(lib.tqsb_reconstruct_with(self._h, self._call(config), _d(frame), rows, cols,
                                         _d(out), refp, C.byref(r)))
        return _report(out, r)

    def reconstruct_batch(self, frames: list, outs: list | None = None,
                          config: ReconstructionConfig | None = None) -> ReconstructionReport:
        """Frames of one shape through the pipelined multi-frame path (video stream)."""
        frames = [np.ascontiguousarray(f, np.float64) for f in frames]
        if not frames:
            raise ValueError("empty batch")
        rows, cols = frames[0].shape
        if any(f.shape != (rows, cols) for f in frames):
            raise ValueError("frames of a batch must share one shape")
        if outs is None:
            outs = [np.empty((2 * rows, 2 * cols)) for _ in frames]
        if len(outs) != len(frames):
            raise ValueError("outs must hold one output per frame")
        outs = [_out_array(o, (2 * rows, 2 * cols), "outs[i]") for o in outs]
        fp = (_dp * len(frames))(*[_d(f) for f in frames])
        op = (_dp * len(outs))(*[_d(o) for o in outs])
        r = _Report()
        _check(lib.tqsb_reconstruct_batch_with(self._h, self._call(config), fp, len(frames), rows,
                                               cols, op, C.byref(r)))
        return _report(outs, r)

    def reconstruct_band(self, frame: np.ndarray, br0: int, br1: int,
                         out: np.ndarray | None = None,
                         config: ReconstructionConfig | None = None) -> ReconstructionReport:
        frame = np.ascontiguousarray(frame, np.float64)
        rows, cols = frame.shape
        B = (config or self.config).block
        r1 = min(br1 * B, 2 * rows)
        out = _out_array(out, (max(0, r1 - br0 * B), 2 * cols))
        r = _Report()
        _check(lib.tqsb_reconstruct_band_with(self._h, self._call(config), _d(frame), rows, cols,
                                              br0, br1, _d(out), C.byref(r)))
        return _report(out, r)

    def reconstruct_device(self, d_frame_ptr: int, rows: int, cols: int, d_out_ptr: int,
                           stream: int = 0, band: tuple[int, int] | None = None) -> _Report:
        """Device-resident form (pointers from e.g. torch tensors); asynchronous."""
        r = _Report()
        if band is None:
            _check(lib.tqsb_reconstruct_device(self._h, C.c_void_p(d_frame_ptr), rows, cols,
                                               C.c_void_p(d_out_ptr), C.c_void_p(stream),
                                               C.byref(r)))
        else:
            _check(lib.tqsb_reconstruct_band_device(self._h, C.c_void_p(d_frame_ptr), rows, cols,
                                                    band[0], band[1], C.c_void_p(d_out_ptr),
                                                    C.c_void_p(stream), C.byref(r)))
        return r

    def export_tables(self, origin_row: int, origin_col: int) -> dict:
        L = C.c_int()
        _check(lib.tqsb_plan_export_tables(self._h, origin_row, origin_col, C.byref(L), None, None,
                                           None, None, None))
        L = L.value
        W = self.config.window
        K = W * W
        bre, bim = np.zeros(K * L), np.zeros(K * L)
        cre, cim = np.zeros(K * K), np.zeros(K * K)
        d = np.zeros(K)
        L2 = C.c_int()
        _check(lib.tqsb_plan_export_tables(self._h, origin_row, origin_col, C.byref(L2), _d(bre),
                                           _d(bim), _d(cre), _d(cim), _d(d)))
        return dict(L=L, b=(bre + 1j * bim).reshape(K, L), c=(cre + 1j * cim).reshape(K, K), d=d)

    def simulate_device(self, d_image_ptr: int, rows: int, cols: int, d_frame_ptr: int,
                        stream: int = 0) -> None:
        """Sensor readout of a device image into a device frame (grid.cpp:46-66)."""
        _check(lib.tqsb_plan_simulate_device(self._h, C.c_void_p(d_image_ptr), rows, cols,
                                             C.c_void_p(d_frame_ptr), C.c_void_p(stream)))

    def save_tables(self, path) -> int:
        """TQSK file of every resident class (save_kernel_cache, rljsde.cpp:398-432)."""
        n = C.c_int()
        _check(lib.tqsb_plan_save_tables(self._h, os.fsencode(path), C.byref(n)))
        return n.value

    def load_tables(self, path) -> int:
        """Make a TQSK file's classes resident (load_kernel_cache, rljsde.cpp:434-475)."""
        n = C.c_int()
        _check(lib.tqsb_plan_load_tables(self._h, os.fsencode(path), C.byref(n)))
        return n.value

    def block_trace(self, origin_row: int, origin_col: int, y_local: np.ndarray):
        it = max(1, self.config.max_iterations)
        W = self.config.window
        picks = np.zeros(it, np.int32)
        gd = np.zeros(2 * it)
        win = np.zeros(W * W)
        n = C.c_int()
        y = np.ascontiguousarray(y_local, np.float64)
        _check(lib.tqsb_plan_block_trace(self._h, origin_row, origin_col, _d(y),
                                         picks.ctypes.data_as(_ip), _d(gd), _d(win), C.byref(n)))
        n = n.value
        return picks[:n], (gd[0::2] + 1j * gd[1::2])[:n], win.reshape(W, W)


def reconstruct(frame: np.ndarray, pattern: QuadrantPattern, config: ReconstructionConfig,
                cache: Plan | None = None, reference: np.ndarray | None = None,
                devices: list[int] | None = None) -> ReconstructionReport:
    """Drop-in for tqs::reconstruct (pipeline.hpp:45-47); `cache` is a Plan."""
    validate_config(config, pattern.period)
    frame = np.ascontiguousarray(frame, np.float64)
    if frame.ndim != 2 or frame.size == 0:
        raise ValueError("empty measurement frame")
    # the reference shares its cache with RL-JSDE only (pipeline.cpp:111-112): an
    # L-JSDE call leaves the cache untouched and reports no cache counters
    if cache is not None and config.algorithm == ALGO_RLJSDE:
        return cache.reconstruct(frame, reference, config=config)
    with Plan(pattern, config, devices) as plan:
        return plan.reconstruct(frame, reference)


def pad_to_block_multiple(image: np.ndarray, block: int):
    """pipeline.cpp:187-209: edge replication to even block multiples."""
    if block < 1:
        raise ValueError("block size must be positive")
    if image.size == 0:
        raise ValueError("empty image")
    step = math.lcm(block, 2)
    rows = -(-image.shape[0] // step) * step
    cols = -(-image.shape[1] // step) * step
    ri = np.minimum(np.arange(rows), image.shape[0] - 1)
    ci = np.minimum(np.arange(cols), image.shape[1] - 1)
    return image[np.ix_(ri, ci)], image.shape[0], image.shape[1]


def reconstruct_image(image: np.ndarray, pattern: QuadrantPattern, config: ReconstructionConfig,
                      cache: Plan | None = None) -> ReconstructionReport:
    """pipeline.cpp:248-256: pad, simulate, reconstruct, crop, PSNR vs the input."""
    padded, r0, c0 = pad_to_block_multiple(np.asarray(image, np.float64), config.block)
    frame = simulate_measurement(padded, pattern)
    rep = reconstruct(frame, pattern, config, cache)
    rep.output = np.ascontiguousarray(rep.output[:r0, :c0])
    rep.psnr_db = psnr(image, rep.output)
    return rep


from .io import (read_frame, read_image_any, read_pattern, read_pgm, read_raw_image,  # noqa: E402
                 write_frame, write_pattern, write_pgm, write_raw_image)
