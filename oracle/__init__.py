"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the CPU checkers of the RL-JSDE path:

* ``Oracle`` -- the plain-C restatement in ``oracle/tqs_oracle.c`` (liboracle.so);
* ``Reference`` -- the UNMODIFIED reference library compiled from
  /root/reference/proj into ``oracle/_ref/`` (see build_ref.sh, ref_shim.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package; the product path
(``paper_2205_02646_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)


def _d(a):
    return a.ctypes.data_as(_dp)


def build(quiet: bool = True) -> None:
    """Compile liboracle.so and (when /root/reference exists) oracle/_ref."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class Oracle:
    def __init__(self):
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.or_generate_pattern.argtypes = [C.c_uint64, C.c_int, C.c_int, _u8p]
        L.or_simulate.argtypes = [_dp, C.c_int, C.c_int, _u8p, C.c_int, _dp]
        L.or_synthetic_image.argtypes = [C.c_int, C.c_int, C.c_uint64, _dp]
        L.or_frequency_weights.argtypes = [C.c_int, C.c_double, _dp]
        L.or_unit_table.argtypes = [C.c_int, _dp, _dp]
        L.or_local_matrix.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip, _ip]
        L.or_tables.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                _dp, _dp, _dp, _dp, _dp, _dp]
        L.or_gather.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.or_block.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int,
                               C.c_double, _ip, _dp, _dp]
        L.or_census.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.POINTER(C.c_longlong), _ip]
        L.or_reconstruct.argtypes = [_dp, C.c_int, C.c_int, _u8p, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, _dp]
        L.or_reconstruct.restype = C.c_longlong
        L.or_psnr.argtypes = [_dp, _dp, C.c_longlong]
        L.or_psnr.restype = C.c_double
        self.lib = L

    def generate_pattern(self, seed, period, block=4):
        out = np.zeros((period // 2) ** 2, np.uint8)
        if self.lib.or_generate_pattern(seed, period, block, out.ctypes.data_as(_u8p)):
            raise ValueError("invalid pattern parameters")
        return out

    def synthetic_image(self, rows, cols, seed):
        out = np.zeros((rows, cols))
        self.lib.or_synthetic_image(rows, cols, seed, _d(out))
        return out

    def simulate(self, image, opaque, period):
        image = np.ascontiguousarray(image, np.float64)
        out = np.zeros((image.shape[0] // 2, image.shape[1] // 2))
        if self.lib.or_simulate(_d(image), image.shape[0], image.shape[1],
                                opaque.ctypes.data_as(_u8p), period, _d(out)):
            raise ValueError("image dimensions must be even")
        return out

    def frequency_weights(self, window, exponent=2.0):
        q = np.zeros(window * window)
        self.lib.or_frequency_weights(window, exponent, _d(q))
        return q

    def local_count(self, opaque, period, orow, ocol, window):
        return self.lib.or_local_matrix(opaque.ctypes.data_as(_u8p), period, orow, ocol, window,
                                        None, None, None)

    def tables(self, opaque, period, orow, ocol, window, decay=0.8):
        L = self.local_count(opaque, period, orow, ocol, window)
        K = window * window
        bre, bim = np.zeros(K * L), np.zeros(K * L)
        cre, cim = np.zeros(K * K), np.zeros(K * K)
        d, w = np.zeros(K), np.zeros(L)
        self.lib.or_tables(opaque.ctypes.data_as(_u8p), period, orow, ocol, window, decay,
                           _d(bre), _d(bim), _d(cre), _d(cim), _d(d), _d(w))
        return dict(L=L, b=(bre + 1j * bim).reshape(K, L), c=(cre + 1j * cim).reshape(K, K),
                    d=d, w=w, _planes=(bre, bim, cre, cim, d))

    def gather(self, frame, orow, ocol, window):
        frame = np.ascontiguousarray(frame, np.float64)
        y = np.zeros(window * window)
        n = self.lib.or_gather(_d(frame), frame.shape[1], orow, ocol, window, _d(y))
        return y[:n]

    def block(self, tabs, q, y, window, iterations=200, step=0.5):
        K = window * window
        bre, bim, cre, cim, d = tabs["_planes"]
        picks = np.full(iterations, -1, np.int32)
        gd = np.zeros(2 * iterations)
        win = np.zeros(K)
        y = np.ascontiguousarray(y, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        n = self.lib.or_block(window, tabs["L"], _d(bre), _d(bim), _d(cre), _d(cim), _d(d),
                              _d(q), _d(y), iterations, step, picks.ctypes.data_as(_ip), _d(gd),
                              _d(win))
        return picks[:n], (gd[0::2] + 1j * gd[1::2])[:n], win.reshape(window, window)

    def census(self, frame_rows, frame_cols, window=32, block=4, period=32, tasks=False):
        out = (C.c_longlong * 3)()
        if self.lib.or_census(frame_rows, frame_cols, window, block, period, out, None):
            raise ValueError("image is smaller than the model window")
        res = dict(blocks=out[0], classes_total=out[1], classes_interior=out[2])
        if tasks:
            t = np.zeros((out[0], 5), np.int32)
            self.lib.or_census(frame_rows, frame_cols, window, block, period, out,
                               t.ctypes.data_as(_ip))
            res["tasks"] = t
        return res

    def reconstruct(self, frame, opaque, period, window=32, block=4, iterations=200, step=0.5,
                    decay=0.8, exponent=2.0, clip=True):
        frame = np.ascontiguousarray(frame, np.float64)
        out = np.zeros((2 * frame.shape[0], 2 * frame.shape[1]))
        n = self.lib.or_reconstruct(_d(frame), frame.shape[0], frame.shape[1],
                                    opaque.ctypes.data_as(_u8p), period, window, block,
                                    iterations, step, decay, exponent, int(clip), _d(out))
        if n < 0:
            raise ValueError("invalid configuration")
        return out

    def psnr(self, ref, est):
        ref = np.ascontiguousarray(ref, np.float64)
        est = np.ascontiguousarray(est, np.float64)
        return self.lib.or_psnr(_d(ref), _d(est), ref.size)


class RefReport(C.Structure):
    _fields_ = [("seconds", C.c_double), ("warm_seconds", C.c_double),
                ("blocks", C.c_longlong), ("classes_total", C.c_longlong),
                ("classes_interior", C.c_longlong), ("classes_created", C.c_longlong),
                ("cache_hits", C.c_longlong), ("cache_misses", C.c_longlong),
                ("psnr_db", C.c_double), ("has_psnr", C.c_int), ("threads_used", C.c_int)]


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " avx512f" in f.read()
    except OSError:
        return False


class Reference:
    """The unmodified reference library (oracle/_ref), via ref_shim.cpp."""

    def __init__(self, isa: str | None = None):
        if isa is None:
            isa = "v4" if _cpu_has_avx512() else "v3"
        path = os.path.join(HERE, "_ref", f"libtqs_ref_{isa}.so")
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build oracle/_ref where /root/reference exists")
        self.isa = isa
        self.path = path
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate_pattern.argtypes = [C.c_uint64, C.c_int, C.c_int, _u8p]
        L.ref_synthetic_image.argtypes = [C.c_int, C.c_int, C.c_uint64, _dp]
        L.ref_simulate.argtypes = [_dp, C.c_int, C.c_int, _u8p, C.c_int, _dp]
        L.ref_frequency_weights.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.ref_cache_new.restype = C.c_void_p
        L.ref_cache_free.argtypes = [C.c_void_p]
        L.ref_reconstruct.argtypes = [_dp, C.c_int, C.c_int, _u8p, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                      C.c_int, C.c_int, C.c_void_p, _dp, _dp,
                                      C.POINTER(RefReport)]
        L.ref_precompute.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                     C.c_double, C.c_int, _ip, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_block_trace.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_int,
                                      C.c_double, C.c_double, C.c_double, C.c_int, _ip, _dp, _dp]
        L.ref_io_write_pgm.argtypes = [C.c_char_p, _dp, C.c_int, C.c_int, C.c_int]
        L.ref_io_read.argtypes = [C.c_char_p, C.c_int, _ip, _ip, _dp]
        L.ref_io_write_tqsm.argtypes = [C.c_char_p, _dp, C.c_int, C.c_int]
        L.ref_io_write_pattern.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_char_p, _u8p]
        L.ref_io_read_pattern.argtypes = [C.c_char_p, _ip, C.POINTER(C.c_uint64), C.c_char_p,
                                          C.c_size_t, _u8p]
        L.ref_pattern_digest.argtypes = [_u8p, C.c_int]
        L.ref_pattern_digest.restype = C.c_uint64
        L.ref_save_cache.argtypes = [C.c_void_p, C.c_char_p, _u8p, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_double]
        L.ref_load_cache.argtypes = L.ref_save_cache.argtypes
        L.ref_memory_report.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_uint64)]
        L.ref_reconstruct_algo.argtypes = [_dp, C.c_int, C.c_int, _u8p, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _dp,
                                           _dp]
        L.ref_ljsde_trace.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_int,
                                      C.c_double, C.c_double, _ip, _dp, _dp]
        self.lib = L

    # ---- file formats (tqs::read_* / write_*, io.cpp)
    def write_pgm(self, path, img, bits=8):
        img = np.ascontiguousarray(img, np.float64)
        rows, cols = img.shape if img.ndim == 2 else (0, 0)
        self._check(self.lib.ref_io_write_pgm(os.fsencode(path), _d(img) if img.size else None,
                                              rows, cols, bits))

    def read(self, path, kind=0):
        r, c = C.c_int(), C.c_int()
        self._check(self.lib.ref_io_read(os.fsencode(path), kind, C.byref(r), C.byref(c), None))
        out = np.zeros((r.value, c.value))
        self._check(self.lib.ref_io_read(os.fsencode(path), kind, C.byref(r), C.byref(c),
                                         _d(out)))
        return out

    def write_tqsm(self, path, v):
        v = np.ascontiguousarray(v, np.float64)
        self._check(self.lib.ref_io_write_tqsm(os.fsencode(path), _d(v), v.shape[0], v.shape[1]))

    def write_pattern(self, path, period, seed, rng, opaque):
        opaque = np.ascontiguousarray(opaque, np.uint8)
        self._check(self.lib.ref_io_write_pattern(os.fsencode(path), period, seed, rng.encode(),
                                                  opaque.ctypes.data_as(_u8p)))

    def read_pattern(self, path):
        per, seed = C.c_int(), C.c_uint64()
        rng = C.create_string_buffer(256)
        self._check(self.lib.ref_io_read_pattern(os.fsencode(path), C.byref(per), C.byref(seed),
                                                 rng, 256, None))
        opq = np.zeros((per.value // 2) ** 2, np.uint8)
        self._check(self.lib.ref_io_read_pattern(os.fsencode(path), C.byref(per), C.byref(seed),
                                                 rng, 256, opq.ctypes.data_as(_u8p)))
        return per.value, seed.value, rng.value.decode(), opq

    # ---- TQSK persistence / accounting
    def pattern_digest(self, opaque, period):
        return self.lib.ref_pattern_digest(np.ascontiguousarray(opaque, np.uint8).ctypes.data_as(_u8p),
                                           period)

    def save_cache(self, cache, path, opaque, period, window, double=True, decay=0.8,
                   exponent=2.0):
        self._check(self.lib.ref_save_cache(cache, os.fsencode(path),
                                            np.ascontiguousarray(opaque, np.uint8).ctypes.data_as(_u8p),
                                            period, window, int(double), decay, exponent))

    def load_cache(self, cache, path, opaque, period, window, double=True, decay=0.8,
                   exponent=2.0):
        return self._check(self.lib.ref_load_cache(
            cache, os.fsencode(path), np.ascontiguousarray(opaque, np.uint8).ctypes.data_as(_u8p),
            period, window, int(double), decay, exponent))

    def memory_report(self, classes, window, double, local=-1):
        out = (C.c_uint64 * 4)()
        self._check(self.lib.ref_memory_report(classes, window, int(double), local, out))
        return dict(b_bytes=out[0], c_bytes=out[1], d_bytes=out[2], total_bytes=out[3])

    # ---- L-JSDE
    def reconstruct_algo(self, frame, opaque, period, algo, window=32, block=4, iterations=200,
                         step=0.5, clip=False, threads=0):
        frame = np.ascontiguousarray(frame, np.float64)
        out = np.zeros((2 * frame.shape[0], 2 * frame.shape[1]))
        sec = C.c_double()
        self._check(self.lib.ref_reconstruct_algo(
            _d(frame), frame.shape[0], frame.shape[1],
            np.ascontiguousarray(opaque, np.uint8).ctypes.data_as(_u8p), period, window, block,
            iterations, step, 0 if algo == "ljsde" else 1, int(clip), threads, _d(out),
            C.byref(sec)))
        return out, sec.value

    def ljsde_trace(self, opaque, period, orow, ocol, window, y, iterations=200, step=0.5,
                    early_stop_scale=0.0):
        n = max(iterations, 1)
        picks = np.full(n, -1, np.int32)
        gd = np.zeros(2 * n)
        win = np.zeros(window * window)
        y = np.ascontiguousarray(y, np.float64)
        k = self._check(self.lib.ref_ljsde_trace(
            np.ascontiguousarray(opaque, np.uint8).ctypes.data_as(_u8p), period, orow, ocol,
            window, _d(y), iterations, step, early_stop_scale, picks.ctypes.data_as(_ip), _d(gd),
            _d(win)))
        return picks[:k], (gd[0::2] + 1j * gd[1::2])[:k], win.reshape(window, window)

    def _check(self, rc):
        if rc < 0:
            msg = self.lib.ref_last_error().decode()
            raise ValueError(msg) if rc == -1 else RuntimeError(msg)
        return rc

    def hardware_threads(self):
        return self.lib.ref_hardware_threads()

    def generate_pattern(self, seed, period, block=4):
        out = np.zeros((period // 2) ** 2, np.uint8)
        self._check(self.lib.ref_generate_pattern(seed, period, block, out.ctypes.data_as(_u8p)))
        return out

    def synthetic_image(self, rows, cols, seed):
        out = np.zeros((rows, cols))
        self._check(self.lib.ref_synthetic_image(rows, cols, seed, _d(out)))
        return out

    def simulate(self, image, opaque, period):
        image = np.ascontiguousarray(image, np.float64)
        out = np.zeros((image.shape[0] // 2, image.shape[1] // 2))
        self._check(self.lib.ref_simulate(_d(image), image.shape[0], image.shape[1],
                                          opaque.ctypes.data_as(_u8p), period, _d(out)))
        return out

    def frequency_weights(self, window, decay=0.8, exponent=2.0):
        q = np.zeros(window * window)
        self._check(self.lib.ref_frequency_weights(window, decay, exponent, _d(q)))
        return q

    def new_cache(self):
        return C.c_void_p(self.lib.ref_cache_new())

    def free_cache(self, c):
        self.lib.ref_cache_free(c)

    def reconstruct(self, frame, opaque, period, window=32, block=4, iterations=200, step=0.5,
                    decay=0.8, exponent=2.0, double=True, clip=True, threads=1, cache=None,
                    reference=None):
        frame = np.ascontiguousarray(frame, np.float64)
        out = np.zeros((2 * frame.shape[0], 2 * frame.shape[1]))
        rep = RefReport()
        refp = None
        if reference is not None:
            reference = np.ascontiguousarray(reference, np.float64)
            refp = _d(reference)
        self._check(self.lib.ref_reconstruct(
            _d(frame), frame.shape[0], frame.shape[1], opaque.ctypes.data_as(_u8p), period,
            window, block, iterations, step, decay, exponent, int(double), int(clip), threads,
            cache, refp, _d(out), C.byref(rep)))
        return out, rep

    def precompute(self, opaque, period, orow, ocol, window, decay=0.8, exponent=2.0,
                   double=True):
        L = C.c_int()
        self._check(self.lib.ref_precompute(opaque.ctypes.data_as(_u8p), period, orow, ocol,
                                            window, decay, exponent, int(double), C.byref(L),
                                            None, None, None, None, None, None))
        L = L.value
        K = window * window
        bre, bim = np.zeros(K * L), np.zeros(K * L)
        cre, cim = np.zeros(K * K), np.zeros(K * K)
        d, w = np.zeros(K), np.zeros(L)
        Lc = C.c_int()
        self._check(self.lib.ref_precompute(opaque.ctypes.data_as(_u8p), period, orow, ocol,
                                            window, decay, exponent, int(double), C.byref(Lc),
                                            _d(bre), _d(bim), _d(cre), _d(cim), _d(d), _d(w)))
        return dict(L=L, b=(bre + 1j * bim).reshape(K, L), c=(cre + 1j * cim).reshape(K, K),
                    d=d, w=w, _planes=(bre, bim, cre, cim, d))

    def block_trace(self, opaque, period, orow, ocol, window, y, iterations=200, step=0.5,
                    decay=0.8, exponent=2.0, double=True):
        picks = np.full(max(iterations, 1), -1, np.int32)
        gd = np.zeros(2 * max(iterations, 1))
        win = np.zeros(window * window)
        y = np.ascontiguousarray(y, np.float64)
        n = self._check(self.lib.ref_block_trace(
            opaque.ctypes.data_as(_u8p), period, orow, ocol, window, _d(y), iterations, step,
            decay, exponent, int(double), picks.ctypes.data_as(_ip), _d(gd), _d(win)))
        return picks[:n], (gd[0::2] + 1j * gd[1::2])[:n], win.reshape(window, window)
