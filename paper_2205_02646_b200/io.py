"""File formats of the reference (include/tqs/io.hpp:1-35): binary PGM, TQSP
pattern files and TQSM float64 containers, through the C ABI (csrc/io.cpp).
Failures raise FormatError ("<path>: <what>", std::runtime_error in the
reference) or ValueError (std::invalid_argument)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import QuadrantPattern, _check, _d, _u8p, lib

_ANY, _PGM, _TQSM = 0, 1, 2


def _read(path, kind: int) -> np.ndarray:
    p = os.fsencode(path)
    r, c = C.c_int(), C.c_int()
    _check(lib.tqsb_io_read(p, kind, C.byref(r), C.byref(c), None))
    out = np.empty((r.value, c.value))
    _check(lib.tqsb_io_read(p, kind, C.byref(r), C.byref(c), _d(out)))
    return out


def read_pgm(path) -> np.ndarray:
    """P5, maxval <= 65535 (16-bit samples big-endian), values = sample / maxval."""
    return _read(path, _PGM)


def write_pgm(path, image: np.ndarray, bit_depth: int = 8) -> None:
    img = np.ascontiguousarray(image, np.float64)
    rows, cols = (img.shape + (0, 0))[:2] if img.ndim == 2 else (0, 0)
    _check(lib.tqsb_io_write_pgm(os.fsencode(path), _d(img) if img.size else None, rows, cols,
                                 bit_depth))


def read_frame(path) -> np.ndarray:
    return _read(path, _TQSM)


def write_frame(path, frame: np.ndarray) -> None:
    f = np.ascontiguousarray(frame, np.float64)
    _check(lib.tqsb_io_write_tqsm(os.fsencode(path), _d(f), f.shape[0], f.shape[1]))


read_raw_image = read_frame
write_raw_image = write_frame


def read_image_any(path) -> np.ndarray:
    """TQSM raw dump when the file starts with "TQSM", else PGM (io.cpp:261-269)."""
    return _read(path, _ANY)


def read_pattern(path) -> QuadrantPattern:
    p = os.fsencode(path)
    period, seed = C.c_int(), C.c_uint64()
    rng = C.create_string_buffer(256)
    _check(lib.tqsb_io_read_pattern(p, C.byref(period), C.byref(seed), rng, 256, None))
    opaque = np.zeros((period.value // 2) ** 2, np.uint8)
    _check(lib.tqsb_io_read_pattern(p, C.byref(period), C.byref(seed), rng, 256,
                                    opaque.ctypes.data_as(_u8p)))
    return QuadrantPattern(period.value, opaque, seed.value, rng.value.decode())


def write_pattern(path, pattern: QuadrantPattern) -> None:
    opq = np.ascontiguousarray(pattern.opaque, np.uint8)
    _check(lib.tqsb_io_write_pattern(os.fsencode(path), pattern.period, pattern.seed,
                                     pattern.rng.encode(), opq.ctypes.data_as(_u8p)))
