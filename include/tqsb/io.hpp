// io.hpp -- header-only C++ face of the file formats (reference include/tqs/io.hpp:1-35):
// binary PGM (P5, 8/16-bit), TQSP pattern files and TQSM float64 containers, with the
// reference's function names and exception types (std::runtime_error "<path>: <what>",
// std::invalid_argument for write validation). Implemented in csrc/io.cpp behind tqsb.h.
#pragma once

#include <string>

#include "reconstruct.hpp"

namespace tqsb {

namespace detail {
inline std::vector<double> io_read(const std::string& path, int kind, int* rows, int* cols) {
    check(tqsb_io_read(path.c_str(), kind, rows, cols, nullptr));
    std::vector<double> v(size_t(*rows) * size_t(*cols));
    check(tqsb_io_read(path.c_str(), kind, rows, cols, v.data()));
    return v;
}
}  // namespace detail

inline Image read_pgm(const std::string& path) {
    Image img;
    img.values = detail::io_read(path, TQSB_IO_PGM, &img.rows, &img.cols);
    return img;
}

inline void write_pgm(const std::string& path, const Image& image, int bitDepth = 8) {
    detail::check(tqsb_io_write_pgm(path.c_str(), image.values.data(), image.rows, image.cols,
                                    bitDepth));
}

inline QuadrantPattern read_pattern(const std::string& path) {
    QuadrantPattern p;
    char rng[256];
    detail::check(tqsb_io_read_pattern(path.c_str(), &p.period, &p.seed, rng, sizeof rng, nullptr));
    p.opaque.resize(size_t(p.period / 2) * size_t(p.period / 2));
    detail::check(tqsb_io_read_pattern(path.c_str(), &p.period, &p.seed, rng, sizeof rng,
                                       p.opaque.data()));
    p.rng = rng;
    return p;
}

inline void write_pattern(const std::string& path, const QuadrantPattern& pattern) {
    detail::check(tqsb_io_write_pattern(path.c_str(), pattern.period, pattern.seed,
                                        pattern.rng.c_str(), pattern.opaque.data()));
}

inline MeasurementFrame read_frame(const std::string& path) {
    MeasurementFrame f;
    f.values = detail::io_read(path, TQSB_IO_TQSM, &f.rows, &f.cols);
    return f;
}

inline void write_frame(const std::string& path, const MeasurementFrame& frame) {
    detail::check(tqsb_io_write_tqsm(path.c_str(), frame.values.data(), frame.rows, frame.cols));
}

inline Image read_raw_image(const std::string& path) {
    Image img;
    img.values = detail::io_read(path, TQSB_IO_TQSM, &img.rows, &img.cols);
    return img;
}

inline void write_raw_image(const std::string& path, const Image& image) {
    detail::check(tqsb_io_write_tqsm(path.c_str(), image.values.data(), image.rows, image.cols));
}

inline Image read_image_any(const std::string& path) {
    Image img;
    img.values = detail::io_read(path, TQSB_IO_ANY, &img.rows, &img.cols);
    return img;
}

}  // namespace tqsb
