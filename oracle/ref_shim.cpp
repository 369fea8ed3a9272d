// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never part of the product path).
//
// A thin extern "C" face over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src/*.cpp by oracle/build_ref.sh into oracle/_ref/.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load it, as the checker and as the CPU baseline.
//
// Every entry point forwards to the reference's own public API:
//   ref_generate_pattern  -> tqs::generate_pattern          (grid.cpp:8-26)
//   ref_synthetic_image   -> tqs::testing::synthetic_image  (tests/support/synthetic.cpp:9-80)
//   ref_simulate          -> tqs::simulate_measurement      (grid.cpp:46-66)
//   ref_reconstruct       -> tqs::reconstruct               (pipeline.cpp:62-185)
//   ref_precompute        -> tqs::extract_local_matrix + spatial_weights +
//                            precompute_kernels             (grid.cpp:75-102, basis.cpp:82-88,
//                                                            rljsde.cpp:186-201)
//   ref_block_trace       -> tqs::rljsde_block with an IterationHook (rljsde.cpp:258-271)
//   ref_frequency_weights -> tqs::frequency_weights         (basis.cpp:99-106)
//   ref_io_*              -> tqs::read_pgm / write_pgm / read_pattern / write_pattern /
//                            read_frame / write_raw_image / read_image_any (io.cpp)
//   ref_pattern_digest, ref_save_cache, ref_load_cache
//                         -> tqs::pattern_digest / save_kernel_cache / load_kernel_cache
//                                                           (rljsde.cpp:337-475)
//   ref_memory_report     -> tqs::kernel_memory_report      (rljsde.cpp:322-335)
//   ref_reconstruct_algo  -> tqs::reconstruct with Algorithm::Ljsde or Rljsde
//   ref_ljsde_trace       -> tqs::ljsde_block with an IterationHook (ljsde.cpp:131-185)
// Exceptions never cross the ABI: they become a negative return code and the
// message is kept for ref_last_error().

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "synthetic.hpp"
#include "tqs/basis.hpp"
#include "tqs/grid.hpp"
#include "tqs/io.hpp"
#include "tqs/ljsde.hpp"
#include "tqs/pipeline.hpp"
#include "tqs/rljsde.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

tqs::QuadrantPattern make_pattern(const uint8_t* opaque, int period) {
    tqs::QuadrantPattern p;
    p.period = period;
    p.rng = "mt19937_64";
    const int pc = period / 2;
    p.opaque.assign(opaque, opaque + static_cast<size_t>(pc) * pc);
    return p;
}

} // namespace

extern "C" {

struct ref_report {
    double seconds;
    double warm_seconds;
    long long blocks;
    long long classes_total;
    long long classes_interior;
    long long classes_created;
    long long cache_hits;
    long long cache_misses;
    double psnr_db;
    int has_psnr;
    int threads_used;
};

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_hardware_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }

int ref_generate_pattern(uint64_t seed, int period, int block, uint8_t* opaque_out) {
    try {
        const tqs::QuadrantPattern p = tqs::generate_pattern(seed, period, block);
        std::memcpy(opaque_out, p.opaque.data(), p.opaque.size());
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

int ref_synthetic_image(int rows, int cols, uint64_t seed, double* out) {
    try {
        const tqs::Image img = tqs::testing::synthetic_image(rows, cols, seed);
        std::memcpy(out, img.values.data(), img.values.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

int ref_simulate(const double* image, int rows, int cols, const uint8_t* opaque, int period,
                 double* frame_out) {
    try {
        tqs::Image img(rows, cols);
        std::memcpy(img.values.data(), image, img.values.size() * sizeof(double));
        const tqs::MeasurementFrame f = tqs::simulate_measurement(img, make_pattern(opaque, period));
        std::memcpy(frame_out, f.values.data(), f.values.size() * sizeof(double));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

int ref_frequency_weights(int window, double spatial_decay, double frequency_exponent,
                          double* q_out) {
    try {
        tqs::WeightingConfig wc;
        wc.spatialDecay = spatial_decay;
        wc.frequencyExponent = frequency_exponent;
        const std::vector<double> q = tqs::frequency_weights(window, wc);
        std::memcpy(q_out, q.data(), q.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// cache_handle: opaque KernelCache* shared across calls (like the reference's
// external cache, pipeline.hpp:45-47); create with ref_cache_new.
void* ref_cache_new(void) { return new tqs::KernelCache(); }
void ref_cache_free(void* c) { delete static_cast<tqs::KernelCache*>(c); }

int ref_reconstruct(const double* frame, int frame_rows, int frame_cols, const uint8_t* opaque,
                    int period, int window, int block, int iterations, double step_width,
                    double spatial_decay, double frequency_exponent, int precision_double,
                    int clip, int threads, void* cache, const double* reference_or_null,
                    double* out, ref_report* rep) {
    try {
        tqs::MeasurementFrame f(frame_rows, frame_cols);
        std::memcpy(f.values.data(), frame, f.values.size() * sizeof(double));
        tqs::ReconstructionConfig cfg;
        cfg.window = window;
        cfg.block = block;
        cfg.solver.maxIterations = iterations;
        cfg.solver.stepWidth = step_width;
        cfg.weighting.spatialDecay = spatial_decay;
        cfg.weighting.frequencyExponent = frequency_exponent;
        cfg.precision = precision_double ? tqs::Precision::Double : tqs::Precision::Single;
        cfg.clipOutput = clip != 0;
        cfg.algorithm = tqs::Algorithm::Rljsde;
        cfg.threads = threads;
        tqs::Image ref;
        const tqs::Image* refp = nullptr;
        if (reference_or_null) {
            ref = tqs::Image(2 * frame_rows, 2 * frame_cols);
            std::memcpy(ref.values.data(), reference_or_null, ref.values.size() * sizeof(double));
            refp = &ref;
        }
        const tqs::ReconstructionReport r = tqs::reconstruct(
            f, make_pattern(opaque, period), cfg, static_cast<tqs::KernelCache*>(cache), refp);
        std::memcpy(out, r.output.values.data(), r.output.values.size() * sizeof(double));
        if (rep) {
            rep->seconds = r.seconds;
            rep->warm_seconds = r.warmSeconds;
            rep->blocks = r.blocksProcessed;
            rep->classes_total = static_cast<long long>(r.classesTotal);
            rep->classes_interior = static_cast<long long>(r.classesInterior);
            rep->classes_created = static_cast<long long>(r.classesCreated);
            rep->cache_hits = static_cast<long long>(r.cacheHits);
            rep->cache_misses = static_cast<long long>(r.cacheMisses);
            rep->has_psnr = r.psnrDb.has_value() ? 1 : 0;
            rep->psnr_db = r.psnrDb.value_or(0.0);
            rep->threads_used = threads == 0 ? static_cast<int>(std::thread::hardware_concurrency())
                                             : threads;
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::logic_error& e) {
        return fail(e, -4);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

// Tables for one window origin: local count, B (k-major [k*L+m]), C (column-major
// [uk*K+sk]) and D, as the reference stores them (rljsde.hpp:34-52), widened to
// double. Pass null outputs to query L only (returned through *local_out).
int ref_precompute(const uint8_t* opaque, int period, int origin_row, int origin_col, int window,
                   double spatial_decay, double frequency_exponent, int precision_double,
                   int* local_out, double* b_re, double* b_im, double* c_re, double* c_im,
                   double* d, double* weights_out) {
    try {
        const tqs::QuadrantPattern p = make_pattern(opaque, period);
        const tqs::LocalMeasurementMatrix m =
            tqs::extract_local_matrix(p, origin_row, origin_col, window);
        tqs::WeightingConfig wc;
        wc.spatialDecay = spatial_decay;
        wc.frequencyExponent = frequency_exponent;
        const std::vector<double> w = tqs::spatial_weights(m, wc);
        *local_out = m.localCount();
        if (!b_re)
            return 0;
        const tqs::KernelSet s = tqs::precompute_kernels(
            m, w, precision_double ? tqs::Precision::Double : tqs::Precision::Single);
        const size_t K = static_cast<size_t>(window) * window, L = s.local;
        auto put = [](double* dst, const auto& src) {
            for (size_t i = 0; i < src.size(); ++i) dst[i] = double(src[i]);
        };
        if (s.precision == tqs::Precision::Double) {
            put(b_re, s.p64.bRe); put(b_im, s.p64.bIm);
            put(c_re, s.p64.cRe); put(c_im, s.p64.cIm); put(d, s.p64.d);
        } else {
            put(b_re, s.p32.bRe); put(b_im, s.p32.bIm);
            put(c_re, s.p32.cRe); put(c_im, s.p32.cIm); put(d, s.p32.d);
        }
        (void)K; (void)L;
        if (weights_out)
            for (size_t i = 0; i < w.size(); ++i) weights_out[i] = w[i];
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

// One block solve through rljsde_block with a hook recording the greedy path:
// picks[i] = chosen flat index, gd[2i..2i+1] = scaled delta. Returns the number
// of completed iterations; window_out receives the synthesized W*W window.
int ref_block_trace(const uint8_t* opaque, int period, int origin_row, int origin_col, int window,
                    const double* y_local, int iterations, double step_width,
                    double spatial_decay, double frequency_exponent, int precision_double,
                    int* picks, double* gd, double* window_out) {
    try {
        const tqs::QuadrantPattern p = make_pattern(opaque, period);
        const tqs::LocalMeasurementMatrix m =
            tqs::extract_local_matrix(p, origin_row, origin_col, window);
        tqs::WeightingConfig wc;
        wc.spatialDecay = spatial_decay;
        wc.frequencyExponent = frequency_exponent;
        const std::vector<double> w = tqs::spatial_weights(m, wc);
        const tqs::KernelSet s = tqs::precompute_kernels(
            m, w, precision_double ? tqs::Precision::Double : tqs::Precision::Single);
        const std::vector<double> q = tqs::frequency_weights(window, wc);
        std::vector<double> y(y_local, y_local + m.localCount());
        tqs::SolverOptions opt;
        opt.maxIterations = iterations;
        opt.stepWidth = step_width;
        int n = 0;
        const std::vector<double> win = tqs::rljsde_block(
            y, s, q, opt, [&](int, int chosen, tqs::cplx g, std::span<const tqs::cplx>) {
                picks[n] = chosen;
                gd[2 * n] = g.real();
                gd[2 * n + 1] = g.imag();
                ++n;
            });
        std::memcpy(window_out, win.data(), win.size() * sizeof(double));
        return n;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

// ---------------------------------------------------------------- file formats
int ref_io_write_pgm(const char* path, const double* img, int rows, int cols, int bits) {
    try {
        tqs::Image im(rows, cols);
        if (rows > 0 && cols > 0) std::memcpy(im.values.data(), img, im.values.size() * sizeof(double));
        tqs::write_pgm(path, im, bits);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

// kind 0: read_image_any, 1: read_pgm, 2: read_frame (TQSM)
int ref_io_read(const char* path, int kind, int* rows, int* cols, double* out) {
    try {
        std::vector<double> v;
        if (kind == 2) {
            const tqs::MeasurementFrame f = tqs::read_frame(path);
            *rows = f.rows, *cols = f.cols, v = f.values;
        } else {
            const tqs::Image im = kind == 1 ? tqs::read_pgm(path) : tqs::read_image_any(path);
            *rows = im.rows, *cols = im.cols, v = im.values;
        }
        if (out) std::memcpy(out, v.data(), v.size() * sizeof(double));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

int ref_io_write_tqsm(const char* path, const double* v, int rows, int cols) {
    try {
        tqs::Image im(rows, cols);
        std::memcpy(im.values.data(), v, im.values.size() * sizeof(double));
        tqs::write_raw_image(path, im);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

int ref_io_write_pattern(const char* path, int period, uint64_t seed, const char* rng,
                         const uint8_t* opaque) {
    try {
        tqs::QuadrantPattern p = make_pattern(opaque, period);
        p.seed = seed;
        p.rng = rng;
        tqs::write_pattern(path, p);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

int ref_io_read_pattern(const char* path, int* period, uint64_t* seed, char* rng, size_t cap,
                        uint8_t* opaque) {
    try {
        const tqs::QuadrantPattern p = tqs::read_pattern(path);
        *period = p.period;
        *seed = p.seed;
        std::snprintf(rng, cap, "%s", p.rng.c_str());
        if (opaque) std::memcpy(opaque, p.opaque.data(), p.opaque.size());
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

// ---------------------------------------------------------------- TQSK persistence
uint64_t ref_pattern_digest(const uint8_t* opaque, int period) {
    return tqs::pattern_digest(make_pattern(opaque, period));
}

static tqs::KernelCacheHeader cache_header(const uint8_t* opaque, int period, int window,
                                           int precision_double, double decay, double exponent) {
    tqs::KernelCacheHeader h;
    h.window = window;
    h.period = period;
    h.precision = precision_double ? tqs::Precision::Double : tqs::Precision::Single;
    h.weighting.spatialDecay = decay;
    h.weighting.frequencyExponent = exponent;
    h.patternDigest = tqs::pattern_digest(make_pattern(opaque, period));
    return h;
}

int ref_save_cache(void* cache, const char* path, const uint8_t* opaque, int period, int window,
                   int precision_double, double decay, double exponent) {
    try {
        tqs::save_kernel_cache(path, *static_cast<tqs::KernelCache*>(cache),
                               cache_header(opaque, period, window, precision_double, decay, exponent));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

int ref_load_cache(void* cache, const char* path, const uint8_t* opaque, int period, int window,
                   int precision_double, double decay, double exponent) {
    try {
        tqs::load_kernel_cache(path, *static_cast<tqs::KernelCache*>(cache),
                               cache_header(opaque, period, window, precision_double, decay, exponent));
        return static_cast<int>(static_cast<tqs::KernelCache*>(cache)->classCount());
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

int ref_memory_report(int classes, int window, int precision_double, int local, uint64_t out[4]) {
    try {
        const tqs::MemoryReport r = tqs::kernel_memory_report(
            classes, window, precision_double ? tqs::Precision::Double : tqs::Precision::Single, local);
        out[0] = r.bBytes, out[1] = r.cBytes, out[2] = r.dBytes, out[3] = r.totalBytes;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    }
}

// ---------------------------------------------------------------- L-JSDE
// tqs::reconstruct with an explicit algorithm (0 = Ljsde, 1 = Rljsde), unclipped
// or clipped, no external cache.
int ref_reconstruct_algo(const double* frame, int frame_rows, int frame_cols, const uint8_t* opaque,
                         int period, int window, int block, int iterations, double step_width,
                         int algo, int clip, int threads, double* out, double* seconds) {
    try {
        tqs::MeasurementFrame f(frame_rows, frame_cols);
        std::memcpy(f.values.data(), frame, f.values.size() * sizeof(double));
        tqs::ReconstructionConfig cfg;
        cfg.window = window;
        cfg.block = block;
        cfg.solver.maxIterations = iterations;
        cfg.solver.stepWidth = step_width;
        cfg.clipOutput = clip != 0;
        cfg.algorithm = algo == 0 ? tqs::Algorithm::Ljsde : tqs::Algorithm::Rljsde;
        cfg.threads = threads;
        const tqs::ReconstructionReport r = tqs::reconstruct(f, make_pattern(opaque, period), cfg);
        std::memcpy(out, r.output.values.data(), r.output.values.size() * sizeof(double));
        if (seconds) *seconds = r.seconds;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

// ljsde_block on the window at (origin_row, origin_col) with the reference's local
// system and weights: picks / scaled deltas per iteration and the W*W synthesis.
int ref_ljsde_trace(const uint8_t* opaque, int period, int origin_row, int origin_col, int window,
                    const double* y_local, int iterations, double step_width,
                    double early_stop_scale, int* picks, double* gd, double* window_out) {
    try {
        const tqs::QuadrantPattern p = make_pattern(opaque, period);
        const tqs::LocalMeasurementMatrix A = tqs::extract_local_matrix(p, origin_row, origin_col, window);
        const std::vector<double> w = tqs::spatial_weights(A, tqs::WeightingConfig{});
        const std::vector<double> q = tqs::frequency_weights(window, tqs::WeightingConfig{});
        tqs::SolverOptions opt;
        opt.maxIterations = iterations;
        opt.stepWidth = step_width;
        opt.earlyStop = early_stop_scale > 0.0;  // <= 0: no energy stop
        if (opt.earlyStop) opt.earlyStopScale = early_stop_scale;
        int n = 0;
        const std::vector<double> y(y_local, y_local + A.localCount());
        const std::vector<double> win = tqs::ljsde_block(
            y, A, w, q, opt, [&](int it, int u, tqs::cplx g, std::span<const tqs::cplx>) {
                picks[it] = u;
                gd[2 * it] = g.real();
                gd[2 * it + 1] = g.imag();
                n = it + 1;
            });
        std::memcpy(window_out, win.data(), win.size() * sizeof(double));
        return n;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

} // extern "C"
