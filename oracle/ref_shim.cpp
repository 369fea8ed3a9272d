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
// Exceptions never cross the ABI: they become a negative return code and the
// message is kept for ref_last_error().

#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "synthetic.hpp"
#include "tqs/basis.hpp"
#include "tqs/grid.hpp"
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

} // extern "C"
