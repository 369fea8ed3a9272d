// reconstruct.hpp -- header-only C++ drop-in for the reference entry point
//
//   tqs::ReconstructionReport tqs::reconstruct(const MeasurementFrame&, const QuadrantPattern&,
//                                              const ReconstructionConfig&, KernelCache* = nullptr,
//                                              const Image* reference = nullptr);
//   (/root/reference/proj/include/tqs/pipeline.hpp:45-47)
//
// The types mirror the reference's (image.hpp:10-27, grid.hpp:19-53, basis.hpp:15-18 and
// 77-82, pipeline.hpp:17-39) field for field, so existing call sites compile against
// namespace tqsb unchanged; the work runs on the GPU through the C ABI in tqsb.h.
// Errors are rethrown as the reference's exception types: std::invalid_argument
// (validation, pipeline.cpp:27-42), std::logic_error (cache window mismatch,
// pipeline.cpp:146-147), std::runtime_error (device failures).
//
// KernelCache is the device-resident table store (the reference's shared KernelCache,
// pipeline.cpp:110-133, rljsde.hpp:81-100): it holds the fp64 B, C, D tables per
// offset class on the GPU, bound to the window (and pattern) of its first use, with
// hits()/misses() counters. Every call through it runs with that call's own config --
// nu, gamma, block, clip, frequency exponent and compute -- like the reference's.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "tqsb.h"

namespace tqsb {

struct Image {
    int rows = 0;
    int cols = 0;
    std::vector<double> values;
    Image() = default;
    Image(int r, int c, double fill = 0.0) : rows(r), cols(c), values(size_t(r) * c, fill) {
        if (r < 0 || c < 0) throw std::invalid_argument("image dimensions must be non-negative");
    }
    double& at(int r, int c) { return values[size_t(r) * cols + c]; }
    double at(int r, int c) const { return values[size_t(r) * cols + c]; }
    size_t size() const { return values.size(); }
    bool same_size(const Image& o) const { return rows == o.rows && cols == o.cols; }
};

struct MeasurementFrame {
    int rows = 0;
    int cols = 0;
    std::vector<double> values;
    MeasurementFrame() = default;
    MeasurementFrame(int r, int c, double fill = 0.0) : rows(r), cols(c), values(size_t(r) * c, fill) {}
    double& at(int r, int c) { return values[size_t(r) * cols + c]; }
    double at(int r, int c) const { return values[size_t(r) * cols + c]; }
    size_t size() const { return values.size(); }
};

struct QuadrantPattern {
    int period = 0;
    uint64_t seed = 0;
    std::string rng;
    std::vector<uint8_t> opaque;
    int cellsPerPeriod() const { return period / 2; }
};

enum class Precision { Single, Double };
enum class Algorithm { Ljsde, Rljsde };
enum class Compute { Fp32, Fp64 };  // device arithmetic (not in the reference)

struct WeightingConfig {
    double spatialDecay = 0.8;
    double frequencyExponent = 2.0;
};

struct SolverOptions {
    int maxIterations = 200;
    double stepWidth = 0.5;
    bool earlyStop = false;  // L-JSDE only (basis.hpp:80-81); ignored by RL-JSDE like the reference
    double earlyStopScale = 1e-14;
};

struct ReconstructionConfig {
    int window = 32;
    int block = 4;
    SolverOptions solver;
    WeightingConfig weighting;
    Precision precision = Precision::Double;
    bool clipOutput = true;
    Algorithm algorithm = Algorithm::Rljsde;
    int threads = 1;
    Compute compute = Compute::Fp32;
    int hotColumns = -1;
    std::vector<int> devices{0};
};

struct ReconstructionReport {
    Image output;
    double seconds = 0.0;
    double warmSeconds = 0.0;
    long blocksProcessed = 0;
    size_t classesTotal = 0;
    size_t classesInterior = 0;
    size_t classesCreated = 0;
    uint64_t cacheHits = 0;
    uint64_t cacheMisses = 0;
    std::optional<double> psnrDb;
    double e2eSeconds = 0.0;
    Compute compute = Compute::Fp32;  // the arithmetic the call ran in (tqsb_report::compute)
};

namespace detail {
[[noreturn]] inline void throw_status(int rc) {
    const std::string msg = tqsb_last_error();
    switch (rc) {
        case TQSB_EINVAL: throw std::invalid_argument(msg);
        case TQSB_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}
inline void check(int rc) {
    if (rc != TQSB_OK) throw_status(rc);
}
inline tqsb_config to_c(const ReconstructionConfig& c) {
    tqsb_config k;
    tqsb_config_default(&k);
    k.window = c.window;
    k.block = c.block;
    k.max_iterations = c.solver.maxIterations;
    k.step_width = c.solver.stepWidth;
    k.spatial_decay = c.weighting.spatialDecay;
    k.frequency_exponent = c.weighting.frequencyExponent;
    k.precision = c.precision == Precision::Double ? TQSB_PRECISION_DOUBLE : TQSB_PRECISION_SINGLE;
    k.clip_output = c.clipOutput ? 1 : 0;
    k.threads = c.threads;
    k.compute = c.compute == Compute::Fp64 ? TQSB_COMPUTE_FP64 : TQSB_COMPUTE_FP32;
    k.hot_columns = c.hotColumns;
    k.algorithm = c.algorithm == Algorithm::Ljsde ? TQSB_ALGO_LJSDE : TQSB_ALGO_RLJSDE;
    k.early_stop = c.solver.earlyStop ? 1 : 0;
    k.early_stop_scale = c.solver.earlyStopScale;
    return k;
}
}  // namespace detail

// Device-resident kernel store (the reference's KernelCache, rljsde.hpp:81-100).
class KernelCache {
public:
    KernelCache() = default;
    KernelCache(const KernelCache&) = delete;
    KernelCache& operator=(const KernelCache&) = delete;
    ~KernelCache() { clear(); }

    size_t classCount() const {
        long long n = 0;
        if (plan_) tqsb_plan_stats(plan_, &n, nullptr);
        return size_t(n);
    }
    uint64_t hits() const { return hits_; }
    uint64_t misses() const { return misses_; }
    void resetStats() { hits_ = misses_ = 0; }
    void clear() {
        if (plan_) tqsb_plan_destroy(plan_);
        plan_ = nullptr;
        window_ = 0;
    }

    // internal: bind on first use; a different window is the reference's logic_error
    // (pipeline.cpp:146-147). The config's solver options are per call, not bound.
    tqsb_plan* bind(const QuadrantPattern& p, const ReconstructionConfig& c) {
        if (plan_) {
            if (window_ != c.window)
                throw std::logic_error("kernel cache holds a different window size");
            return plan_;
        }
        const tqsb_config k = detail::to_c(c);
        detail::check(tqsb_plan_create(p.opaque.data(), p.period, &k, c.devices.data(),
                                       int(c.devices.size()), &plan_));
        window_ = c.window;
        return plan_;
    }
    void count(uint64_t h, uint64_t m) {
        hits_ += h;
        misses_ += m;
    }

private:
    tqsb_plan* plan_ = nullptr;
    int window_ = 0;
    uint64_t hits_ = 0, misses_ = 0;
};

inline ReconstructionReport reconstruct(const MeasurementFrame& frame, const QuadrantPattern& pattern,
                                        const ReconstructionConfig& config,
                                        KernelCache* cache = nullptr,
                                        const Image* reference = nullptr) {
    const tqsb_config k = detail::to_c(config);
    detail::check(tqsb_validate_config(&k, pattern.period));
    if (frame.rows < 1 || frame.cols < 1) throw std::invalid_argument("empty measurement frame");
    if (reference && (reference->rows != 2 * frame.rows || reference->cols != 2 * frame.cols))
        throw std::invalid_argument("reference dimensions do not match the reconstruction");
    // the reference shares its cache with RL-JSDE only (pipeline.cpp:111-112): an
    // L-JSDE call leaves a caller's cache untouched
    KernelCache local;
    KernelCache* kc = cache && config.algorithm == Algorithm::Rljsde ? cache : &local;
    tqsb_plan* plan = kc->bind(pattern, config);
    ReconstructionReport rep;
    rep.output = Image(2 * frame.rows, 2 * frame.cols);
    tqsb_report r;
    detail::check(tqsb_reconstruct_with(plan, &k, frame.values.data(), frame.rows, frame.cols,
                                        rep.output.values.data(),
                                        reference ? reference->values.data() : nullptr, &r));
    rep.compute = r.compute == TQSB_COMPUTE_FP64 ? Compute::Fp64 : Compute::Fp32;
    rep.seconds = r.seconds;
    rep.warmSeconds = r.warm_seconds;
    rep.e2eSeconds = r.e2e_seconds;
    rep.blocksProcessed = long(r.blocks_processed);
    rep.classesTotal = size_t(r.classes_total);
    rep.classesInterior = size_t(r.classes_interior);
    rep.classesCreated = size_t(r.classes_created);
    rep.cacheHits = uint64_t(r.cache_hits);
    rep.cacheMisses = uint64_t(r.cache_misses);
    if (r.has_psnr) rep.psnrDb = r.psnr_db;
    if (config.algorithm == Algorithm::Ljsde) {  // no cache, no counters (pipeline.cpp:173-177)
        rep.cacheHits = rep.cacheMisses = 0;
        rep.classesCreated = 0;
    }
    kc->count(rep.cacheHits, rep.cacheMisses);
    return rep;
}

// ---- pipeline.hpp:49-64 helpers (pipeline.cpp:187-256) ----
struct PaddedImage {
    Image image;
    int originalRows = 0;
    int originalCols = 0;
};

// edge-replication padding to even, block-multiple dimensions (pipeline.cpp:187-209)
inline PaddedImage pad_to_block_multiple(const Image& image, int block) {
    if (block < 1) throw std::invalid_argument("block size must be positive");
    if (image.rows < 1 || image.cols < 1) throw std::invalid_argument("empty image");
    const int step = std::lcm(block, 2);
    PaddedImage out;
    out.originalRows = image.rows;
    out.originalCols = image.cols;
    const int rows = (image.rows + step - 1) / step * step, cols = (image.cols + step - 1) / step * step;
    if (rows == image.rows && cols == image.cols) {
        out.image = image;
        return out;
    }
    out.image = Image(rows, cols);
    for (int r = 0; r < rows; ++r) {
        const double* src = &image.values[size_t(std::min(r, image.rows - 1)) * image.cols];
        double* dst = &out.image.values[size_t(r) * cols];
        std::copy(src, src + image.cols, dst);
        std::fill(dst + image.cols, dst + cols, src[image.cols - 1]);
    }
    return out;
}

// top-left rows x cols (pipeline.cpp:211-219)
inline Image crop_image(const Image& image, int rows, int cols) {
    if (rows < 0 || cols < 0 || rows > image.rows || cols > image.cols)
        throw std::invalid_argument("crop exceeds image bounds");
    Image out(rows, cols);
    for (int r = 0; r < rows; ++r)
        std::copy_n(&image.values[size_t(r) * image.cols], cols, &out.values[size_t(r) * cols]);
    return out;
}

// each measurement value copied to its 2x2 cell, the quality baseline (pipeline.cpp:235-246)
inline Image nn_upsample(const MeasurementFrame& frame) {
    Image out(2 * frame.rows, 2 * frame.cols);
    for (int r = 0; r < frame.rows; ++r)
        for (int c = 0; c < frame.cols; ++c) {
            const double v = frame.at(r, c);
            out.at(2 * r, 2 * c) = v;
            out.at(2 * r, 2 * c + 1) = v;
            out.at(2 * r + 1, 2 * c) = v;
            out.at(2 * r + 1, 2 * c + 1) = v;
        }
    return out;
}

inline MeasurementFrame simulate_measurement(const Image& image, const QuadrantPattern& pattern);
inline double psnr(const Image& reference, const Image& estimate);

// simulate + reconstruct + PSNR against the unpadded input (pipeline.cpp:248-256): the
// acceptance and benchmark call shape
inline ReconstructionReport reconstruct_image(const Image& image, const QuadrantPattern& pattern,
                                              const ReconstructionConfig& config,
                                              KernelCache* cache = nullptr) {
    PaddedImage padded = pad_to_block_multiple(image, config.block);
    MeasurementFrame frame = simulate_measurement(padded.image, pattern);
    ReconstructionReport report = reconstruct(frame, pattern, config, cache);
    report.output = crop_image(report.output, padded.originalRows, padded.originalCols);
    report.psnrDb = psnr(image, report.output);
    return report;
}

// ---- bench (pipeline.hpp:78-100, pipeline.cpp:258-329) ----
struct BenchResult {
    int images = 0;
    double ljsdeMeanSeconds = 0.0;
    double rljsdeMeanSeconds = 0.0;      // excluding table precompute
    double rljsdeMeanWarmSeconds = 0.0;  // precompute, averaged over runs
    double speedup = 0.0;                // ljsde / rljsde (excl. precompute)
    double speedupInclWarm = 0.0;
    double maxAbsDifference = 0.0;       // worst pixel deviation across the set
    bool scalingMeasured = false;        // per-block times at W=16 vs the config's window
    double ljsdePerBlockSmall = 0.0, ljsdePerBlockLarge = 0.0;
    double rljsdePerBlockSmall = 0.0, rljsdePerBlockLarge = 0.0;
    double ljsdeScalingRatio = 0.0;
    double rljsdeScalingRatio = 0.0;
};

// thrown when the two algorithms diverge beyond the threshold (pipeline.hpp:94-97)
class EquivalenceError : public std::runtime_error {
public:
    EquivalenceError(const std::string& what, double maxAbs)
        : std::runtime_error(what), maxAbsDifference(maxAbs) {}
    double maxAbsDifference;
};

// L-JSDE vs RL-JSDE on the same frames, both on the device: L-JSDE always runs in
// fp64; RL-JSDE in the config's compute (Compute::Fp64 reproduces the reference's
// arithmetic and meets its 1e-6 bar; the fp32 product path meets the product tolerance).
inline BenchResult bench(const std::vector<Image>& images, const QuadrantPattern& pattern,
                         const ReconstructionConfig& config, double equivalenceThreshold = 1e-6,
                         bool measureScaling = false) {
    if (images.empty()) throw std::invalid_argument("bench requires at least one image");
    ReconstructionConfig cfgL = config;
    cfgL.algorithm = Algorithm::Ljsde;
    cfgL.threads = 1;
    cfgL.clipOutput = false;
    ReconstructionConfig cfgR = cfgL;
    cfgR.algorithm = Algorithm::Rljsde;
    BenchResult result;
    result.images = int(images.size());
    KernelCache cache;
    double sumL = 0.0, sumR = 0.0, sumWarm = 0.0;
    for (const Image& image : images) {
        PaddedImage padded = pad_to_block_multiple(image, config.block);
        MeasurementFrame frame = simulate_measurement(padded.image, pattern);
        ReconstructionReport runL = reconstruct(frame, pattern, cfgL);
        ReconstructionReport runR = reconstruct(frame, pattern, cfgR, &cache);
        sumL += runL.seconds;
        sumR += runR.seconds;
        sumWarm += runR.warmSeconds;
        for (size_t i = 0; i < runL.output.size(); ++i)
            result.maxAbsDifference = std::max(
                result.maxAbsDifference, std::abs(runL.output.values[i] - runR.output.values[i]));
    }
    result.ljsdeMeanSeconds = sumL / result.images;
    result.rljsdeMeanSeconds = sumR / result.images;
    result.rljsdeMeanWarmSeconds = sumWarm / result.images;
    result.speedup = result.rljsdeMeanSeconds > 0.0 ? result.ljsdeMeanSeconds / result.rljsdeMeanSeconds
                                                    : std::numeric_limits<double>::infinity();
    const double inclusive = result.rljsdeMeanSeconds + result.rljsdeMeanWarmSeconds;
    result.speedupInclWarm = inclusive > 0.0 ? result.ljsdeMeanSeconds / inclusive
                                             : std::numeric_limits<double>::infinity();
    if (result.maxAbsDifference > equivalenceThreshold)
        throw EquivalenceError("algorithms diverged: max abs difference " +
                                   std::to_string(result.maxAbsDifference) + " exceeds " +
                                   std::to_string(equivalenceThreshold),
                               result.maxAbsDifference);
    if (measureScaling) {
        PaddedImage padded = pad_to_block_multiple(images.front(), config.block);
        MeasurementFrame frame = simulate_measurement(padded.image, pattern);
        // one untimed call first (the window's kernels load lazily on first launch and the
        // tables are built), then the best of three: a single device call on a small frame
        // is otherwise dominated by one-off costs
        auto perBlock = [&](Algorithm algo, int window, double& out) {
            ReconstructionConfig cfg = cfgL;
            cfg.algorithm = algo;
            cfg.window = window;
            KernelCache scalingCache;  // tables are window-specific
            KernelCache* cache = algo == Algorithm::Rljsde ? &scalingCache : nullptr;
            reconstruct(frame, pattern, cfg, cache);
            out = std::numeric_limits<double>::infinity();
            for (int rep = 0; rep < 3; ++rep) {
                const ReconstructionReport run = reconstruct(frame, pattern, cfg, cache);
                out = std::min(out, run.seconds / double(run.blocksProcessed));
            }
        };
        perBlock(Algorithm::Ljsde, 16, result.ljsdePerBlockSmall);
        perBlock(Algorithm::Ljsde, config.window, result.ljsdePerBlockLarge);
        perBlock(Algorithm::Rljsde, 16, result.rljsdePerBlockSmall);
        perBlock(Algorithm::Rljsde, config.window, result.rljsdePerBlockLarge);
        result.ljsdeScalingRatio = result.ljsdePerBlockLarge / result.ljsdePerBlockSmall;
        result.rljsdeScalingRatio = result.rljsdePerBlockLarge / result.rljsdePerBlockSmall;
        result.scalingMeasured = true;
    }
    return result;
}

// ---- kernel-cache persistence and accounting (rljsde.hpp:102-131) ----
struct KernelCacheHeader {
    int window = 0;
    int period = 0;
    Precision precision = Precision::Double;
    WeightingConfig weighting;
    uint64_t patternDigest = 0;
};

// pattern_digest (rljsde.cpp:322-333)
inline uint64_t pattern_digest(const QuadrantPattern& pattern) {
    return tqsb_pattern_digest(pattern.opaque.data(), pattern.period);
}

// TQSK files (rljsde.cpp:337-475). The device store must be bound to its pattern and
// config first (KernelCache::bind); the header is validated against that binding.
inline void save_kernel_cache(const std::string& path, KernelCache& cache, const QuadrantPattern& p,
                              const ReconstructionConfig& c) {
    detail::check(tqsb_plan_save_tables(cache.bind(p, c), path.c_str(), nullptr));
}
inline size_t load_kernel_cache(const std::string& path, KernelCache& cache, const QuadrantPattern& p,
                                const ReconstructionConfig& c) {
    int n = 0;
    detail::check(tqsb_plan_load_tables(cache.bind(p, c), path.c_str(), &n));
    return size_t(n);
}

struct MemoryReport {
    uint64_t bBytes = 0, cBytes = 0, dBytes = 0, totalBytes = 0;
    double bMegabytes() const { return double(bBytes) / 1e6; }
    double cMegabytes() const { return double(cBytes) / 1e6; }
    double dMegabytes() const { return double(dBytes) / 1e6; }
    double totalMegabytes() const { return double(totalBytes) / 1e6; }
};

// kernel_memory_report (rljsde.cpp:322-335)
inline MemoryReport kernel_memory_report(int classes, int window, Precision precision, int local = -1) {
    uint64_t o[4];
    detail::check(tqsb_kernel_memory_report(
        classes, window, precision == Precision::Single ? TQSB_PRECISION_SINGLE : TQSB_PRECISION_DOUBLE,
        local, o));
    return MemoryReport{o[0], o[1], o[2], o[3]};
}

// generate_pattern (grid.cpp:8-26)
inline QuadrantPattern generate_pattern(uint64_t seed, int period, int blockSize = 4) {
    QuadrantPattern p;
    p.period = period;
    p.seed = seed;
    p.rng = "mt19937_64";
    if (period < 4 || period % 2 != 0)
        throw std::invalid_argument("pattern period must be even and >= 4");
    p.opaque.resize(size_t(period / 2) * (period / 2));
    detail::check(tqsb_generate_pattern(seed, period, blockSize, p.opaque.data()));
    return p;
}

// simulate_measurement (grid.cpp:46-66)
inline MeasurementFrame simulate_measurement(const Image& image, const QuadrantPattern& pattern) {
    if (image.rows % 2 != 0 || image.cols % 2 != 0)
        throw std::invalid_argument("image dimensions must be even");
    MeasurementFrame f(image.rows / 2, image.cols / 2);
    detail::check(tqsb_simulate(image.values.data(), image.rows, image.cols,
                                pattern.opaque.data(), pattern.period, f.values.data()));
    return f;
}

// psnr (pipeline.cpp:221-233)
inline double psnr(const Image& reference, const Image& estimate) {
    if (!reference.same_size(estimate)) throw std::invalid_argument("psnr: dimension mismatch");
    return tqsb_psnr(reference.values.data(), estimate.values.data(),
                     (long long)reference.values.size());
}

namespace testing {
// tests/support/synthetic.cpp:9-80
inline Image synthetic_image(int rows, int cols, uint64_t seed) {
    Image img(rows, cols);
    detail::check(tqsb_synthetic_image(rows, cols, seed, img.values.data()));
    return img;
}
}  // namespace testing

}  // namespace tqsb
