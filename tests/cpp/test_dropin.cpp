// C++ drop-in check: the reference's pipeline test cases (test_pipeline.cpp) written
// against include/tqsb/reconstruct.hpp -- the same call shapes as tqs::reconstruct,
// the same exception types -- running on the GPU through libtqsb.so.
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "tqsb/reconstruct.hpp"

using namespace tqsb;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(cond)) {                                                         \
            ++g_fail;                                                          \
            std::printf("  FAILED %s:%d  %s\n", __FILE__, __LINE__, #cond);    \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                               \
    do {                                                                       \
        ++g_checks;                                                            \
        bool ok = false;                                                       \
        try { (void)(expr); } catch (const T&) { ok = true; } catch (...) {}   \
        if (!ok) { ++g_fail; std::printf("  FAILED %s:%d  %s throws %s\n", __FILE__, __LINE__, #expr, #T); } \
    } while (0)

static void run(const char* name, const std::function<void()>& f) {
    const int before = g_fail;
    try {
        f();
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("  EXCEPTION %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

static ReconstructionConfig test_config(int window = 16, int iterations = 30) {
    ReconstructionConfig cfg;
    cfg.window = window;
    cfg.block = 4;
    cfg.solver.maxIterations = iterations;
    cfg.clipOutput = false;
    cfg.threads = 1;
    return cfg;
}

int main() {
    run("configuration validation (test_pipeline.cpp:105-147)", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const Image img = testing::synthetic_image(64, 64, 4);
        const MeasurementFrame f = simulate_measurement(img, p);
        auto expectThrow = [&](ReconstructionConfig cfg) {
            CHECK_THROWS_AS(reconstruct(f, p, cfg), std::invalid_argument);
        };
        ReconstructionConfig cfg = test_config(); cfg.window = 7; expectThrow(cfg);
        cfg = test_config(); cfg.block = 3; expectThrow(cfg);
        cfg = test_config(6); cfg.block = 3; expectThrow(cfg);
        cfg = test_config(); cfg.solver.maxIterations = -1; expectThrow(cfg);
        cfg = test_config(); cfg.solver.stepWidth = 0.0; expectThrow(cfg);
        cfg = test_config(); cfg.solver.stepWidth = 1.5; expectThrow(cfg);
        cfg = test_config(); cfg.threads = -2; expectThrow(cfg);
        const QuadrantPattern p6 = generate_pattern(3, 6, 2);
        CHECK_THROWS_AS(reconstruct(f, p6, test_config()), std::invalid_argument);
        const Image tiny = testing::synthetic_image(16, 16, 5);
        const MeasurementFrame tf = simulate_measurement(tiny, p);
        CHECK_THROWS_AS(reconstruct(tf, p, test_config(32)), std::invalid_argument);
        CHECK_THROWS_AS(reconstruct(MeasurementFrame(), p, test_config()), std::invalid_argument);
    });

    run("block tiling covers the frame exactly (test_pipeline.cpp:149-167)", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const Image img(64, 64, 0.6);
        const MeasurementFrame f = simulate_measurement(img, p);
        ReconstructionConfig cfg = test_config(16, 1);
        cfg.solver.stepWidth = 1.0;
        cfg.compute = Compute::Fp64;
        const ReconstructionReport report = reconstruct(f, p, cfg, nullptr, &img);
        CHECK(report.blocksProcessed == 256);
        CHECK(report.output.rows == 64 && report.output.cols == 64);
        bool all = true;
        for (double v : report.output.values) all = all && std::abs(v - 0.6) <= 0.6 * 1e-10;
        CHECK(all);
        CHECK(report.psnrDb.has_value() && *report.psnrDb >= 60.0);
    });

    run("offset class accounting on an aligned image (test_pipeline.cpp:169-190)", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const Image img = testing::synthetic_image(64, 64, 6);
        const MeasurementFrame f = simulate_measurement(img, p);
        const ReconstructionReport r32 = reconstruct(f, p, test_config(32, 2));
        CHECK(r32.classesInterior == 64);
        CHECK(r32.classesTotal == 81);
        CHECK(r32.classesCreated == 81);
        CHECK(r32.cacheMisses == 81);
        CHECK(r32.cacheHits == 256);
        const ReconstructionReport r16 = reconstruct(f, p, test_config(16, 2));
        CHECK(r16.classesInterior == 64);
        CHECK(r16.classesTotal == 100);
    });

    run("external kernel cache is reused across runs (test_pipeline.cpp:192-217)", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const Image img = testing::synthetic_image(64, 64, 7);
        const MeasurementFrame f = simulate_measurement(img, p);
        ReconstructionConfig cfg = test_config(16, 3);
        KernelCache cache;
        const ReconstructionReport first = reconstruct(f, p, cfg, &cache);
        CHECK(first.classesCreated == first.classesTotal);
        CHECK(cache.classCount() == first.classesTotal);
        const ReconstructionReport second = reconstruct(f, p, cfg, &cache);
        CHECK(second.classesCreated == 0);
        CHECK(second.cacheMisses == 0);
        CHECK(second.output.values == first.output.values);
        CHECK_THROWS_AS(reconstruct(f, p, test_config(32, 3), &cache), std::logic_error);

        // the baseline path never touches the cache
        ReconstructionConfig cfgL = cfg;
        cfgL.algorithm = Algorithm::Ljsde;
        cfgL.solver.maxIterations = 2;
        KernelCache untouched;
        const ReconstructionReport viaL = reconstruct(f, p, cfgL, &untouched);
        CHECK(untouched.classCount() == 0);
        CHECK(viaL.cacheHits == 0);
        CHECK(viaL.cacheMisses == 0);
        CHECK(viaL.compute == Compute::Fp64);
    });

    run("one shared cache, per-call solver options (pipeline.cpp:108-166)", [] {
        // every call through one cache must equal a fresh, cache-less call with the same
        // config bit for bit: nu, gamma, clip, frequency exponent, block and compute are
        // the call's, never the first call's
        const QuadrantPattern p = generate_pattern(7, 32);
        const Image img = testing::synthetic_image(64, 64, 12);
        const MeasurementFrame f = simulate_measurement(img, p);
        KernelCache cache;
        struct V { int nu; double gamma; bool clip; double expo; int block; Compute compute; };
        const V vs[] = {{50, 1.0, false, 2.0, 4, Compute::Fp32}, {200, 0.5, true, 2.0, 4, Compute::Fp32},
                        {50, 0.5, false, 1.0, 4, Compute::Fp32}, {200, 1.0, true, 1.0, 2, Compute::Fp32},
                        {50, 0.5, false, 2.0, 4, Compute::Fp64}, {120, 1.0, true, 1.0, 2, Compute::Fp64},
                        {50, 1.0, false, 2.0, 4, Compute::Fp32}};
        size_t created = 0;
        for (const V& v : vs) {
            ReconstructionConfig cfg = test_config(16, v.nu);
            cfg.solver.stepWidth = v.gamma;
            cfg.clipOutput = v.clip;
            cfg.weighting.frequencyExponent = v.expo;
            cfg.block = v.block;
            cfg.compute = v.compute;
            const ReconstructionReport viaCache = reconstruct(f, p, cfg, &cache);
            const ReconstructionReport fresh = reconstruct(f, p, cfg);
            CHECK(viaCache.output.values == fresh.output.values);
            CHECK(viaCache.compute == v.compute);
            created += viaCache.classesCreated;
        }
        CHECK(created == cache.classCount());  // tables were built once per class
    });

    run("outputs are bitwise reproducible across runs (test_pipeline.cpp:238-262)", [] {
        const QuadrantPattern p = generate_pattern(11, 32);
        const Image img = testing::synthetic_image(64, 64, 9);
        const MeasurementFrame f = simulate_measurement(img, p);
        const ReconstructionConfig cfg = test_config(16, 25);
        const ReconstructionReport a = reconstruct(f, p, cfg);
        const ReconstructionReport b = reconstruct(f, p, cfg);
        CHECK(a.output.values == b.output.values);
    });

    run("clipping bounds the output to the display range (test_pipeline.cpp:264-276)", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const Image img = testing::synthetic_image(64, 64, 10);
        const MeasurementFrame f = simulate_measurement(img, p);
        ReconstructionConfig cfg = test_config(16, 40);
        cfg.clipOutput = true;
        const ReconstructionReport report = reconstruct(f, p, cfg);
        bool ok = true;
        for (double v : report.output.values) ok = ok && v >= 0.0 && v <= 1.0;
        CHECK(ok);
    });

    run("odd-sized images go through padding and come back cropped (test_pipeline.cpp:278-294)", [] {
        const QuadrantPattern p = generate_pattern(13, 32);
        const Image img = testing::synthetic_image(33, 38, 11);
        ReconstructionConfig cfg = test_config(16, 20);
        cfg.clipOutput = true;
        const ReconstructionReport report = reconstruct_image(img, p, cfg);
        CHECK(report.output.rows == 33);
        CHECK(report.output.cols == 38);
        CHECK(report.psnrDb.has_value());
        CHECK(std::isfinite(*report.psnrDb));
        CHECK(*report.psnrDb > 10.0);
        const MeasurementFrame f = simulate_measurement(pad_to_block_multiple(img, 4).image, p);
        const Image wrongRef(10, 10);
        CHECK_THROWS_AS(reconstruct(f, p, cfg, nullptr, &wrongRef), std::invalid_argument);
        // the helpers themselves (pipeline.cpp:187-246)
        const PaddedImage pad = pad_to_block_multiple(img, 4);
        CHECK(pad.image.rows == 36 && pad.image.cols == 40);
        CHECK(pad.originalRows == 33 && pad.originalCols == 38);
        CHECK(pad.image.at(35, 39) == img.at(32, 37) && pad.image.at(2, 39) == img.at(2, 37));
        CHECK(crop_image(pad.image, 33, 38).values == img.values);
        CHECK_THROWS_AS(crop_image(img, 34, 38), std::invalid_argument);
        CHECK_THROWS_AS(pad_to_block_multiple(img, 0), std::invalid_argument);
        const Image nn = nn_upsample(f);
        CHECK(nn.rows == 2 * f.rows && nn.at(3, 5) == f.at(1, 2));
    });

    run("bench compares the algorithms end to end (test_pipeline.cpp:296-320)", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const std::vector<Image> images{testing::synthetic_image(48, 48, 20),
                                        testing::synthetic_image(48, 48, 21)};
        ReconstructionConfig cfg = test_config(16, 25);
        cfg.compute = Compute::Fp64;  // the reference's arithmetic: its 1e-6 bar
        const BenchResult result = bench(images, p, cfg, 1e-6, false);
        CHECK(result.images == 2);
        CHECK(result.maxAbsDifference <= 1e-6);
        CHECK(result.ljsdeMeanSeconds > 0.0);
        CHECK(result.rljsdeMeanSeconds > 0.0);
        CHECK(result.speedup > 0.0);
        CHECK(result.speedupInclWarm <= result.speedup);
        CHECK(!result.scalingMeasured);
        bool threw = false;
        try {
            bench(images, p, cfg, -1.0, false);
        } catch (const EquivalenceError& e) {
            threw = e.maxAbsDifference >= 0.0 && std::string(e.what()).find("diverged") != std::string::npos;
        }
        CHECK(threw);
        CHECK_THROWS_AS(bench({}, p, cfg, 1e-6, false), std::invalid_argument);
        cfg.compute = Compute::Fp32;  // the product path within the product tolerance
        CHECK(bench(images, p, cfg, 1e-2, false).maxAbsDifference <= 1e-2);
    });

    run("bench scaling pass separates the two iteration costs (test_pipeline.cpp:322-345)", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const std::vector<Image> images{testing::synthetic_image(64, 64, 22)};
        ReconstructionConfig cfg = test_config(32, 30);
        cfg.compute = Compute::Fp64;
        const BenchResult result = bench(images, p, cfg, 1e-6, true);
        CHECK(result.scalingMeasured);
        CHECK(result.ljsdePerBlockSmall > 0.0 && result.ljsdePerBlockLarge > 0.0);
        CHECK(result.rljsdePerBlockSmall > 0.0 && result.rljsdePerBlockLarge > 0.0);
        CHECK(std::abs(result.ljsdeScalingRatio - result.ljsdePerBlockLarge / result.ljsdePerBlockSmall) < 1e-12);
        CHECK(std::abs(result.rljsdeScalingRatio - result.rljsdePerBlockLarge / result.rljsdePerBlockSmall) < 1e-12);
        CHECK(result.ljsdePerBlockLarge > result.ljsdePerBlockSmall);
        CHECK(result.rljsdePerBlockLarge > result.rljsdePerBlockSmall);
    });

    run("B > 16 runs like the reference (fp64 kernel), not EINVAL", [] {
        const QuadrantPattern p = generate_pattern(7, 32);
        const Image img = testing::synthetic_image(64, 64, 13);
        const MeasurementFrame f = simulate_measurement(img, p);
        ReconstructionConfig cfg = test_config(32, 20);
        cfg.block = 32;  // W = B = 32: W - B = 0 is even, B | P
        const ReconstructionReport r = reconstruct(f, p, cfg, nullptr, &img);
        CHECK(r.compute == Compute::Fp64);
        CHECK(r.blocksProcessed == 4);
        ReconstructionConfig c64 = cfg;
        c64.compute = Compute::Fp64;
        CHECK(reconstruct(f, p, c64).output.values == r.output.values);
    });

    run("production defaults beat nearest-neighbour upsampling", [] {
        const QuadrantPattern p = generate_pattern(7, 8);
        const Image img = testing::synthetic_image(128, 128, 301);
        const MeasurementFrame f = simulate_measurement(img, p);
        ReconstructionConfig cfg;  // W=32 B=4 nu=200 gamma=0.5, clip on, fp32
        const ReconstructionReport r = reconstruct(f, p, cfg, nullptr, &img);
        Image nn(128, 128);
        for (int y = 0; y < 128; ++y)
            for (int x = 0; x < 128; ++x) nn.at(y, x) = f.at(y / 2, x / 2);
        CHECK(r.psnrDb.has_value() && *r.psnrDb > psnr(img, nn));
        CHECK(r.blocksProcessed == 1024 && r.classesTotal == 9);
    });

    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
