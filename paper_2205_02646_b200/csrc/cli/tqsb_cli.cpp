// tqsb_cli.cpp -- `tqsb`, the command-line toolbox on the device library: the
// reference's `tqs` tool (tools/tqs.cpp:1-445) with the same subcommands, flags,
// defaults, text/JSON report layouts and exit codes:
//
//   pattern        --seed --period -o            generate_pattern -> TQSP file
//   simulate       --image --pattern -o          simulate_measurement -> TQSM frame
//   reconstruct    --input --pattern -o ...      tqsb::reconstruct (RL-JSDE or L-JSDE on the GPU)
//   compare        a b [--reference --threshold] max |a-b| gate, PSNR vs a reference
//   bench          --images DIR --pattern ...    L-JSDE vs RL-JSDE timing + equivalence gate
//   kernel-report  --classes --window ...        table byte accounting
//
// Exit codes (tqs.cpp:25-27): 0 success, 1 comparison failed or the algorithms
// diverged (EquivalenceError), 2 usage / input errors ("error: <what>" on stderr).
// JSON reports reproduce nlohmann::json::dump(2) (sorted keys, two-space indent,
// shortest round-trip numbers). Extensions beyond the reference are marked (ext).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <functional>
#include <iostream>
#include <map>
#include <numeric>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tqsb/io.hpp"
#include "tqsb/reconstruct.hpp"

namespace fs = std::filesystem;

namespace {

constexpr int kExitOk = 0;
constexpr int kExitCompareFailed = 1;
constexpr int kExitUsage = 2;

struct EquivalenceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ JSON output
// Numbers follow nlohmann's to_chars: the shortest digit string that round-trips,
// fixed notation for decimal exponents in (-4, 15] (integral values get ".0"),
// otherwise d.ddde+XX.
std::string json_number(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[40];
    int prec = 1;
    for (; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s(buf);
    std::string sign;
    if (s[0] == '-') sign = "-", s = s.substr(1);
    const size_t epos = s.find('e');
    std::string digits = s.substr(0, epos);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int e10 = std::atoi(s.c_str() + epos + 1);  // value = d.ddd x 10^e10
    const int k = int(digits.size()), n = e10 + 1;    // decimal point after n digits
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(size_t(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int ex = n - 1;
        char eb[8];
        std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', std::abs(ex));
        out += eb;
    }
    return sign + out;
}

std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (char ch : s) {
        switch (ch) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\t': o += "\\t"; break;
            default:
                if (static_cast<unsigned char>(ch) < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", ch);
                    o += b;
                } else {
                    o += ch;
                }
        }
    }
    return o + "\"";
}

class JsonObject {  // flat object, keys sorted like nlohmann's std::map-backed json
public:
    void num(const std::string& k, double v) { kv_[k] = json_number(v); }
    void integer(const std::string& k, long long v) { kv_[k] = std::to_string(v); }
    void uinteger(const std::string& k, unsigned long long v) { kv_[k] = std::to_string(v); }
    void boolean(const std::string& k, bool v) { kv_[k] = v ? "true" : "false"; }
    void str(const std::string& k, const std::string& v) { kv_[k] = json_string(v); }
    std::string dump() const {
        if (kv_.empty()) return "{}";
        std::string o = "{\n";
        size_t i = 0;
        for (const auto& [k, v] : kv_) o += "  " + json_string(k) + ": " + v + (++i < kv_.size() ? ",\n" : "\n");
        return o + "}";
    }

private:
    std::map<std::string, std::string> kv_;
};

// PSNR for reports: "identical" when +inf (tqs.cpp:41-54)
void psnr_json(JsonObject& j, const std::string& key, double db) {
    if (std::isinf(db))
        j.str(key, "identical");
    else
        j.num(key, db);
}
std::string psnr_text(double db) {
    if (std::isinf(db)) return "identical";
    char b[32];
    std::snprintf(b, sizeof b, "%.4f", db);
    return b;
}

// ------------------------------------------------------------------ argument parsing
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct HelpRequest {};

struct Opt {
    std::vector<std::string> names;  // e.g. {"-o", "--output"}
    std::string help;
    bool flag = false;
    bool required = false;
    std::function<void(const std::string&)> set;  // throws UsageError on bad values
    std::string shown_default;
    bool seen = false;
};

struct Positional {
    std::string name, help;
    bool required = true;
    std::function<void(const std::string&)> set;
    bool seen = false;
};

int to_int(const std::string& name, const std::string& v) {
    char* end = nullptr;
    errno = 0;
    const long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end || errno || x < INT32_MIN || x > INT32_MAX)
        throw UsageError("Could not convert: " + name + " = " + v);
    return int(x);
}
double to_double(const std::string& name, const std::string& v) {
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end) throw UsageError("Could not convert: " + name + " = " + v);
    return x;
}
uint64_t to_u64(const std::string& name, const std::string& v) {
    char* end = nullptr;
    errno = 0;
    const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
    if (v.empty() || *end || errno || v[0] == '-') throw UsageError("Could not convert: " + name + " = " + v);
    return x;
}

class Command {
public:
    Command(std::string name, std::string desc) : name_(std::move(name)), desc_(std::move(desc)) {}

    Command& opt(std::vector<std::string> names, std::string help, int& target, bool req = false) {
        const std::string n = names.back();
        add(names, help, false, req, [&target, n](const std::string& v) { target = to_int(n, v); },
            std::to_string(target));
        return *this;
    }
    Command& opt(std::vector<std::string> names, std::string help, double& target, bool req = false) {
        const std::string n = names.back();
        add(names, help, false, req, [&target, n](const std::string& v) { target = to_double(n, v); },
            json_number(target));
        return *this;
    }
    Command& opt(std::vector<std::string> names, std::string help, uint64_t& target, bool req = false) {
        const std::string n = names.back();
        add(names, help, false, req, [&target, n](const std::string& v) { target = to_u64(n, v); },
            std::to_string(target));
        return *this;
    }
    Command& opt(std::vector<std::string> names, std::string help, std::string& target, bool req = false,
                 std::vector<std::string> members = {}) {
        const std::string n = names.back();
        add(names, help, false, req,
            [&target, n, members](const std::string& v) {
                if (!members.empty() && std::find(members.begin(), members.end(), v) == members.end())
                    throw UsageError(n + ": " + v + " not in {" + join(members) + "}");
                target = v;
            },
            target);
        return *this;
    }
    Command& flag(std::vector<std::string> names, std::string help, bool& target) {
        add(names, help, true, false, [&target](const std::string&) { target = true; }, "");
        return *this;
    }
    Command& positional(std::string name, std::string help, std::string& target) {
        pos_.push_back(Positional{name, help, true, [&target](const std::string& v) { target = v; }});
        return *this;
    }

    void parse(const std::vector<std::string>& args) {
        size_t p = 0;
        for (size_t i = 0; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a == "--help" || a == "-h") throw HelpRequest{};
            if (a.size() > 1 && a[0] == '-' && !looks_numeric(a)) {
                std::string key = a, val;
                bool inline_val = false;
                const size_t eq = a.find('=');
                if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                    key = a.substr(0, eq);
                    val = a.substr(eq + 1);
                    inline_val = true;
                }
                Opt* o = find(key);
                if (!o) throw UsageError("The following arguments were not expected: " + a);
                if (o->flag) {
                    if (inline_val) throw UsageError(key + ": flag does not take a value");
                    o->set("");
                } else {
                    if (!inline_val) {
                        if (i + 1 >= args.size()) throw UsageError(key + " requires 1 argument");
                        val = args[++i];
                    }
                    o->set(val);
                }
                o->seen = true;
            } else {
                if (p >= pos_.size()) throw UsageError("The following arguments were not expected: " + a);
                pos_[p].set(a);
                pos_[p++].seen = true;
            }
        }
        for (const Opt& o : opts_)
            if (o.required && !o.seen) throw UsageError(o.names.back() + " is required");
        for (const Positional& q : pos_)
            if (q.required && !q.seen) throw UsageError(q.name + " is required");
    }

    std::string help() const {
        std::string h = desc_ + "\nUsage: tqsb " + name_ + " [OPTIONS]";
        for (const auto& q : pos_) h += " " + q.name;
        h += "\n\n";
        if (!pos_.empty()) {
            h += "Positionals:\n";
            for (const auto& q : pos_) h += "  " + pad(q.name) + q.help + " REQUIRED\n";
            h += "\n";
        }
        h += "Options:\n  " + pad("-h,--help") + "Print this help message and exit\n";
        for (const auto& o : opts_) {
            std::string n = join(o.names, ",");
            h += "  " + pad(n) + o.help;
            if (o.required) h += " REQUIRED";
            if (!o.flag && !o.shown_default.empty()) h += " [" + o.shown_default + "]";
            h += "\n";
        }
        return h;
    }
    const std::string& name() const { return name_; }
    const std::string& desc() const { return desc_; }

private:
    static bool looks_numeric(const std::string& a) {
        char* end = nullptr;
        std::strtod(a.c_str(), &end);
        return end && *end == '\0';
    }
    static std::string join(const std::vector<std::string>& v, const std::string& sep = ",") {
        std::string o;
        for (size_t i = 0; i < v.size(); ++i) o += (i ? sep : "") + v[i];
        return o;
    }
    static std::string pad(const std::string& s) { return s.size() < 28 ? s + std::string(28 - s.size(), ' ') : s + " "; }
    void add(std::vector<std::string> names, std::string help, bool flag, bool req,
             std::function<void(const std::string&)> set, std::string def) {
        Opt o;
        o.names = std::move(names);
        o.help = std::move(help);
        o.flag = flag;
        o.required = req;
        o.set = std::move(set);
        o.shown_default = std::move(def);
        opts_.push_back(std::move(o));
    }
    Opt* find(const std::string& key) {
        for (auto& o : opts_)
            for (const auto& n : o.names)
                if (n == key) return &o;
        return nullptr;
    }
    std::string name_, desc_;
    std::vector<Opt> opts_;
    std::vector<Positional> pos_;
};

// ------------------------------------------------------------------ shared helpers
struct FormatOption {
    std::string value = "text";
    bool json() const { return value == "json"; }
};

void add_format(Command& c, FormatOption& f) {
    c.opt({"--format"}, "Report format (text|json)", f.value, false, {"text", "json"});
}

struct ReconstructArgs {
    std::string input, pattern, output, raw, cache, reference;
    std::string algo = "rljsde", precision = "double";
    std::string compute = "fp32";   // (ext) device arithmetic of RL-JSDE
    std::string devices = "0";      // (ext) comma-separated CUDA devices (row bands)
    int window = 32, block = 4, iterations = 200, threads = 0, bits = 8;
    double step = 0.5, decay = 0.8, exponent = 2.0;
    bool no_clip = false;
    FormatOption format;
};

std::vector<int> parse_devices(const std::string& s) {
    std::vector<int> d;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) d.push_back(to_int("--devices", tok));
    if (d.empty()) throw UsageError("--devices: empty device list");
    return d;
}

tqsb::ReconstructionConfig to_config(const ReconstructArgs& a) {
    tqsb::ReconstructionConfig c;
    c.window = a.window;
    c.block = a.block;
    c.solver.maxIterations = a.iterations;
    c.solver.stepWidth = a.step;
    c.weighting.spatialDecay = a.decay;
    c.weighting.frequencyExponent = a.exponent;
    c.precision = a.precision == "single" ? tqsb::Precision::Single : tqsb::Precision::Double;
    c.clipOutput = !a.no_clip;
    c.algorithm = a.algo == "ljsde" ? tqsb::Algorithm::Ljsde : tqsb::Algorithm::Rljsde;
    c.threads = a.threads;
    c.compute = a.compute == "fp64" ? tqsb::Compute::Fp64 : tqsb::Compute::Fp32;
    c.devices = parse_devices(a.devices);
    return c;
}

void add_solver_options(Command& c, ReconstructArgs& a) {
    c.opt({"--window"}, "Model window size", a.window)
        .opt({"--block"}, "Target block size", a.block)
        .opt({"--iterations"}, "Iterations per block", a.iterations)
        .opt({"--step"}, "Update step width", a.step);
}

// ------------------------------------------------------------------ subcommands
int run_pattern(uint64_t seed, int period, const std::string& out) {
    const tqsb::QuadrantPattern p = tqsb::generate_pattern(seed, period);
    tqsb::write_pattern(out, p);
    std::printf("pattern: period=%d seed=%llu -> %s (%dx%d cells)\n", p.period,
                static_cast<unsigned long long>(p.seed), out.c_str(), p.cellsPerPeriod(),
                p.cellsPerPeriod());
    return kExitOk;
}

int run_simulate(const std::string& imagePath, const std::string& patternPath, const std::string& out) {
    const tqsb::Image image = tqsb::read_image_any(imagePath);
    const tqsb::QuadrantPattern pattern = tqsb::read_pattern(patternPath);
    const tqsb::MeasurementFrame frame = tqsb::simulate_measurement(image, pattern);
    tqsb::write_frame(out, frame);
    std::printf("simulate: %dx%d image -> %dx%d frame (%zu measurements) -> %s\n", image.rows,
                image.cols, frame.rows, frame.cols, frame.size(), out.c_str());
    return kExitOk;
}

void print_report(const tqsb::ReconstructionReport& r, const ReconstructArgs& a) {
    if (a.format.json()) {
        JsonObject j;
        j.str("algorithm", a.algo);
        j.integer("window", a.window);
        j.integer("block", a.block);
        j.integer("iterations", a.iterations);
        j.num("step_width", a.step);
        j.str("precision", a.precision);
        j.integer("blocks", r.blocksProcessed);
        j.num("seconds", r.seconds);
        j.num("warm_seconds", r.warmSeconds);
        j.uinteger("classes_total", r.classesTotal);
        j.uinteger("classes_interior", r.classesInterior);
        j.uinteger("classes_created", r.classesCreated);
        j.uinteger("cache_hits", r.cacheHits);
        j.uinteger("cache_misses", r.cacheMisses);
        j.integer("rows", r.output.rows);
        j.integer("cols", r.output.cols);
        if (r.psnrDb) psnr_json(j, "psnr_db", *r.psnrDb);
        std::cout << j.dump() << "\n";
        return;
    }
    std::printf("algorithm:        %s\n", a.algo.c_str());
    std::printf("window/block:     %d/%d\n", a.window, a.block);
    std::printf("iterations:       %d (step width %g)\n", a.iterations, a.step);
    std::printf("precision:        %s\n", a.precision.c_str());
    std::printf("output:           %dx%d\n", r.output.rows, r.output.cols);
    std::printf("blocks:           %ld\n", r.blocksProcessed);
    std::printf("seconds:          %.3f\n", r.seconds);
    std::printf("warm seconds:     %.3f\n", r.warmSeconds);
    std::printf("offset classes:   %zu total, %zu interior, %zu created\n", r.classesTotal,
                r.classesInterior, r.classesCreated);
    std::printf("kernel cache:     %llu hits, %llu misses\n",
                static_cast<unsigned long long>(r.cacheHits),
                static_cast<unsigned long long>(r.cacheMisses));
    if (r.psnrDb) std::printf("psnr vs ref:      %s dB\n", psnr_text(*r.psnrDb).c_str());
}

int run_reconstruct(const ReconstructArgs& a) {
    const tqsb::MeasurementFrame frame = tqsb::read_frame(a.input);
    const tqsb::QuadrantPattern pattern = tqsb::read_pattern(a.pattern);
    const tqsb::ReconstructionConfig cfg = to_config(a);
    const bool recurrent = cfg.algorithm == tqsb::Algorithm::Rljsde;

    tqsb::KernelCache cache;
    const bool useCacheFile = !a.cache.empty() && recurrent;
    bool cacheLoaded = false;
    if (useCacheFile && fs::exists(a.cache)) {
        tqsb::load_kernel_cache(a.cache, cache, pattern, cfg);
        cacheLoaded = true;
    }
    tqsb::Image reference;
    const tqsb::Image* refPtr = nullptr;
    if (!a.reference.empty()) {
        reference = tqsb::read_image_any(a.reference);
        refPtr = &reference;
    }
    const tqsb::ReconstructionReport report =
        tqsb::reconstruct(frame, pattern, cfg, recurrent ? &cache : nullptr, refPtr);
    if (useCacheFile && !cacheLoaded) tqsb::save_kernel_cache(a.cache, cache, pattern, cfg);

    tqsb::write_pgm(a.output, report.output, a.bits);
    if (!a.raw.empty()) tqsb::write_raw_image(a.raw, report.output);
    print_report(report, a);
    return kExitOk;
}

// Pixelwise difference statistics of two equally sized images (the `compare`
// subcommand's numbers; squared differences summed in pixel order).
struct DiffStats {
    double max_abs = 0.0;
    double mse = 0.0;
};

DiffStats diff_stats(const tqsb::Image& x, const tqsb::Image& y) {
    DiffStats st;
    double sq = 0.0;
    const double* px = x.values.data();
    const double* py = y.values.data();
    const size_t n = x.size();
    for (size_t i = 0; i < n; ++i) {
        const double e = std::fabs(px[i] - py[i]);
        if (e > st.max_abs) st.max_abs = e;
        sq += e * e;
    }
    st.mse = sq / static_cast<double>(n);
    return st;
}

int run_compare(const std::string& pa, const std::string& pb, const std::string& pref, double threshold,
                const FormatOption& fmt) {
    const tqsb::Image imgA = tqsb::read_image_any(pa);
    const tqsb::Image imgB = tqsb::read_image_any(pb);
    if (!imgA.same_size(imgB)) throw std::invalid_argument("compare: image dimensions differ");
    const DiffStats st = diff_stats(imgA, imgB);
    const bool ok = st.max_abs <= threshold;
    // PSNR of each input against the optional ground truth
    std::optional<std::pair<double, double>> vsRef;
    if (!pref.empty()) {
        const tqsb::Image truth = tqsb::read_image_any(pref);
        vsRef = std::make_pair(tqsb::psnr(truth, imgA), tqsb::psnr(truth, imgB));
    }
    if (fmt.json()) {
        JsonObject j;
        j.num("max_abs_diff", st.max_abs);
        j.num("mse", st.mse);
        j.num("threshold", threshold);
        j.boolean("pass", ok);
        if (vsRef) {
            psnr_json(j, "psnr_a_vs_ref", vsRef->first);
            psnr_json(j, "psnr_b_vs_ref", vsRef->second);
        }
        std::cout << j.dump() << "\n";
        return ok ? kExitOk : kExitCompareFailed;
    }
    std::printf("max abs diff:     %.3e\n", st.max_abs);
    std::printf("mse:              %.3e\n", st.mse);
    if (vsRef) {
        std::printf("psnr A vs ref:    %s dB\n", psnr_text(vsRef->first).c_str());
        std::printf("psnr B vs ref:    %s dB\n", psnr_text(vsRef->second).c_str());
    }
    std::printf("result:           %s (threshold %.3e)\n", ok ? "PASS" : "FAIL", threshold);
    return ok ? kExitOk : kExitCompareFailed;
}

// bench (pipeline.cpp:258-329 / tqs.cpp:219-285) on the device: L-JSDE (fp64) and
// RL-JSDE in its fp64 parity mode, both unclipped, must agree within the threshold;
// (ext) the RL-JSDE fp32 product path is timed alongside.
int run_bench(const std::string& dir, const ReconstructArgs& a, bool scaling, double threshold) {
    if (!fs::is_directory(dir)) throw std::invalid_argument("bench: not a directory: " + dir);
    std::vector<fs::path> paths;
    for (const auto& e : fs::directory_iterator(dir)) {
        const std::string ext = e.path().extension().string();
        if (ext == ".pgm" || ext == ".tqsm") paths.push_back(e.path());
    }
    std::sort(paths.begin(), paths.end());
    if (paths.empty()) throw std::invalid_argument("bench: no .pgm/.tqsm images in " + dir);
    std::vector<tqsb::Image> images;
    for (const auto& p : paths) images.push_back(tqsb::read_image_any(p.string()));
    const tqsb::QuadrantPattern pattern = tqsb::read_pattern(a.pattern);

    tqsb::ReconstructionConfig cfgL = to_config(a);
    cfgL.algorithm = tqsb::Algorithm::Ljsde;
    cfgL.threads = 1;
    cfgL.clipOutput = false;
    tqsb::ReconstructionConfig cfgR = cfgL;
    cfgR.algorithm = tqsb::Algorithm::Rljsde;
    cfgR.compute = tqsb::Compute::Fp64;
    tqsb::ReconstructionConfig cfgF = cfgR;
    cfgF.compute = tqsb::Compute::Fp32;

    tqsb::KernelCache cacheR, cacheF;
    double sumL = 0, sumR = 0, sumWarm = 0, sumF = 0, maxDiff = 0;
    for (const tqsb::Image& img : images) {
        const tqsb::MeasurementFrame frame =
            tqsb::simulate_measurement(tqsb::pad_to_block_multiple(img, cfgL.block).image, pattern);
        const tqsb::ReconstructionReport rl = tqsb::reconstruct(frame, pattern, cfgL);
        const tqsb::ReconstructionReport rr = tqsb::reconstruct(frame, pattern, cfgR, &cacheR);
        const tqsb::ReconstructionReport rf = tqsb::reconstruct(frame, pattern, cfgF, &cacheF);
        sumL += rl.seconds;
        sumR += rr.seconds;
        sumWarm += rr.warmSeconds;
        sumF += rf.seconds;
        for (size_t i = 0; i < rl.output.size(); ++i)
            maxDiff = std::max(maxDiff, std::abs(rl.output.values[i] - rr.output.values[i]));
    }
    const double n = double(images.size());
    const double meanL = sumL / n, meanR = sumR / n, meanWarm = sumWarm / n;
    const double inf = std::numeric_limits<double>::infinity();
    const double speedup = meanR > 0 ? meanL / meanR : inf;
    const double speedupWarm = meanR + meanWarm > 0 ? meanL / (meanR + meanWarm) : inf;
    if (maxDiff > threshold)
        throw EquivalenceError("algorithms diverged: max abs difference " + std::to_string(maxDiff) +
                               " exceeds " + std::to_string(threshold));

    double lSmall = 0, lLarge = 0, rSmall = 0, rLarge = 0;
    if (scaling) {
        const tqsb::MeasurementFrame frame =
            tqsb::simulate_measurement(tqsb::pad_to_block_multiple(images.front(), cfgL.block).image, pattern);
        auto perBlock = [&](tqsb::Algorithm algo, int window) {
            tqsb::ReconstructionConfig c = algo == tqsb::Algorithm::Ljsde ? cfgL : cfgR;
            c.window = window;
            const tqsb::ReconstructionReport r = tqsb::reconstruct(frame, pattern, c);
            return r.seconds / double(r.blocksProcessed);
        };
        lSmall = perBlock(tqsb::Algorithm::Ljsde, 16);
        lLarge = perBlock(tqsb::Algorithm::Ljsde, a.window);
        rSmall = perBlock(tqsb::Algorithm::Rljsde, 16);
        rLarge = perBlock(tqsb::Algorithm::Rljsde, a.window);
    }
    if (a.format.json()) {
        JsonObject j;
        j.integer("images", int(images.size()));
        j.num("ljsde_mean_seconds", meanL);
        j.num("rljsde_mean_seconds", meanR);
        j.num("rljsde_mean_warm_seconds", meanWarm);
        j.num("rljsde_fp32_mean_seconds", sumF / n);
        j.num("speedup", speedup);
        j.num("speedup_incl_warm", speedupWarm);
        j.num("max_abs_difference", maxDiff);
        if (scaling) {
            j.num("ljsde_per_block_w16", lSmall);
            j.num("ljsde_per_block_large", lLarge);
            j.num("rljsde_per_block_w16", rSmall);
            j.num("rljsde_per_block_large", rLarge);
            j.num("ljsde_scaling_ratio", lLarge / lSmall);
            j.num("rljsde_scaling_ratio", rLarge / rSmall);
        }
        std::cout << j.dump() << "\n";
    } else {
        std::printf("images:                 %d\n", int(images.size()));
        std::printf("ljsde mean seconds:     %.3f\n", meanL);
        std::printf("rljsde mean seconds:    %.3f (+%.3f warm)\n", meanR, meanWarm);
        std::printf("rljsde fp32 seconds:    %.3f\n", sumF / n);
        std::printf("speedup:                %.2fx (%.2fx incl. warm)\n", speedup, speedupWarm);
        std::printf("max abs difference:     %.3e\n", maxDiff);
        if (scaling) {
            std::printf("ljsde per-block:        %.3e s (W=16)  %.3e s (W=%d)  ratio %.2f\n", lSmall, lLarge,
                        a.window, lLarge / lSmall);
            std::printf("rljsde per-block:       %.3e s (W=16)  %.3e s (W=%d)  ratio %.2f\n", rSmall, rLarge,
                        a.window, rLarge / rSmall);
        }
    }
    return kExitOk;
}

int run_kernel_report(int classes, int window, const std::string& precision, int local,
                      const FormatOption& fmt) {
    const tqsb::MemoryReport r = tqsb::kernel_memory_report(
        classes, window, precision == "double" ? tqsb::Precision::Double : tqsb::Precision::Single, local);
    if (fmt.json()) {
        JsonObject j;
        j.integer("classes", classes);
        j.integer("window", window);
        j.str("precision", precision);
        j.uinteger("b_bytes", r.bBytes);
        j.uinteger("c_bytes", r.cBytes);
        j.uinteger("d_bytes", r.dBytes);
        j.uinteger("total_bytes", r.totalBytes);
        j.num("b_mb", r.bMegabytes());
        j.num("c_mb", r.cMegabytes());
        j.num("d_mb", r.dMegabytes());
        j.num("total_mb", r.totalMegabytes());
        std::cout << j.dump() << "\n";
    } else {
        std::printf("classes:    %d\n", classes);
        std::printf("window:     %d\n", window);
        std::printf("precision:  %s\n", precision.c_str());
        std::printf("B:          %12.6f MB  (%llu bytes)\n", r.bMegabytes(), (unsigned long long)r.bBytes);
        std::printf("C:          %12.6f MB  (%llu bytes)\n", r.cMegabytes(), (unsigned long long)r.cBytes);
        std::printf("D:          %12.6f MB  (%llu bytes)\n", r.dMegabytes(), (unsigned long long)r.dBytes);
        std::printf("total:      %12.6f MB  (%llu bytes)\n", r.totalMegabytes(),
                    (unsigned long long)r.totalBytes);
    }
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    // pattern
    uint64_t seed = 1;
    int period = 32;
    std::string patternOut;
    Command cPattern("pattern", "Generate a sampling pattern file");
    cPattern.opt({"--seed"}, "Random seed", seed)
        .opt({"--period"}, "Repetition period in pixels", period)
        .opt({"-o", "--output"}, "Output pattern file", patternOut, true);
    // simulate
    std::string simImage, simPattern, simOut;
    Command cSimulate("simulate", "Simulate sensor measurements");
    cSimulate.opt({"--image"}, "Input image (.pgm or .tqsm)", simImage, true)
        .opt({"--pattern"}, "Pattern file", simPattern, true)
        .opt({"-o", "--output"}, "Output measurement file", simOut, true);
    // reconstruct
    ReconstructArgs rec;
    Command cRec("reconstruct", "Reconstruct an image");
    cRec.opt({"--input"}, "Measurement file", rec.input, true)
        .opt({"--pattern"}, "Pattern file", rec.pattern, true)
        .opt({"-o", "--output"}, "Output image (.pgm)", rec.output, true)
        .opt({"--raw"}, "Full-precision output dump (.tqsm)", rec.raw)
        .opt({"--algo"}, "Algorithm", rec.algo, false, {"ljsde", "rljsde"});
    add_solver_options(cRec, rec);
    cRec.opt({"--spatial-decay"}, "Spatial weight decay", rec.decay)
        .opt({"--frequency-exponent"}, "Frequency weight exponent", rec.exponent)
        .opt({"--precision"}, "Kernel storage precision", rec.precision, false, {"single", "double"})
        .opt({"--threads"}, "Worker threads (0 = all cores; accepted, the work runs on the GPU)", rec.threads)
        .opt({"--bits"}, "Output bit depth (8|16)", rec.bits)
        .flag({"--no-clip"}, "Skip clipping output to [0,1]", rec.no_clip)
        .opt({"--kernel-cache"}, "Kernel cache file (.tqsk), loaded if present, else written", rec.cache)
        .opt({"--reference"}, "Reference image for PSNR", rec.reference)
        .opt({"--compute"}, "(ext) RL-JSDE device arithmetic", rec.compute, false, {"fp32", "fp64"})
        .opt({"--devices"}, "(ext) CUDA devices, comma-separated (row bands)", rec.devices);
    add_format(cRec, rec.format);
    // compare
    std::string cmpA, cmpB, cmpRef;
    double cmpThreshold = 1e-6;
    FormatOption cmpFormat;
    Command cCompare("compare", "Compare two images");
    cCompare.positional("a", "First image", cmpA)
        .positional("b", "Second image", cmpB)
        .opt({"--reference"}, "Reference image for PSNR", cmpRef)
        .opt({"--threshold"}, "Max abs difference for exit 0", cmpThreshold);
    add_format(cCompare, cmpFormat);
    // bench
    ReconstructArgs ben;
    std::string benchDir;
    bool benchScaling = false;
    double benchThreshold = 1e-6;
    Command cBench("bench", "Benchmark both algorithms on an image set");
    cBench.opt({"--images"}, "Directory of .pgm/.tqsm images", benchDir, true)
        .opt({"--pattern"}, "Pattern file", ben.pattern, true);
    add_solver_options(cBench, ben);
    cBench.opt({"--threshold"}, "Equivalence threshold", benchThreshold)
        .flag({"--scaling"}, "Also measure per-block window scaling", benchScaling)
        .opt({"--devices"}, "(ext) CUDA devices, comma-separated", ben.devices);
    add_format(cBench, ben.format);
    // kernel-report
    int krClasses = 64, krWindow = 32, krLocal = -1;
    std::string krPrecision = "single";
    FormatOption krFormat;
    Command cKr("kernel-report", "Kernel memory accounting");
    cKr.opt({"--classes"}, "Offset class count", krClasses)
        .opt({"--window"}, "Model window size", krWindow)
        .opt({"--precision"}, "Storage precision", krPrecision, false, {"single", "double"})
        .opt({"--local"}, "Local measurement count (-1 = interior default)", krLocal);
    add_format(cKr, krFormat);

    std::vector<Command*> cmds{&cPattern, &cSimulate, &cRec, &cCompare, &cBench, &cKr};
    auto top_help = [&] {
        std::string h = "three-quarter sampling reconstruction toolbox (B200)\nUsage: tqsb [OPTIONS] SUBCOMMAND\n\n"
                        "Options:\n  -h,--help                   Print this help message and exit\n\nSubcommands:\n";
        for (auto* c : cmds) h += "  " + c->name() + std::string(15 - c->name().size(), ' ') + c->desc() + "\n";
        return h;
    };
    const std::vector<std::string> args(argv + 1, argv + argc);
    Command* cmd = nullptr;
    try {
        if (args.empty()) throw UsageError("A subcommand is required");
        if (args[0] == "--help" || args[0] == "-h") {
            std::cout << top_help();
            return kExitOk;
        }
        for (auto* c : cmds)
            if (c->name() == args[0]) cmd = c;
        if (!cmd) throw UsageError("The following arguments were not expected: " + args[0]);
        cmd->parse(std::vector<std::string>(args.begin() + 1, args.end()));
        if (cmd == &cRec && rec.bits != 8 && rec.bits != 16)
            throw UsageError("--bits: " + std::to_string(rec.bits) + " not in {8,16}");
    } catch (const HelpRequest&) {
        std::cout << cmd->help();
        return kExitOk;
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return kExitUsage;
    }

    try {
        if (cmd == &cPattern) return run_pattern(seed, period, patternOut);
        if (cmd == &cSimulate) return run_simulate(simImage, simPattern, simOut);
        if (cmd == &cRec) return run_reconstruct(rec);
        if (cmd == &cCompare) return run_compare(cmpA, cmpB, cmpRef, cmpThreshold, cmpFormat);
        if (cmd == &cBench) return run_bench(benchDir, ben, benchScaling, benchThreshold);
        if (cmd == &cKr) return run_kernel_report(krClasses, krWindow, krPrecision, krLocal, krFormat);
    } catch (const EquivalenceError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitCompareFailed;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    }
    return kExitUsage;
}
