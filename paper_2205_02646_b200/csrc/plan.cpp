// plan.cpp -- host side of libtqsb: the C ABI (include/tqsb/tqsb.h), validation,
// block enumeration and class census, the device-resident table store (the
// KernelCache analogue) and multi-device row-band dispatch.
//
// Reference correspondences (/root/reference/proj/...):
//   validate             src/pipeline.cpp:27-42 (+ frame checks 66-67, 74-75)
//   enumerate_blocks     src/pipeline.cpp:84-106, offset_class src/rljsde.cpp:12-17
//   local_system         src/grid.cpp:31-42, 70-102; spatial_weight src/basis.cpp:75-80
//   frequency weights    src/basis.cpp:90-106; unit table src/basis.cpp:15-26
//   table store / warm   include/tqs/rljsde.hpp:81-100, src/pipeline.cpp:110-133
//   report counters      src/pipeline.cpp:168-184; psnr src/pipeline.cpp:221-233
// The per-block solve, synthesis and placement run on the device (solve_f32.cu,
// solve_f64.cu); the tables are built on the device (tables.cu). There is no CPU
// fallback: without a CUDA device every compute entry point fails with TQSB_ENODEV.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <tuple>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tqsb/tqsb.h"
#include "tqsb_internal.hpp"

using namespace tqsb;

namespace {

thread_local std::string g_error;

int set_error(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return set_error(_e == cudaErrorMemoryAllocation ? TQSB_ENOMEM : TQSB_ECUDA,       \
                             std::string(#expr) + ": " + cudaGetErrorString(_e));             \
    } while (0)

// in functions that report through BandResult (void): record the failure and return
#define CUDA_TRY_V(expr)                                                                       \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return fail(set_error(_e == cudaErrorMemoryAllocation ? TQSB_ENOMEM : TQSB_ECUDA,  \
                                  std::string(#expr) + ": " + cudaGetErrorString(_e)));       \
    } while (0)

#define TQSB_TRY(expr)            \
    do {                          \
        int _rc = (expr);         \
        if (_rc != TQSB_OK) return _rc; \
    } while (0)

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// validation: the reference's messages, pipeline.cpp:27-42
// ---------------------------------------------------------------------------
int validate(const tqsb_config& c, int period) {
    if (c.window < 2 || c.window % 2 != 0)
        return set_error(TQSB_EINVAL, "window size must be even and >= 2");
    if (c.block < 1 || c.window % c.block != 0)
        return set_error(TQSB_EINVAL, "block size must divide the window size");
    if ((c.window - c.block) % 2 != 0)
        return set_error(TQSB_EINVAL, "window/block sizes must center the target block");
    if (period <= 0 || period % c.block != 0)
        return set_error(TQSB_EINVAL, "block size must divide the pattern period");
    if (c.max_iterations < 0) return set_error(TQSB_EINVAL, "iteration count must be non-negative");
    if (!(c.step_width > 0.0 && c.step_width <= 1.0))
        return set_error(TQSB_EINVAL, "step width must lie in (0,1]");
    if (c.threads < 0) return set_error(TQSB_EINVAL, "thread count must be non-negative");
    if (c.compute != TQSB_COMPUTE_FP32 && c.compute != TQSB_COMPUTE_FP64)
        return set_error(TQSB_EINVAL, "unknown compute mode");
    if (c.precision != TQSB_PRECISION_SINGLE && c.precision != TQSB_PRECISION_DOUBLE)
        return set_error(TQSB_EINVAL, "unknown precision");
    if (c.algorithm != TQSB_ALGO_LJSDE && c.algorithm != TQSB_ALGO_RLJSDE)
        return set_error(TQSB_EINVAL, "unknown algorithm");
    return TQSB_OK;
}

// the fp32 product kernel serves the call (else the fp64 kernel: compute=fp64, or a
// configuration outside the fp32 kernel's instantiations -- W > 32, where it holds a
// window row per warp, or B > 16, beyond its 8 kept pixels per lane -- which the
// reference accepts and the fp64 kernel runs on the reference's exact greedy paths)
bool uses_f32(const tqsb_config& c) {
    return c.algorithm == TQSB_ALGO_RLJSDE && c.compute == TQSB_COMPUTE_FP32 &&
           c.window <= kMaxWindowF32 && c.block * c.block <= 256;
}

// the fp64 RL-JSDE kernel on Precision::Single planes, like the reference's float
// KernelPlanes (the fp32 product builds its own tables; L-JSDE uses no planes there)
int round_single(const tqsb_config& c) {
    return c.precision == TQSB_PRECISION_SINGLE && c.algorithm == TQSB_ALGO_RLJSDE && !uses_f32(c);
}

struct Geometry {
    int M, N, padM, padN, lead, B, W;
};

int geometry(const tqsb_config& c, int frame_rows, int frame_cols, Geometry* g) {
    if (frame_rows < 1 || frame_cols < 1) return set_error(TQSB_EINVAL, "empty measurement frame");
    g->W = c.window;
    g->B = c.block;
    g->M = 2 * frame_rows;
    g->N = 2 * frame_cols;
    const int step = std::lcm(c.block, 2);
    g->padM = round_up(g->M, step);
    g->padN = round_up(g->N, step);
    if (g->padM < c.window || g->padN < c.window)
        return set_error(TQSB_EINVAL, "image is smaller than the model window");
    g->lead = (c.window - c.block) / 2;
    return TQSB_OK;
}

// ---------------------------------------------------------------------------
// block enumeration (pipeline.cpp:84-106)
// ---------------------------------------------------------------------------
struct Enumerated {
    std::vector<Task> tasks;          // row-major order
    std::vector<int> keys;            // class key per task (row*P + col)
    std::vector<int> class_order;     // distinct keys in first-seen order
    std::map<int, std::pair<int, int>> representative;
    long long classes_total = 0, classes_interior = 0;
};

void enumerate(const Geometry& g, int period, int br_begin, int br_end, Enumerated* e) {
    std::vector<char> seen(size_t(period) * period, 0), seen_int(size_t(period) * period, 0);
    for (int bri = br_begin; bri < br_end; ++bri) {
        const int br = bri * g.B;
        for (int bc = 0; bc + g.B <= g.padN; bc += g.B) {
            const int wr = br - g.lead, wc = bc - g.lead;
            const int orow = std::clamp(wr, 0, g.padM - g.W), ocol = std::clamp(wc, 0, g.padN - g.W);
            const bool interior = orow == wr && ocol == wc;
            const int key = (orow % period) * period + (ocol % period);
            if (!seen[key]) {
                seen[key] = 1;
                ++e->classes_total;
                e->class_order.push_back(key);
                e->representative.emplace(key, std::make_pair(orow, ocol));
            }
            if (interior && !seen_int[key]) {
                seen_int[key] = 1;
                ++e->classes_interior;
            }
            e->tasks.push_back(Task{br, bc, orow, ocol});
            e->keys.push_back(key);
        }
    }
}

// ---------------------------------------------------------------------------
// local measurement system of a window (grid.cpp:31-42, 70-102) and weights
// ---------------------------------------------------------------------------
struct LocalSystem {
    int L = 0;
    std::vector<short> px;         // L*6
    std::vector<double> w;         // L
    std::vector<float> mask32;     // W*W
};

LocalSystem local_system(const std::vector<uint8_t>& opaque, int period, int orow, int ocol,
                         const tqsb_config& c) {
    LocalSystem s;
    const int W = c.window, pc = period / 2;
    const int r0 = (orow + 1) / 2, r1 = (orow + W - 2) / 2;
    const int c0 = (ocol + 1) / 2, c1 = (ocol + W - 2) / 2;
    s.mask32.assign(size_t(W) * W, 0.f);
    const double center = (W - 1) / 2.0;
    for (int r = r0; r <= r1; ++r)
        for (int cc = c0; cc <= c1; ++cc) {
            const int ce = 2 * r - orow, cg = 2 * cc - ocol;
            const int q = opaque[size_t(((r % pc) + pc) % pc) * pc + ((cc % pc) + pc) % pc];
            const double dr = (ce + 0.5) - center, dc = (cg + 0.5) - center;
            const double w = std::pow(c.spatial_decay, std::sqrt(dr * dr + dc * dc));
            s.w.push_back(w);
            for (int quad = 0; quad < 4; ++quad) {  // transparent quadrants, row-major
                if (quad == q) continue;
                const int eta = ce + quad / 2, gam = cg + quad % 2;
                s.px.push_back(static_cast<short>(eta));
                s.px.push_back(static_cast<short>(gam));
                s.mask32[size_t(eta) * W + gam] = float(w * (1.0 / 3.0));
            }
            ++s.L;
        }
    return s;
}

// ---------------------------------------------------------------------------
// window constants: unit table, q, rank permutation
// ---------------------------------------------------------------------------
struct WindowTables {
    int W = 0, K = 0, NS = 0, K_pad = 0;
    std::vector<double> unit64;  // 2W
    std::vector<float> unit32;   // 2W
    std::vector<int> perm, src;  // K_pad
};

// frequency_weights (basis.cpp:90-106): q_k = (1 - |centred k| / (sqrt2 (W/2)(1+1e-6)))^p
std::vector<double> frequency_weights(int W, double exponent) {
    std::vector<double> q(size_t(W) * W);
    const int half = W / 2;
    for (int s = 0; s < W; ++s)
        for (int r = 0; r < W; ++r) {
            const int cs = s <= half ? s : W - s, cr = r <= half ? r : W - r;
            const double radius = std::sqrt(double(cs) * cs + double(cr) * cr);
            const double maxr = 1.41421356237309504880 * half * (1.0 + 1e-6);
            q[size_t(s) * W + r] = std::pow(1.0 - radius / maxr, exponent);
        }
    return q;
}

WindowTables window_tables(const tqsb_config& c) {
    WindowTables t;
    const int W = c.window;
    t.W = W;
    t.K = W * W;
    const int ns = (t.K + 63) / 64;
    // fp32 register slots per lane (power of two, W <= 32); above that the rank tables
    // only need to cover K (the fp64 kernel does not use them)
    t.NS = ns <= 1 ? 1 : ns <= 2 ? 2 : ns <= 4 ? 4 : ns <= 8 ? 8 : ns <= 16 ? 16 : ns;
    t.K_pad = 64 * t.NS;
    t.unit64.assign(2 * W, 0.0);
    t.unit64[0] = 1.0;
    t.unit64[2 * (W / 2)] = -1.0;
    for (int k = 1; k < W / 2; ++k) {  // FourierTable (basis.cpp:15-26)
        const double a = 2.0 * 3.14159265358979323846 * k / W;
        t.unit64[2 * k] = std::cos(a);
        t.unit64[2 * k + 1] = std::sin(a);
        t.unit64[2 * (W - k)] = t.unit64[2 * k];
        t.unit64[2 * (W - k) + 1] = -t.unit64[2 * k + 1];
    }
    t.unit32.resize(2 * W);
    for (int i = 0; i < 2 * W; ++i) t.unit32[i] = float(t.unit64[i]);
    const int half = W / 2;
    // Rank order: by centred radius (hot first), conjugate pairs k / -k on adjacent
    // ranks 2j (smaller flat k) and 2j+1, i.e. the two halves of one lane's slot, so
    // the packed selection key resolves their bitwise ties to the smaller flat k like
    // the reference's strict '>' scan (rljsde.cpp:147-156). The four self-conjugate
    // frequencies pair among themselves: DC with (W/2, W/2) on ranks 0/1, (0, W/2)
    // with (W/2, 0) at their radius.
    std::vector<std::tuple<int, int, int>> order;  // (group radius^2, pair id, k)
    for (int s = 0; s < W; ++s)
        for (int r = 0; r < W; ++r) {
            const int cs = s <= half ? s : W - s, cr = r <= half ? r : W - r;
            const int k = s * W + r, kc = ((W - s) % W) * W + (W - r) % W;
            int grp = cs * cs + cr * cr, pid = std::min(k, kc);
            if (k == kc && cs == half && cr == half) grp = 0, pid = 0;  // (W/2, W/2) next to DC
            order.emplace_back(grp, pid, k);
        }
    std::sort(order.begin(), order.end());
    t.perm.assign(t.K_pad, -1);
    t.src.assign(t.K_pad, 0);
    for (int r = 0; r < t.K; ++r) {
        const int k = std::get<2>(order[r]), s = k / W, rho = k % W;
        t.perm[r] = k;
        // half-spectrum source: rows sigma <= W/2, with the self-conjugate rows
        // 0 and W/2 taking rho > W/2 from their mirror
        const bool direct = s < half || ((s == 0 || s == half) && rho <= half);
        if (direct)
            t.src[r] = s * W + rho;
        else
            t.src[r] = (((W - s) % W) * W + (W - rho) % W) | (1 << 30);
    }
    return t;
}

// ---------------------------------------------------------------------------
// per-device state
// ---------------------------------------------------------------------------
struct ClassSlab {
    void* base = nullptr;
    size_t bytes = 0;
};

struct WorkKey {
    int rows, cols, br0, br1, block, chunk, stream;
    bool operator<(const WorkKey& o) const {
        return std::tie(rows, cols, br0, br1, block, chunk, stream) <
               std::tie(o.rows, o.cols, o.br0, o.br1, o.block, o.chunk, o.stream);
    }
};

struct Work {
    Task* d_tasks = nullptr;
    WorkItem* d_items = nullptr;
    int* d_task_cls = nullptr;       // class slot per (class-sorted) task
    int n_tasks = 0, n_items = 0;
    int frame_row0 = 0, frame_row1 = 0;  // frame rows the band needs
    std::vector<int> keys;                // classes used
    long long classes_total = 0, classes_interior = 0;
    // streamed completion (stream > 0 chunks): tasks ordered chunk by chunk (class-sorted
    // within a chunk); chunk s holds chunk_count[s] blocks covering block rows
    // [chunk_br[s], chunk_br[s+1])
    std::vector<int> chunk_count, chunk_br;
    std::vector<int> chunk_fr_hi;  // frame rows [frame_row0, chunk_fr_hi[s]) cover chunk s
};
constexpr int kStreamChunks = 16;       // output chunks of a streamed host-buffer call (max)
constexpr int kStreamMinTasks = 8192;   // below this a frame is not worth streaming
constexpr int kStreamMinTasksPinned = 262144;  // ... into a pinned caller buffer

// The per-call derived tables of one option set. The cache proper is the fp64 planes
// (B, C, D per offset class: the reference's KernelSet, rljsde.hpp:34-52), which
// depend only on the pattern, the window and the spatial weights. The frequency
// weights q (frequency exponent) and, for the fp32 product kernel, the scaled tables
// s = sqrt(q/D), C' = s C and fac = gamma/(s D) depend on per-call options
// (pipeline.cpp:108, 143-155), so they are derived from the planes lazily per
// (exponent, gamma) -- k_scale + k_pack32, ~8 us per class -- and kept for reuse.
struct Derived {
    double exponent = 0.0, step = 0.0;  // step is 0 for fp64 sets (gamma is a kernel argument)
    bool f32 = false;
    double* d_q64 = nullptr;           // K frequency weights
    std::vector<ClassSlab> slabs;      // per class slot: cpack, scale, fac (fp32 sets)
    std::vector<ClassTab> tabs;        // per class slot: the planes + this set's tables
    ClassTab* d_tabs = nullptr;
    size_t d_tabs_cap = 0;
    uint64_t last_use = 0;
};
constexpr size_t kMaxDerived = 4;     // option sets kept per device (LRU beyond)
constexpr int kCounterRing = 64;      // per-launch task-queue heads (see launch())

struct Device {
    int id = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;            // solve
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // copy engines
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_h2d[4] = {}, ev_comp[4] = {};
    int* d_perm = nullptr;
    int* d_src = nullptr;
    float* d_unit32 = nullptr;
    double* d_unit64 = nullptr;
    uint8_t* d_opaque = nullptr;   // the pattern's (P/2)^2 quadrant indices (device readout)
    int* d_progress = nullptr;     // blocks finished per chunk of a streamed call (device)
    cudaEvent_t ev_chunk[64] = {}; // chunk s copied to the pinned staging
    int* d_counters = nullptr;     // kCounterRing dynamic task-queue heads
    unsigned counter_next = 0;
    std::map<int, int> slot_of;    // class key -> slot
    std::vector<ClassTab> tabs;    // host mirror of the planes per slot (derived fields null)
    std::vector<ClassSlab> slabs;
    std::vector<std::unique_ptr<Derived>> derived;
    uint64_t use_clock = 0;
    std::map<WorkKey, Work> works;
    double* d_frame = nullptr;
    size_t frame_cap = 0;
    double* d_out = nullptr;
    size_t out_cap = 0;
    double* h_in = nullptr;   // pinned staging
    size_t h_in_cap = 0;
    double* h_out = nullptr;
    size_t h_out_cap = 0;
    // multi-frame pipeline (tqsb_reconstruct_batch): double-buffered frames/staging
    double* d_fs[2] = {};
    size_t fs_cap[2] = {};
    double* h_in_s[2] = {};
    size_t h_in_s_cap[2] = {};
    double* h_out_s[2] = {};
    size_t h_out_s_cap[2] = {};
    size_t table_bytes = 0;
};

} // namespace

struct tqsb_plan {
    tqsb_config cfg;
    int period = 0;
    std::vector<uint8_t> opaque;
    WindowTables wt;
    std::vector<std::unique_ptr<Device>> devs;
    std::mutex mu;
};

namespace {

int device_init(tqsb_plan* p, Device* d) {
    CUDA_TRY(cudaSetDevice(d->id));
    CUDA_TRY(cudaDeviceGetAttribute(&d->num_sms, cudaDevAttrMultiProcessorCount, d->id));
    CUDA_TRY(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreate(&d->ev0));
    CUDA_TRY(cudaEventCreate(&d->ev1));
    CUDA_TRY(cudaStreamCreateWithFlags(&d->s_h2d, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&d->s_d2h, cudaStreamNonBlocking));
    for (int k = 0; k < 4; ++k) {
        CUDA_TRY(cudaEventCreateWithFlags(&d->ev_h2d[k], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&d->ev_comp[k], cudaEventDisableTiming));
    }
    const WindowTables& t = p->wt;
    CUDA_TRY(cudaMalloc(&d->d_perm, sizeof(int) * t.K_pad));
    CUDA_TRY(cudaMalloc(&d->d_src, sizeof(int) * t.K_pad));
    CUDA_TRY(cudaMalloc(&d->d_unit32, sizeof(float) * 2 * t.W));
    CUDA_TRY(cudaMalloc(&d->d_unit64, sizeof(double) * 2 * t.W));
    CUDA_TRY(cudaMalloc(&d->d_opaque, p->opaque.size()));
    CUDA_TRY(cudaMalloc(&d->d_counters, sizeof(int) * kCounterRing));
    CUDA_TRY(cudaMemcpy(d->d_opaque, p->opaque.data(), p->opaque.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d->d_perm, t.perm.data(), sizeof(int) * t.K_pad, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d->d_src, t.src.data(), sizeof(int) * t.K_pad, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d->d_unit32, t.unit32.data(), sizeof(float) * 2 * t.W, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d->d_unit64, t.unit64.data(), sizeof(double) * 2 * t.W, cudaMemcpyHostToDevice));
    return TQSB_OK;
}

void derived_free(Derived* v) {
    for (auto& s : v->slabs) cudaFree(s.base);
    cudaFree(v->d_tabs);
    cudaFree(v->d_q64);
}

void device_free(Device* d) {
    if (!d) return;
    cudaSetDevice(d->id);
    for (auto& s : d->slabs) cudaFree(s.base);
    for (auto& v : d->derived) derived_free(v.get());
    for (auto& kv : d->works) {
        cudaFree(kv.second.d_tasks);
        cudaFree(kv.second.d_items);
        cudaFree(kv.second.d_task_cls);
    }
    cudaFree(d->d_perm);
    cudaFree(d->d_src);
    cudaFree(d->d_unit32);
    cudaFree(d->d_unit64);
    cudaFree(d->d_opaque);
    cudaFree(d->d_counters);
    cudaFree(d->d_progress);
    for (auto& e : d->ev_chunk)
        if (e) cudaEventDestroy(e);
    cudaFree(d->d_frame);
    cudaFree(d->d_out);
    if (d->h_in) cudaFreeHost(d->h_in);
    if (d->h_out) cudaFreeHost(d->h_out);
    for (int k = 0; k < 2; ++k) {
        cudaFree(d->d_fs[k]);
        if (d->h_in_s[k]) cudaFreeHost(d->h_in_s[k]);
        if (d->h_out_s[k]) cudaFreeHost(d->h_out_s[k]);
    }
    if (d->ev0) cudaEventDestroy(d->ev0);
    if (d->ev1) cudaEventDestroy(d->ev1);
    for (int k = 0; k < 4; ++k) {
        if (d->ev_h2d[k]) cudaEventDestroy(d->ev_h2d[k]);
        if (d->ev_comp[k]) cudaEventDestroy(d->ev_comp[k]);
    }
    if (d->s_h2d) cudaStreamDestroy(d->s_h2d);
    if (d->s_d2h) cudaStreamDestroy(d->s_d2h);
    if (d->stream) cudaStreamDestroy(d->stream);
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// memcpy of large host buffers (pageable <-> pinned staging) on up to max_threads threads
void par_memcpy(void* dst, const void* src, size_t bytes, unsigned max_threads = 16) {
    const size_t kPerThread = size_t(1) << 20;  // at least 1 MB per thread
    unsigned nt = std::min<unsigned>(max_threads, std::max(1u, std::thread::hardware_concurrency()));
    nt = unsigned(std::min<size_t>(nt, bytes / kPerThread));
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    const size_t chunk = (bytes + nt - 1) / nt;
    for (unsigned i = 0; i < nt; ++i) {
        const size_t off = i * chunk;
        if (off >= bytes) break;
        const size_t n = std::min(chunk, bytes - off);
        th.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, n);
        });
    }
    for (auto& t : th) t.join();
}

// Allocate the device slab of one class's fp64 planes (and its local system) on
// device d, upload the local system and register it under `key`; cb receives the
// build descriptor. The spatial weights come from the config of the call that
// creates the class, like the reference's make_kernels (pipeline.cpp:114-121).
int alloc_class(tqsb_plan* p, Device* d, const tqsb_config& c, int key, int orow, int ocol,
                ClassBuild* cb) {
    const WindowTables& t = p->wt;
    const size_t K = t.K, W = t.W;
    LocalSystem ls = local_system(p->opaque, p->period, orow, ocol, c);
    const size_t L = ls.L;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const size_t o_c64 = take(K * K * 2 * 8), o_b64 = take(K * L * 2 * 8),
                 o_t64 = take(K * L * 2 * 8), o_d64 = take(K * 8), o_mask = take(W * W * 4),
                 o_px = take(L * 12 + 8), o_w = take(L * 8 + 8);
    ClassSlab slab;
    slab.bytes = off;
    CUDA_TRY(cudaMalloc(&slab.base, slab.bytes));
    char* b = static_cast<char*>(slab.base);
    CUDA_TRY(cudaMemcpyAsync(b + o_px, ls.px.data(), L * 12, cudaMemcpyHostToDevice, d->stream));
    CUDA_TRY(cudaMemcpyAsync(b + o_w, ls.w.data(), L * 8, cudaMemcpyHostToDevice, d->stream));
    CUDA_TRY(cudaMemcpyAsync(b + o_mask, ls.mask32.data(), W * W * 4, cudaMemcpyHostToDevice,
                             d->stream));
    CUDA_TRY(cudaStreamSynchronize(d->stream));  // host vectors die at scope end
    *cb = ClassBuild{};
    cb->local = int(L);
    cb->px = reinterpret_cast<const short*>(b + o_px);
    cb->w = reinterpret_cast<const double*>(b + o_w);
    cb->t64 = reinterpret_cast<double*>(b + o_t64);
    cb->b64 = reinterpret_cast<double*>(b + o_b64);
    cb->c64 = reinterpret_cast<double*>(b + o_c64);
    cb->d64 = reinterpret_cast<double*>(b + o_d64);
    ClassTab tab{};
    tab.mask32 = reinterpret_cast<const float*>(b + o_mask);
    tab.b64 = cb->b64;
    tab.c64 = cb->c64;
    tab.d64 = cb->d64;
    tab.cells = nullptr;
    tab.w64 = cb->w;
    tab.bt64 = cb->t64;  // B transposed, written over the T scratch after the build
    tab.local = int(L);
    d->slot_of[key] = int(d->tabs.size());
    d->tabs.push_back(tab);
    d->slabs.push_back(slab);
    d->table_bytes += slab.bytes;
    return TQSB_OK;
}

// Build the fp64 planes of every class in `keys` that is not resident on device d
// (batched; the serial warm pass of pipeline.cpp:127-133). Returns the number of
// classes created through *created.
int ensure_classes(tqsb_plan* p, Device* d, const tqsb_config& c, const std::vector<int>& keys,
                   const std::map<int, std::pair<int, int>>& rep, int* created, int* launches) {
    std::vector<int> missing;
    for (int k : keys)
        if (!d->slot_of.count(k)) missing.push_back(k);
    *created = int(missing.size());
    if (missing.empty()) return TQSB_OK;
    CUDA_TRY(cudaSetDevice(d->id));
    std::vector<ClassBuild> descs;
    int max_local = 1;
    for (int key : missing) {
        const auto [orow, ocol] = rep.at(key);
        ClassBuild cb;
        TQSB_TRY(alloc_class(p, d, c, key, orow, ocol, &cb));
        max_local = std::max(max_local, cb.local);
        descs.push_back(cb);
    }
    int rc = launch_tables_build(descs.data(), int(descs.size()), p->wt.W, d->d_unit64, max_local,
                                 d->stream, launches, round_single(c));
    if (rc != 0) return set_error(TQSB_ECUDA, std::string("table build: ") +
                                                  cudaGetErrorString(cudaError_t(rc)));
    CUDA_TRY(cudaStreamSynchronize(d->stream));
    return TQSB_OK;
}

// The derived tables of the call's options on device d, extended to every resident
// class (see Derived). Least recently used sets beyond kMaxDerived are released.
int ensure_derived(tqsb_plan* p, Device* d, const tqsb_config& c, Derived** out, int* launches) {
    const bool f32 = uses_f32(c);
    const double step = f32 ? c.step_width : 0.0;
    Derived* dv = nullptr;
    for (auto& x : d->derived)
        if (x->f32 == f32 && x->exponent == c.frequency_exponent && x->step == step) dv = x.get();
    CUDA_TRY(cudaSetDevice(d->id));
    const WindowTables& t = p->wt;
    if (!dv) {
        if (d->derived.size() >= kMaxDerived) {
            auto lru = std::min_element(d->derived.begin(), d->derived.end(),
                                        [](const auto& x, const auto& y) { return x->last_use < y->last_use; });
            CUDA_TRY(cudaDeviceSynchronize());  // device-API launches may still read it
            for (auto& sl : (*lru)->slabs) d->table_bytes -= sl.bytes;
            derived_free(lru->get());
            d->derived.erase(lru);
        }
        auto nd = std::make_unique<Derived>();
        nd->exponent = c.frequency_exponent;
        nd->step = step;
        nd->f32 = f32;
        const std::vector<double> q = frequency_weights(t.W, c.frequency_exponent);
        CUDA_TRY(cudaMalloc(&nd->d_q64, sizeof(double) * t.K));
        CUDA_TRY(cudaMemcpy(nd->d_q64, q.data(), sizeof(double) * t.K, cudaMemcpyHostToDevice));
        dv = nd.get();
        d->derived.push_back(std::move(nd));
    }
    dv->last_use = ++d->use_clock;
    const size_t n0 = dv->tabs.size(), n = d->tabs.size();
    if (n0 < n) {
        const size_t K_pad = t.K_pad;
        std::vector<ClassBuild> descs;
        for (size_t i = n0; i < n; ++i) {
            ClassTab tab = d->tabs[i];
            ClassSlab slab;
            if (f32) {
                const size_t o_cpack = 0, o_scale = align_up(K_pad * K_pad * 8, 256),
                             o_fac = o_scale + align_up(K_pad * 4, 256);
                slab.bytes = o_fac + align_up(K_pad * 4, 256);
                CUDA_TRY(cudaMalloc(&slab.base, slab.bytes));
                char* b = static_cast<char*>(slab.base);
                ClassBuild cb{};
                cb.local = tab.local;
                cb.c64 = const_cast<double*>(tab.c64);
                cb.d64 = const_cast<double*>(tab.d64);
                cb.cpack = reinterpret_cast<float*>(b + o_cpack);
                cb.scale = reinterpret_cast<float*>(b + o_scale);
                cb.fac = reinterpret_cast<float*>(b + o_fac);
                tab.cpack = cb.cpack;
                tab.scale = cb.scale;
                tab.fac = cb.fac;
                descs.push_back(cb);
                d->table_bytes += slab.bytes;
            }
            dv->slabs.push_back(slab);
            dv->tabs.push_back(tab);
        }
        if (!descs.empty()) {
            const int rc = launch_tables_derive(descs.data(), int(descs.size()), t.W, t.K_pad, step,
                                                dv->d_q64, d->d_perm, d->stream, launches);
            if (rc != 0)
                return set_error(TQSB_ECUDA, std::string("table derive: ") +
                                                 cudaGetErrorString(cudaError_t(rc)));
        }
        if (dv->tabs.size() > dv->d_tabs_cap) {
            CUDA_TRY(cudaStreamSynchronize(d->stream));
            cudaFree(dv->d_tabs);
            dv->d_tabs = nullptr;
            dv->d_tabs_cap = std::max<size_t>(dv->tabs.size() * 2, 16);
            CUDA_TRY(cudaMalloc(&dv->d_tabs, sizeof(ClassTab) * dv->d_tabs_cap));
        }
        CUDA_TRY(cudaMemcpyAsync(dv->d_tabs, dv->tabs.data(), sizeof(ClassTab) * dv->tabs.size(),
                                 cudaMemcpyHostToDevice, d->stream));
        CUDA_TRY(cudaStreamSynchronize(d->stream));
    }
    *out = dv;
    return TQSB_OK;
}

// Class-sorted tasks and CTA work items for a band of block rows on device d;
// the band's classes are made resident first (cached per frame shape and band).
int prepare_band(tqsb_plan* p, Device* d, const tqsb_config& c, const Geometry& g, int frame_rows,
                 int frame_cols, int br0, int br1, Work** out, int* created, int* launches,
                 int stream = 0, int order_chunks = 0) {
    *created = 0;
    const int chunk = (uses_f32(c) ? kWarpsF32 : kWarpsF64) * 4;
    // order_chunks: the same chunk-by-chunk order without the chunk tags (experiment knob)
    const WorkKey wkey{frame_rows, frame_cols, br0, br1, g.B, chunk, stream > 0 ? stream : -order_chunks};
    Enumerated e;
    auto it = d->works.find(wkey);
    if (it != d->works.end()) {
        // the work list is cached; its classes may have been created under another
        // option set, so make sure they are (still) resident
        bool all = true;
        for (int k : it->second.keys) all = all && d->slot_of.count(k);
        if (all) {
            *out = &it->second;
            return TQSB_OK;
        }
    }
    enumerate(g, p->period, br0, br1, &e);
    TQSB_TRY(ensure_classes(p, d, c, e.class_order, e.representative, created, launches));
    if (it != d->works.end()) {
        *out = &it->second;
        return TQSB_OK;
    }
    Work w;
    w.keys = e.class_order;
    w.classes_total = e.classes_total;
    w.classes_interior = e.classes_interior;
    w.n_tasks = int(e.tasks.size());
    int omin = std::numeric_limits<int>::max(), omax = 0;
    for (const Task& t : e.tasks) {
        omin = std::min(omin, t.origin_row);
        omax = std::max(omax, t.origin_row);
    }
    if (e.tasks.empty()) omin = omax = 0;
    w.frame_row0 = std::min(omin / 2, frame_rows - 1);
    w.frame_row1 = std::min(frame_rows, (omax + g.W - 1) / 2 + 1);
    // class-sorted (stable) task list, cut into CTA work items of one class each; a
    // streamed list is ordered chunk by chunk of block rows first (class-sorted inside
    // each chunk) and carries the chunk in task_cls
    const int n_chunks = stream > 0 ? stream : order_chunks > 0 ? order_chunks : 1;
    const int nbr = br1 - br0;
    // chunk boundaries shrink toward the end (fraction 1 - (1 - s/S)^2): the rows handed
    // over after the kernel ends -- the exposed tail -- are the last, smallest chunk
    for (int s = 0; s <= n_chunks; ++s) {
        const double f = 1.0 - (1.0 - double(s) / n_chunks) * (1.0 - double(s) / n_chunks);
        int b = br0 + int(std::lround(nbr * f));
        if (s > 0) b = std::max(b, w.chunk_br.back());
        w.chunk_br.push_back(s == n_chunks ? br1 : b);
    }
    w.chunk_count.assign(n_chunks, 0);
    w.chunk_fr_hi.assign(n_chunks, w.frame_row0);
    std::vector<Task> sorted;
    std::vector<WorkItem> items;
    std::vector<int> task_cls;
    sorted.reserve(e.tasks.size());
    task_cls.reserve(e.tasks.size());
    for (int ch = 0; ch < n_chunks; ++ch) {
        std::vector<std::vector<Task>> by_key(size_t(p->period) * p->period);
        for (size_t i = 0; i < e.tasks.size(); ++i) {
            const int bri = e.tasks[i].block_row / g.B;
            if (bri >= w.chunk_br[ch] && bri < w.chunk_br[ch + 1]) {
                by_key[e.keys[i]].push_back(e.tasks[i]);
                // frame rows the chunk's windows read: through (origin + W - 1) / 2
                w.chunk_fr_hi[ch] = std::max(
                    w.chunk_fr_hi[ch], std::min(frame_rows, (e.tasks[i].origin_row + g.W - 1) / 2 + 1));
            }
        }
        for (int k : e.class_order) {
            const auto& v = by_key[k];
            for (size_t s = 0; s < v.size(); s += chunk) {
                WorkItem wi{};
                wi.cls = d->slot_of.at(k);
                wi.start = int(sorted.size() + s);
                wi.count = int(std::min<size_t>(chunk, v.size() - s));
                items.push_back(wi);
            }
            sorted.insert(sorted.end(), v.begin(), v.end());
            task_cls.insert(task_cls.end(), v.size(),
                            d->slot_of.at(k) | (stream > 0 ? ch << kTaskClsBits : 0));
            w.chunk_count[ch] += int(v.size());
        }
    }
    w.n_items = int(items.size());
    CUDA_TRY(cudaSetDevice(d->id));
    CUDA_TRY(cudaMalloc(&w.d_tasks, sizeof(Task) * std::max<size_t>(1, sorted.size())));
    CUDA_TRY(cudaMalloc(&w.d_items, sizeof(WorkItem) * std::max<size_t>(1, items.size())));
    CUDA_TRY(cudaMemcpy(w.d_tasks, sorted.data(), sizeof(Task) * sorted.size(),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(w.d_items, items.data(), sizeof(WorkItem) * items.size(),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc(&w.d_task_cls, sizeof(int) * std::max<size_t>(1, task_cls.size())));
    CUDA_TRY(cudaMemcpy(w.d_task_cls, task_cls.data(), sizeof(int) * task_cls.size(),
                        cudaMemcpyHostToDevice));
    auto ins = d->works.emplace(wkey, std::move(w));
    *out = &ins.first->second;
    return TQSB_OK;
}

int ensure_buffer(double** buf, size_t* cap, size_t n) {
    if (*cap >= n) return TQSB_OK;
    cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    CUDA_TRY(cudaMalloc(buf, sizeof(double) * std::max<size_t>(n, 1)));
    *cap = n;
    return TQSB_OK;
}

int ensure_pinned(double** buf, size_t* cap, size_t n) {
    if (*cap >= n) return TQSB_OK;
    if (*buf) cudaFreeHost(*buf);
    *buf = nullptr;
    *cap = 0;
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(buf), sizeof(double) * std::max<size_t>(n, 1),
                           cudaHostAllocDefault));
    *cap = n;
    return TQSB_OK;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// kernel arguments of one call: the call's solver options (nu, gamma, clip, block,
// early stop) over the derived tables of its option set
SolveArgs base_args(tqsb_plan* p, Device* d, const tqsb_config& c, const Derived* dv) {
    SolveArgs a{};
    a.tabs = dv->d_tabs;
    a.wc.perm = d->d_perm;
    a.wc.src = d->d_src;
    a.wc.unit32 = d->d_unit32;
    a.wc.unit64 = d->d_unit64;
    a.wc.q64 = dv->d_q64;
    a.window = c.window;
    a.block = c.block;
    a.iterations = c.max_iterations;
    a.step = c.step_width;
    a.clip = c.clip_output;
    // TMEM column tier: off unless asked for (auto = 0; with predicated per-chunk loads it
    // costs more issue slots than it saves: 4K frame 40.6 ms with 8 hot columns vs 40.1)
    const int maxhot = std::min(solve_f32_max_hot(p->wt.NS, d->id), p->wt.K_pad);
    a.hot = uses_f32(c) && c.hot_columns > 0 ? std::min(c.hot_columns, maxhot) : 0;
    a.early_stop = c.early_stop;
    a.early_stop_scale = c.early_stop_scale;
    // a fresh queue head per launch (zeroed on the launch stream in launch()), so
    // reconstructions in flight on different streams never share one
    a.counter = d->d_counters + (d->counter_next++ % kCounterRing);
    return a;
}

int launch(const tqsb_config& c, Device* d, const SolveArgs& a, cudaStream_t s, int n_slots) {
    if (a.counter) CUDA_TRY(cudaMemsetAsync(a.counter, 0, sizeof(int), s));
    int rc;
    if (c.algorithm == TQSB_ALGO_LJSDE) {
        rc = launch_solve_ljsde(a, s, d->num_sms);
    } else if (uses_f32(c)) {
        rc = launch_solve_f32(a, n_slots, s, d->num_sms);
    } else {  // fp64 mode: register-resident kernel where it applies, else the general one
        rc = launch_solve_f64r(a, s, d->num_sms);
        if (rc == cudaErrorNotSupported) rc = launch_solve_f64(a, s, d->num_sms);
    }
    if (rc != 0)
        return set_error(TQSB_ECUDA, std::string("solve launch: ") +
                                         cudaGetErrorString(cudaError_t(rc)));
    return TQSB_OK;
}

struct BandResult {
    int rc = TQSB_OK;
    std::string err;
    float ms = 0.f;
    double warm = 0.0;
    int created = 0;
    int launches = 0;
    long long classes_total = 0, classes_interior = 0, blocks = 0;
};

// First-touch population of a caller's output buffer while the GPU works, so the
// hand-over copies find resident pages (a fresh std::vector / numpy array faults on
// every 4 KB page: ~16 k faults for a 4K frame). MADV_POPULATE_WRITE (Linux 5.14)
// populates without changing contents, so it may run alongside the copies; on older
// kernels it fails harmlessly and the copies fault as before.
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
std::thread prefault_async(void* p, size_t bytes) {
    static const bool enabled = [] {
        const char* v = std::getenv("TQSB_PREFAULT");
        return !(v && v[0] == '0');
    }();
    if (!enabled || bytes < (size_t(1) << 20)) return std::thread();
    return std::thread([p, bytes] {
        const uintptr_t pg = uintptr_t(sysconf(_SC_PAGESIZE));
        uintptr_t a = (reinterpret_cast<uintptr_t>(p) + pg - 1) / pg * pg;
        const uintptr_t end = (reinterpret_cast<uintptr_t>(p) + bytes) / pg * pg;
        const uintptr_t step = uintptr_t(4) << 20;  // in order, 4 MB at a time
        for (; a < end; a += step)
            if (madvise(reinterpret_cast<void*>(a), std::min(step, end - a), MADV_POPULATE_WRITE) != 0)
                break;
    });
}

// cuStreamWaitValue32 (stream memory operations, driver API) through the runtime's
// driver entry-point query; null when the driver or device does not offer it
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32Fn wait_value32() {
    static WaitValue32Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return WaitValue32Fn(nullptr);
        }
        return reinterpret_cast<WaitValue32Fn>(f);
    }();
    return fn;
}

// Host-buffer band run on device d: H2D of the band's frame rows (halo included),
// one solve launch whose B x B output tiles are stored straight into pinned host
// memory (zero-copy: the caller's buffer when it is pinned, else the plan's pinned
// staging), so the output transfer overlaps the solve instead of following it.
void run_band_host(tqsb_plan* p, Device* d, const tqsb_config& c, const Geometry& g,
                   const double* frame, int frame_rows, int frame_cols, int br0, int br1,
                   double* out_band, BandResult* r) {
    auto fail = [&](int rc) {
        r->rc = rc;
        r->err = g_error;
    };
    if (cudaSetDevice(d->id) != cudaSuccess) return fail(set_error(TQSB_ECUDA, "cudaSetDevice"));
    const bool out_pinned = is_pinned(out_band);
    // A pageable output on the fp32 kernel streams: the kernel stores into device memory
    // and counts finished blocks per chunk of block rows; a copy stream waits on each
    // chunk's count (cuStreamWaitValue32) and moves its rows to pinned staging, and the
    // host hands them to the caller's buffer -- so the staging copy and the first-touch
    // page faults of a fresh buffer overlap the solve instead of following it.
    const long long n_est = (long long)(br1 - br0) * (g.padN / g.B);
    // Chunk-major order interleaves the classes: every chunk sweeps all of them, which is
    // free while their C' tables share the L2 (P = 8: 4 interior classes, 32 MB) and costs
    // HBM re-reads when they do not (P = 32: 64 classes, 512 MB) -- fewer chunks then.
    const int per_axis = p->period / std::gcd(p->period, c.block);
    const int n_chunks = std::clamp(128 / std::max(1, per_axis * per_axis), 1, kStreamChunks);
    // (the warp-scheduled kernel only: the TMEM column tier runs CTA work items)
    // (pinned outputs only for large frames: below ~half a 4K frame the kernel's zero-copy
    // stores beat the chunk copies -- 1 MP, P = 8: 211.4 vs 206.6 MP/s)
    const int stream = uses_f32(c) && c.algorithm == TQSB_ALGO_RLJSDE &&
                               c.hot_columns <= 0 &&
                               solve_f32_streams(p->wt.NS, c.block * c.block) &&
                               n_est >= (out_pinned ? kStreamMinTasksPinned : kStreamMinTasks) &&
                               br1 - br0 >= kStreamChunks &&
                               n_chunks >= 2 && wait_value32() != nullptr
                           ? n_chunks
                           : 0;
    Work* w = nullptr;
    Derived* dv = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    int rc = prepare_band(p, d, c, g, frame_rows, frame_cols, br0, br1, &w, &r->created, &r->launches,
                          stream);
    if (!rc) rc = ensure_derived(p, d, c, &dv, &r->launches);
    if (rc) return fail(rc);
    r->warm = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r->classes_total = w->classes_total;
    r->classes_interior = w->classes_interior;
    r->blocks = w->n_tasks;
    const int fr0 = w->frame_row0, fr1 = w->frame_row1;
    const size_t in_n = size_t(fr1 - fr0) * frame_cols;
    const int orow0 = br0 * g.B, orow1 = std::min(br1 * g.B, g.M);
    const size_t out_n = size_t(std::max(0, orow1 - orow0)) * g.N;
    if ((rc = ensure_buffer(&d->d_frame, &d->frame_cap, in_n))) return fail(rc);
    if (!out_pinned && (rc = ensure_pinned(&d->h_out, &d->h_out_cap, out_n))) return fail(rc);
    if (stream) {
        if ((rc = ensure_buffer(&d->d_out, &d->out_cap, out_n))) return fail(rc);
        if (!d->d_progress) {
            CUDA_TRY_V(cudaMalloc(&d->d_progress, sizeof(int) * 64));
            for (auto& e : d->ev_chunk) CUDA_TRY_V(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    const double* src = frame + size_t(fr0) * frame_cols;
    // The input goes in one asynchronous copy before the launch; a pageable frame is staged
    // by the driver, which pipelines its bounce buffers with the DMA (measured at 4K: +0.9
    // to 1.3 ms over a pinned frame, against +1.2 / 1.6 / 2.6 ms for our own staging copy
    // on 4 / 8 / 16 threads and +2.7 ms for cudaHostRegister + unregister per call). A
    // kernel waiting on rows staged after its launch was faster still but would deadlock
    // wherever launches are synchronous (CUDA_LAUNCH_BLOCKING=1, compute-sanitizer, ncu),
    // so the kernel never waits on later stream work.
    double* host_out = out_pinned ? out_band : d->h_out;
    double* dev_view = nullptr;  // the pinned output as seen from the device (UVA)
    if (stream) {
        dev_view = d->d_out;
    } else if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev_view), host_out, 0) != cudaSuccess) {
        cudaGetLastError();
        return fail(set_error(TQSB_ECUDA, "output buffer is not device-mapped pinned memory"));
    }
    // A streamed call with a pageable frame runs as two launches: the first chunk (the
    // largest, ~1/8 of the rows at 16 chunks) starts once its frame rows are copied, and
    // the remaining rows are copied (the driver's host-side staging included) while it
    // runs; the second launch waits for them through an event. Only stream order is
    // involved -- nothing spins, so synchronous launches stay correct.
    const bool split = stream >= 2 && !is_pinned(frame);
    const int half = 1;
    size_t in_first = in_n;
    if (split) {
        const int hi = std::max(w->chunk_fr_hi[half - 1], fr0);
        in_first = std::min(in_n, size_t(hi - fr0) * frame_cols);
    }
    CUDA_TRY_V(cudaMemcpyAsync(d->d_frame, src, sizeof(double) * in_first, cudaMemcpyHostToDevice,
                               d->stream));
    SolveArgs a = base_args(p, d, c, dv);
    a.frame = d->d_frame;
    a.frame_rows = frame_rows;
    a.frame_cols = frame_cols;
    a.frame_row0 = fr0;
    a.frame_pitch = frame_cols;
    a.out = dev_view;
    a.out_row0 = orow0;
    a.out_rows = g.M;
    a.out_cols = g.N;
    a.tasks = w->d_tasks;
    a.items = w->d_items;
    a.n_items = w->n_items;
    a.task_cls = w->d_task_cls;
    a.n_tasks = w->n_tasks;
    // rows [chunk_br[s] * B, chunk_br[s+1] * B) of the output, cropped to M, relative to orow0
    auto chunk_rows = [&](int s, size_t* off, size_t* n) {
        const int r0 = std::min(w->chunk_br[s] * g.B, g.M), r1 = std::min(w->chunk_br[s + 1] * g.B, g.M);
        *off = size_t(std::max(0, r0 - orow0)) * g.N;
        *n = size_t(std::max(0, r1 - r0)) * g.N;
    };
    if (stream) {
        a.progress = d->d_progress;
        CUDA_TRY_V(cudaMemsetAsync(d->d_progress, 0, sizeof(int) * stream, d->stream));
        CUDA_TRY_V(cudaEventRecord(d->ev_h2d[2], d->stream));  // counters zeroed
        CUDA_TRY_V(cudaStreamWaitEvent(d->s_d2h, d->ev_h2d[2], 0));
    }
    cudaEventRecord(d->ev0, d->stream);
    if (split && w->n_items > 0) {
        int first = 0;
        for (int s2 = 0; s2 < half; ++s2) first += w->chunk_count[s2];
        SolveArgs a1 = a;
        a1.n_tasks = first;
        if ((rc = launch(c, d, a1, d->stream, p->wt.NS))) return fail(rc);
        // the rest of the frame on the copy stream while the first half solves
        CUDA_TRY_V(cudaMemcpyAsync(d->d_frame + in_first, src + in_first,
                                   sizeof(double) * (in_n - in_first), cudaMemcpyHostToDevice,
                                   d->s_h2d));
        CUDA_TRY_V(cudaEventRecord(d->ev_h2d[3], d->s_h2d));
        CUDA_TRY_V(cudaStreamWaitEvent(d->stream, d->ev_h2d[3], 0));
        SolveArgs a2 = a;
        a2.counter = d->d_counters + (d->counter_next++ % kCounterRing);  // its own queue head
        a2.tasks = a.tasks + first;
        a2.task_cls = a.task_cls + first;
        a2.n_tasks = a.n_tasks - first;
        if ((rc = launch(c, d, a2, d->stream, p->wt.NS))) return fail(rc);
        r->launches += 2;
    } else if (w->n_items > 0) {
        if ((rc = launch(c, d, a, d->stream, p->wt.NS))) return fail(rc);
        r->launches += 1;
    }
    cudaEventRecord(d->ev1, d->stream);
    std::thread prefault;  // joined before returning (the buffer is the caller's)
    struct Joiner {
        std::thread& t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } joiner{prefault};
    if (stream && !out_pinned) prefault = prefault_async(out_band, sizeof(double) * out_n);
    if (stream) {
        WaitValue32Fn waitv = wait_value32();
        for (int s = 0; s < stream; ++s) {
            size_t off, n;
            chunk_rows(s, &off, &n);
            if (waitv(reinterpret_cast<CUstream>(d->s_d2h),
                      reinterpret_cast<CUdeviceptr>(d->d_progress + s),
                      cuuint32_t(w->chunk_count[s]), CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return fail(set_error(TQSB_ECUDA, "cuStreamWaitValue32 failed"));
            // straight into a pinned caller buffer, else into the pinned staging
            if (n) cudaMemcpyAsync(host_out + off, d->d_out + off, sizeof(double) * n,
                                   cudaMemcpyDeviceToHost, d->s_d2h);
            cudaEventRecord(d->ev_chunk[s], d->s_d2h);
        }
        // hand the chunks over as they land; a failed solve releases the copy stream
        int s = 0;
        for (; s < stream; ++s) {
            cudaError_t q;
            std::chrono::steady_clock::time_point done_at{};
            bool solve_done = false;
            while ((q = cudaEventQuery(d->ev_chunk[s])) == cudaErrorNotReady) {
                const cudaError_t m = cudaStreamQuery(d->stream);
                if (m != cudaErrorNotReady && m != cudaSuccess) break;  // the solve failed
                if (m == cudaSuccess) {  // solved: the chunk copies must land promptly
                    if (!solve_done) done_at = std::chrono::steady_clock::now(), solve_done = true;
                    else if (std::chrono::steady_clock::now() - done_at > std::chrono::seconds(5)) break;
                }
                std::this_thread::yield();
            }
            if (q != cudaSuccess) break;
            if (!out_pinned) {
                size_t off, n;
                chunk_rows(s, &off, &n);
                par_memcpy(out_band + off, d->h_out + off, sizeof(double) * n, 4);
            }
        }
        if (s < stream) {  // the solve failed: unblock the waits so the copy stream drains
            const cudaError_t err = cudaStreamSynchronize(d->stream);
            std::vector<int> big(stream, 0x7fffffff);
            cudaMemcpy(d->d_progress, big.data(), sizeof(int) * stream, cudaMemcpyHostToDevice);
            cudaStreamSynchronize(d->s_d2h);
            cudaGetLastError();
            return fail(set_error(TQSB_ECUDA, std::string("solve: ") + cudaGetErrorString(
                                                  err != cudaSuccess ? err : cudaErrorUnknown)));
        }
    }
    cudaError_t e = cudaStreamSynchronize(d->stream);
    if (e != cudaSuccess)
        return fail(set_error(TQSB_ECUDA, std::string("solve: ") + cudaGetErrorString(e)));
    cudaEventElapsedTime(&r->ms, d->ev0, d->ev1);
    if (!stream && !out_pinned) par_memcpy(out_band, d->h_out, sizeof(double) * out_n);
}

// Multi-frame pipeline on one device: frame i+1's H2D (copy stream) overlaps frame
// i's solve; outputs are stored zero-copy into pinned host memory by the kernel.
// Pageable frames/outputs go through double-buffered pinned staging.
void run_batch_host(tqsb_plan* p, Device* d, const tqsb_config& c, const Geometry& g,
                    const double* const* frames, int frame_rows, int frame_cols,
                    double* const* outs, int n, BandResult* r) {
    auto fail = [&](int rc) {
        r->rc = rc;
        r->err = g_error;
    };
    if (n <= 0) return;
    if (cudaSetDevice(d->id) != cudaSuccess) return fail(set_error(TQSB_ECUDA, "cudaSetDevice"));
    Work* w = nullptr;
    Derived* dv = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const int nbr = g.padM / g.B;
    int rc = prepare_band(p, d, c, g, frame_rows, frame_cols, 0, nbr, &w, &r->created, &r->launches);
    if (!rc) rc = ensure_derived(p, d, c, &dv, &r->launches);
    if (rc) return fail(rc);
    r->warm = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r->classes_total = w->classes_total;
    r->classes_interior = w->classes_interior;
    r->blocks = (long long)w->n_tasks * n;
    const size_t in_n = size_t(frame_rows) * frame_cols;
    const size_t out_n = size_t(g.M) * g.N;
    for (int k = 0; k < 2; ++k) {
        if ((rc = ensure_buffer(&d->d_fs[k], &d->fs_cap[k], in_n))) return fail(rc);
        if ((rc = ensure_pinned(&d->h_in_s[k], &d->h_in_s_cap[k], in_n))) return fail(rc);
        if ((rc = ensure_pinned(&d->h_out_s[k], &d->h_out_s_cap[k], out_n))) return fail(rc);
    }
    std::vector<char> out_pinned(n);
    for (int i = 0; i < n; ++i) out_pinned[i] = is_pinned(outs[i]);
    for (int i = 0; i < n; ++i) {
        const int s = i & 1;
        const double* src = frames[i];
        if (!is_pinned(src)) {
            if (i >= 2) cudaEventSynchronize(d->ev_h2d[s]);  // staging slot free again
            par_memcpy(d->h_in_s[s], src, sizeof(double) * in_n);
            src = d->h_in_s[s];
        }
        if (i >= 2) cudaStreamWaitEvent(d->s_h2d, d->ev_comp[s], 0);  // frame i-2 done with d_fs[s]
        cudaMemcpyAsync(d->d_fs[s], src, sizeof(double) * in_n, cudaMemcpyHostToDevice, d->s_h2d);
        cudaEventRecord(d->ev_h2d[s], d->s_h2d);
        cudaStreamWaitEvent(d->stream, d->ev_h2d[s], 0);
        // frame i-2 staged its output in h_out_s[s]: hand it over before anything may
        // reuse the slot (whether or not frame i needs staging itself)
        if (i >= 2 && !out_pinned[i - 2]) {
            cudaEventSynchronize(d->ev_comp[s]);
            par_memcpy(outs[i - 2], d->h_out_s[s], sizeof(double) * out_n);
        }
        double* host_out = out_pinned[i] ? outs[i] : d->h_out_s[s];
        double* dev_view = nullptr;
        if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev_view), host_out, 0) != cudaSuccess) {
            cudaGetLastError();
            return fail(set_error(TQSB_ECUDA, "output buffer is not device-mapped pinned memory"));
        }
        SolveArgs a = base_args(p, d, c, dv);
        a.frame = d->d_fs[s];
        a.frame_rows = frame_rows;
        a.frame_cols = frame_cols;
        a.frame_row0 = 0;
        a.frame_pitch = frame_cols;
        a.out = dev_view;
        a.out_row0 = 0;
        a.out_rows = g.M;
        a.out_cols = g.N;
        a.tasks = w->d_tasks;
        a.items = w->d_items;
        a.n_items = w->n_items;
        a.task_cls = w->d_task_cls;
        a.n_tasks = w->n_tasks;
        if (i == 0) cudaEventRecord(d->ev0, d->stream);
        if (w->n_items > 0) {
            if ((rc = launch(c, d, a, d->stream, p->wt.NS))) return fail(rc);
            r->launches += 1;
        }
        cudaEventRecord(d->ev_comp[s], d->stream);
    }
    cudaEventRecord(d->ev1, d->stream);
    cudaError_t e = cudaStreamSynchronize(d->stream);
    if (e != cudaSuccess)
        return fail(set_error(TQSB_ECUDA, std::string("solve: ") + cudaGetErrorString(e)));
    for (int i = std::max(0, n - 2); i < n; ++i)
        if (!out_pinned[i]) par_memcpy(outs[i], d->h_out_s[i & 1], sizeof(double) * out_n);
    cudaEventElapsedTime(&r->ms, d->ev0, d->ev1);
}

void fill_report(tqsb_report* rep, const std::vector<BandResult>& rs, const tqsb_config& c,
                 long long classes_total, long long classes_interior, double e2e) {
    if (!rep) return;
    std::memset(rep, 0, sizeof(*rep));
    double sec = 0, warm = 0;
    long long blocks = 0, created = 0;
    int launches = 0;
    for (const auto& r : rs) {
        sec = std::max(sec, double(r.ms) * 1e-3);
        warm = std::max(warm, r.warm);
        blocks += r.blocks;
        created = std::max<long long>(created, r.created);
        launches += r.launches;
    }
    rep->seconds = sec;
    rep->warm_seconds = warm;
    rep->e2e_seconds = e2e;
    rep->blocks_processed = blocks;
    rep->classes_total = classes_total;
    rep->classes_interior = classes_interior;
    rep->classes_created = created;
    // reference semantics: one lookup per class in the warm pass, one per block
    rep->cache_misses = created;
    rep->cache_hits = blocks + (classes_total - created);
    rep->psnr_db = 0.0;
    rep->has_psnr = 0;
    rep->gpu_launches = launches;
    rep->compute = uses_f32(c) ? TQSB_COMPUTE_FP32 : TQSB_COMPUTE_FP64;
}

// L-JSDE keeps no kernel cache in the reference (pipeline.cpp:111-112, 173-177):
// its report carries no cache counters (the device still builds B and D per class)
void ljsde_report(const tqsb_config& c, tqsb_report* rep) {
    if (!rep || c.algorithm != TQSB_ALGO_LJSDE) return;
    rep->classes_created = 0;
    rep->cache_hits = 0;
    rep->cache_misses = 0;
}

double psnr_impl(const double* a, const double* b, long long n) {
    double sum = 0.0;
    for (long long i = 0; i < n; ++i) {
        const double d = a[i] - b[i];
        sum += d * d;
    }
    const double mse = sum / double(n);
    if (mse == 0.0) return std::numeric_limits<double>::infinity();
    return -10.0 * std::log10(mse);
}

} // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* tqsb_last_error(void) { return g_error.c_str(); }
const char* tqsb_version(void) { return "tqsb 0.1 (sm_100a)"; }

void tqsb_config_default(tqsb_config* c) {
    c->window = 32;
    c->block = 4;
    c->max_iterations = 200;
    c->step_width = 0.5;
    c->spatial_decay = 0.8;
    c->frequency_exponent = 2.0;
    c->precision = TQSB_PRECISION_DOUBLE;
    c->clip_output = 1;
    c->threads = 1;
    c->compute = TQSB_COMPUTE_FP32;
    c->hot_columns = -1;
    c->algorithm = TQSB_ALGO_RLJSDE;
    c->early_stop = 0;
    c->early_stop_scale = 1e-14;
}

int tqsb_validate_config(const tqsb_config* cfg, int period) {
    if (!cfg) return set_error(TQSB_EINVAL, "null config");
    return validate(*cfg, period);
}

int tqsb_census(int frame_rows, int frame_cols, const tqsb_config* cfg, int period,
                long long out[3]) {
    if (!cfg || !out) return set_error(TQSB_EINVAL, "null argument");
    TQSB_TRY(validate(*cfg, period));
    Geometry g;
    TQSB_TRY(geometry(*cfg, frame_rows, frame_cols, &g));
    Enumerated e;
    enumerate(g, period, 0, g.padM / g.B, &e);
    out[0] = (long long)e.tasks.size();
    out[1] = e.classes_total;
    out[2] = e.classes_interior;
    return TQSB_OK;
}

int tqsb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int tqsb_plan_create(const uint8_t* opaque, int period, const tqsb_config* cfg,
                     const int* devices, int n_devices, tqsb_plan** out) {
    if (!out || !cfg || !opaque) return set_error(TQSB_EINVAL, "null argument");
    *out = nullptr;
    if (period < 4 || period % 2 != 0)
        return set_error(TQSB_EINVAL, "pattern period must be even and >= 4");
    TQSB_TRY(validate(*cfg, period));
    if (n_devices < 1) return set_error(TQSB_EINVAL, "at least one device is required");
    const int have = tqsb_device_count();
    if (have < 1) return set_error(TQSB_ENODEV, "no CUDA device available (no CPU fallback)");
    auto p = std::make_unique<tqsb_plan>();
    p->cfg = *cfg;
    p->period = period;
    p->opaque.assign(opaque, opaque + size_t(period / 2) * (period / 2));
    for (uint8_t q : p->opaque)
        if (q > 3) return set_error(TQSB_EINVAL, "quadrant indices must be in 0..3");
    p->wt = window_tables(*cfg);
    for (int i = 0; i < n_devices; ++i) {
        const int id = devices ? devices[i] : i;
        if (id < 0 || id >= have) return set_error(TQSB_ENODEV, "device index out of range");
        auto d = std::make_unique<Device>();
        d->id = id;
        int rc = device_init(p.get(), d.get());
        p->devs.push_back(std::move(d));
        if (rc) {
            for (auto& dd : p->devs) device_free(dd.get());
            return rc;
        }
    }
    *out = p.release();
    return TQSB_OK;
}

int tqsb_plan_destroy(tqsb_plan* p) {
    if (!p) return TQSB_OK;
    for (auto& d : p->devs) device_free(d.get());
    delete p;
    return TQSB_OK;
}

int tqsb_plan_stats(const tqsb_plan* p, long long* classes, long long* bytes) {
    if (!p) return set_error(TQSB_EINVAL, "null plan");
    if (classes) *classes = p->devs.empty() ? 0 : (long long)p->devs[0]->tabs.size();
    if (bytes) *bytes = p->devs.empty() ? 0 : (long long)p->devs[0]->table_bytes;
    return TQSB_OK;
}

int tqsb_plan_warm(tqsb_plan* p, int frame_rows, int frame_cols, double* warm_seconds) {
    if (!p) return set_error(TQSB_EINVAL, "null plan");
    std::lock_guard<std::mutex> lk(p->mu);
    Geometry g;
    TQSB_TRY(geometry(p->cfg, frame_rows, frame_cols, &g));
    const auto t0 = std::chrono::steady_clock::now();
    Enumerated e;
    enumerate(g, p->period, 0, g.padM / g.B, &e);
    for (auto& d : p->devs) {
        int created = 0, launches = 0;
        Derived* dv = nullptr;
        TQSB_TRY(ensure_classes(p, d.get(), p->cfg, e.class_order, e.representative, &created,
                                &launches));
        TQSB_TRY(ensure_derived(p, d.get(), p->cfg, &dv, &launches));
    }
    for (auto& d : p->devs) {
        cudaSetDevice(d->id);
        CUDA_TRY(cudaStreamSynchronize(d->stream));
    }
    if (warm_seconds)
        *warm_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return TQSB_OK;
}

} // extern "C"

namespace {

// The configuration a call runs with: the plan's own, or the caller's per-call config
// over the plan's tables (the reference's shared KernelCache: each call brings its own
// q, nu, gamma, block, clip and algorithm, pipeline.cpp:108-166; the cache only pins
// the window, pipeline.cpp:146-147).
int call_config(const tqsb_plan* p, const tqsb_config* call, tqsb_config* out) {
    if (!call) {
        *out = p->cfg;
        return TQSB_OK;
    }
    TQSB_TRY(validate(*call, p->period));
    if (call->window != p->cfg.window)
        return set_error(TQSB_ELOGIC, "kernel cache holds a different window size");
    *out = *call;
    return TQSB_OK;
}

int reconstruct_band_impl(tqsb_plan* p, const tqsb_config* call, const double* frame,
                          int frame_rows, int frame_cols, int br0, int br1, double* out_band,
                          tqsb_report* rep) {
    if (!p || !frame || !out_band) return set_error(TQSB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(p->mu);
    const auto t0 = std::chrono::steady_clock::now();
    tqsb_config c;
    TQSB_TRY(call_config(p, call, &c));
    Geometry g;
    TQSB_TRY(geometry(c, frame_rows, frame_cols, &g));
    if (br0 < 0 || br1 > g.padM / g.B || br0 > br1)
        return set_error(TQSB_EINVAL, "block-row band out of range");
    std::vector<BandResult> rs(1);
    run_band_host(p, p->devs[0].get(), c, g, frame, frame_rows, frame_cols, br0, br1, out_band, &rs[0]);
    if (rs[0].rc) return set_error(rs[0].rc, rs[0].err);
    fill_report(rep, rs, c, rs[0].classes_total, rs[0].classes_interior,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    ljsde_report(c, rep);
    return TQSB_OK;
}

int reconstruct_impl(tqsb_plan* p, const tqsb_config* call, const double* frame, int frame_rows,
                     int frame_cols, double* out, const double* reference, tqsb_report* rep) {
    if (!p || !frame || !out) return set_error(TQSB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(p->mu);
    const auto t0 = std::chrono::steady_clock::now();
    tqsb_config c;
    TQSB_TRY(call_config(p, call, &c));
    Geometry g;
    TQSB_TRY(geometry(c, frame_rows, frame_cols, &g));
    const int nbr = g.padM / g.B;
    const int nd = std::min<int>(int(p->devs.size()), std::max(1, nbr));
    std::vector<BandResult> rs(nd);
    std::vector<int> cut(nd + 1);
    for (int i = 0; i <= nd; ++i) cut[i] = int((long long)nbr * i / nd);
    if (nd == 1) {
        run_band_host(p, p->devs[0].get(), c, g, frame, frame_rows, frame_cols, 0, nbr, out, &rs[0]);
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < nd; ++i)
            th.emplace_back([&, i] {
                double* ob = out + size_t(cut[i]) * g.B * g.N;
                run_band_host(p, p->devs[i].get(), c, g, frame, frame_rows, frame_cols, cut[i],
                              cut[i + 1], ob, &rs[i]);
            });
        for (auto& t : th) t.join();
    }
    for (auto& r : rs)
        if (r.rc) return set_error(r.rc, r.err);
    // census of the whole frame (bands may share classes)
    Enumerated e;
    long long ct = rs[0].classes_total, ci = rs[0].classes_interior;
    if (nd > 1) {
        enumerate(g, p->period, 0, nbr, &e);
        ct = e.classes_total;
        ci = e.classes_interior;
    }
    const double e2e = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill_report(rep, rs, c, ct, ci, e2e);
    ljsde_report(c, rep);
    if (reference) {
        const double v = psnr_impl(reference, out, (long long)g.M * g.N);
        if (rep) {
            rep->psnr_db = v;
            rep->has_psnr = 1;
        }
    }
    return TQSB_OK;
}

int reconstruct_batch_impl(tqsb_plan* p, const tqsb_config* call, const double* const* frames,
                           int n_frames, int frame_rows, int frame_cols, double* const* outs,
                           tqsb_report* rep) {
    if (!p || !frames || !outs || n_frames < 0) return set_error(TQSB_EINVAL, "null argument");
    for (int i = 0; i < n_frames; ++i)
        if (!frames[i] || !outs[i]) return set_error(TQSB_EINVAL, "null frame or output pointer");
    std::lock_guard<std::mutex> lk(p->mu);
    const auto t0 = std::chrono::steady_clock::now();
    tqsb_config c;
    TQSB_TRY(call_config(p, call, &c));
    Geometry g;
    TQSB_TRY(geometry(c, frame_rows, frame_cols, &g));
    const int nd = std::max(1, std::min<int>(int(p->devs.size()), n_frames));
    std::vector<BandResult> rs(nd);
    std::vector<int> cut(nd + 1);
    for (int i = 0; i <= nd; ++i) cut[i] = int((long long)n_frames * i / nd);
    if (nd == 1) {
        run_batch_host(p, p->devs[0].get(), c, g, frames, frame_rows, frame_cols, outs, n_frames, &rs[0]);
    } else {  // whole frames per device, one host thread each
        std::vector<std::thread> th;
        for (int i = 0; i < nd; ++i)
            th.emplace_back([&, i] {
                run_batch_host(p, p->devs[i].get(), c, g, frames + cut[i], frame_rows, frame_cols,
                               outs + cut[i], cut[i + 1] - cut[i], &rs[i]);
            });
        for (auto& t : th) t.join();
    }
    for (auto& r : rs)
        if (r.rc) return set_error(r.rc, r.err);
    const double e2e = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill_report(rep, rs, c, rs[0].classes_total, rs[0].classes_interior, e2e);
    ljsde_report(c, rep);
    return TQSB_OK;
}

int device_band(tqsb_plan* p, const tqsb_config* call, const double* d_frame, int frame_rows,
                int frame_cols, int br0, int br1, double* d_out, void* stream, tqsb_report* rep) {
    std::lock_guard<std::mutex> lk(p->mu);
    tqsb_config c;
    TQSB_TRY(call_config(p, call, &c));
    Geometry g;
    TQSB_TRY(geometry(c, frame_rows, frame_cols, &g));
    if (br0 < 0 || br1 > g.padM / g.B || br0 > br1)
        return set_error(TQSB_EINVAL, "block-row band out of range");
    Device* d = p->devs[0].get();
    CUDA_TRY(cudaSetDevice(d->id));
    Work* w = nullptr;
    Derived* dv = nullptr;
    int created = 0, launches = 0;
    static const int order_env = [] {  // experiment knob: task order of the device path
        const char* v = std::getenv("TQSB_ORDER_CHUNKS");
        return v ? std::atoi(v) : 0;
    }();
    TQSB_TRY(prepare_band(p, d, c, g, frame_rows, frame_cols, br0, br1, &w, &created, &launches, 0,
                          uses_f32(c) ? order_env : 0));
    TQSB_TRY(ensure_derived(p, d, c, &dv, &launches));
    SolveArgs a = base_args(p, d, c, dv);
    a.frame = d_frame;
    a.frame_rows = frame_rows;
    a.frame_cols = frame_cols;
    a.frame_row0 = 0;
    a.frame_pitch = frame_cols;
    a.out = d_out;
    a.out_row0 = br0 * g.B;
    a.out_rows = g.M;
    a.out_cols = g.N;
    a.tasks = w->d_tasks;
    a.items = w->d_items;
    a.n_items = w->n_items;
    a.task_cls = w->d_task_cls;
    a.n_tasks = w->n_tasks;
    if (w->n_items > 0) {
        TQSB_TRY(launch(c, d, a, static_cast<cudaStream_t>(stream), p->wt.NS));
        launches += 1;
    }
    if (rep) {
        std::memset(rep, 0, sizeof(*rep));
        rep->blocks_processed = w->n_tasks;
        rep->classes_total = w->classes_total;
        rep->classes_interior = w->classes_interior;
        rep->classes_created = created;
        rep->cache_misses = created;
        rep->cache_hits = w->n_tasks + (w->classes_total - created);
        rep->gpu_launches = launches;
        rep->compute = uses_f32(c) ? TQSB_COMPUTE_FP32 : TQSB_COMPUTE_FP64;
        ljsde_report(c, rep);
    }
    return TQSB_OK;
}

}  // namespace

extern "C" {

int tqsb_reconstruct_band(tqsb_plan* p, const double* frame, int frame_rows, int frame_cols,
                          int br0, int br1, double* out_band, tqsb_report* rep) {
    return reconstruct_band_impl(p, nullptr, frame, frame_rows, frame_cols, br0, br1, out_band, rep);
}

int tqsb_reconstruct_band_with(tqsb_plan* p, const tqsb_config* call, const double* frame,
                               int frame_rows, int frame_cols, int br0, int br1, double* out_band,
                               tqsb_report* rep) {
    return reconstruct_band_impl(p, call, frame, frame_rows, frame_cols, br0, br1, out_band, rep);
}

int tqsb_reconstruct(tqsb_plan* p, const double* frame, int frame_rows, int frame_cols,
                     double* out, const double* reference, tqsb_report* rep) {
    return reconstruct_impl(p, nullptr, frame, frame_rows, frame_cols, out, reference, rep);
}

int tqsb_reconstruct_with(tqsb_plan* p, const tqsb_config* call, const double* frame,
                          int frame_rows, int frame_cols, double* out, const double* reference,
                          tqsb_report* rep) {
    return reconstruct_impl(p, call, frame, frame_rows, frame_cols, out, reference, rep);
}

int tqsb_reconstruct_batch(tqsb_plan* p, const double* const* frames, int n_frames,
                           int frame_rows, int frame_cols, double* const* outs, tqsb_report* rep) {
    return reconstruct_batch_impl(p, nullptr, frames, n_frames, frame_rows, frame_cols, outs, rep);
}

int tqsb_reconstruct_batch_with(tqsb_plan* p, const tqsb_config* call, const double* const* frames,
                                int n_frames, int frame_rows, int frame_cols, double* const* outs,
                                tqsb_report* rep) {
    return reconstruct_batch_impl(p, call, frames, n_frames, frame_rows, frame_cols, outs, rep);
}

int tqsb_reconstruct_device(tqsb_plan* p, const double* d_frame, int frame_rows, int frame_cols,
                            double* d_out, void* stream, tqsb_report* rep) {
    return tqsb_reconstruct_device_with(p, nullptr, d_frame, frame_rows, frame_cols, d_out, stream,
                                        rep);
}

int tqsb_reconstruct_device_with(tqsb_plan* p, const tqsb_config* call, const double* d_frame,
                                 int frame_rows, int frame_cols, double* d_out, void* stream,
                                 tqsb_report* rep) {
    if (!p || !d_frame || !d_out) return set_error(TQSB_EINVAL, "null argument");
    tqsb_config c;
    TQSB_TRY(call_config(p, call, &c));
    Geometry g;
    TQSB_TRY(geometry(c, frame_rows, frame_cols, &g));
    return device_band(p, call, d_frame, frame_rows, frame_cols, 0, g.padM / g.B, d_out, stream, rep);
}

int tqsb_reconstruct_band_device(tqsb_plan* p, const double* d_frame, int frame_rows,
                                 int frame_cols, int br0, int br1, double* d_out, void* stream,
                                 tqsb_report* rep) {
    if (!p || !d_frame || !d_out) return set_error(TQSB_EINVAL, "null argument");
    return device_band(p, nullptr, d_frame, frame_rows, frame_cols, br0, br1, d_out, stream, rep);
}

int tqsb_plan_export_tables(tqsb_plan* p, int orow, int ocol, int* local_out, double* b_re,
                            double* b_im, double* c_re, double* c_im, double* dd) {
    if (!p || !local_out) return set_error(TQSB_EINVAL, "null argument");
    if (orow < 0 || ocol < 0) return set_error(TQSB_EINVAL, "window origin must be non-negative");
    std::lock_guard<std::mutex> lk(p->mu);
    Device* d = p->devs[0].get();
    const int key = (orow % p->period) * p->period + (ocol % p->period);
    std::map<int, std::pair<int, int>> rep{{key, {orow, ocol}}};
    int created = 0, launches = 0;
    TQSB_TRY(ensure_classes(p, d, p->cfg, {key}, rep, &created, &launches));
    const ClassTab& t = d->tabs[d->slot_of.at(key)];
    *local_out = t.local;
    if (!b_re) return TQSB_OK;
    const size_t K = p->wt.K, L = t.local;
    std::vector<double> b(K * L * 2), c(K * K * 2);
    CUDA_TRY(cudaSetDevice(d->id));
    CUDA_TRY(cudaMemcpy(b.data(), t.b64, sizeof(double) * b.size(), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(c.data(), t.c64, sizeof(double) * c.size(), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(dd, t.d64, sizeof(double) * K, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < K * L; ++i) {
        b_re[i] = b[2 * i];
        b_im[i] = b[2 * i + 1];
    }
    for (size_t i = 0; i < K * K; ++i) {
        c_re[i] = c[2 * i];
        c_im[i] = c[2 * i + 1];
    }
    return TQSB_OK;
}

// ---------------------------------------------------------------------------
// TQSK table persistence (rljsde.cpp:337-475): header (window, period, precision,
// spatial decay, frequency exponent, pattern digest, class count) then, per class in
// (row, col) order, (row, col, L) and the planes bRe, bIm [k*L+m], cRe, cIm
// [uk*K+sk], d in the header's precision. Files written here load in the reference
// and vice versa; loading skips the fp64 precompute (K1) and derives only the fp32
// product tables on the device.
// ---------------------------------------------------------------------------
uint64_t tqsb_pattern_digest(const uint8_t* opaque, int period) {
    uint64_t h = 14695981039346656037ull;  // FNV-1a over period (LE bytes) then quadrants
    auto mix = [&h](uint8_t x) {
        h ^= x;
        h *= 1099511628211ull;
    };
    for (int i = 0; i < 4; ++i) mix(uint8_t(uint32_t(period) >> (8 * i)));
    if (opaque && period >= 2)
        for (int i = 0; i < (period / 2) * (period / 2); ++i) mix(opaque[i]);
    return h;
}

int tqsb_kernel_memory_report(int classes, int window, int precision, int local, uint64_t out[4]) {
    if (!out) return set_error(TQSB_EINVAL, "null argument");
    if (classes < 0 || window <= 0)
        return set_error(TQSB_EINVAL, "kernel_memory_report: invalid shape");
    const uint64_t K = uint64_t(window) * window, L = local < 0 ? K / 4 : uint64_t(local);
    const uint64_t cb = precision == TQSB_PRECISION_SINGLE ? 8 : 16;  // bytes per complex
    out[0] = uint64_t(classes) * L * K * cb;
    out[1] = uint64_t(classes) * K * K * cb;
    out[2] = uint64_t(classes) * K * cb;  // D counted as complex, like the reference
    out[3] = out[0] + out[1] + out[2];
    return TQSB_OK;
}

namespace {

struct TqskWriter {
    std::FILE* f;
    bool ok = true;
    void raw(const void* p, size_t n) { ok = ok && std::fwrite(p, 1, n, f) == n; }
    void u32(uint32_t v) {
        unsigned char b[4];
        for (int i = 0; i < 4; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
        raw(b, 4);
    }
    void u64(uint64_t v) {
        unsigned char b[8];
        for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
        raw(b, 8);
    }
    void f64(double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        u64(u);
    }
    // one plane: component `comp` of an interleaved complex array (comp < 0: real array)
    void plane(const double* v, size_t n, int comp, bool single) {
        std::vector<unsigned char> buf(n * (single ? 4 : 8));
        for (size_t i = 0; i < n; ++i) {
            const double x = comp < 0 ? v[i] : v[2 * i + comp];
            if (single) {
                const float y = float(x);
                uint32_t u;
                std::memcpy(&u, &y, 4);
                for (int k = 0; k < 4; ++k) buf[4 * i + k] = static_cast<unsigned char>(u >> (8 * k));
            } else {
                uint64_t u;
                std::memcpy(&u, &x, 8);
                for (int k = 0; k < 8; ++k) buf[8 * i + k] = static_cast<unsigned char>(u >> (8 * k));
            }
        }
        raw(buf.data(), buf.size());
    }
};

struct TqskReader {
    std::FILE* f;
    bool ok = true;
    void raw(void* p, size_t n) { ok = ok && std::fread(p, 1, n, f) == n; }
    uint64_t le(int n) {
        unsigned char b[8] = {};
        raw(b, size_t(n));
        uint64_t v = 0;
        for (int i = 0; i < n; ++i) v |= uint64_t(b[i]) << (8 * i);
        return v;
    }
    double f64() {
        const uint64_t u = le(8);
        double v;
        std::memcpy(&v, &u, 8);
        return v;
    }
    // a plane of n values into component `comp` of interleaved `v` (comp < 0: real)
    void plane(double* v, size_t n, int comp, bool single) {
        std::vector<unsigned char> buf(n * (single ? 4 : 8));
        raw(buf.data(), buf.size());
        if (!ok) return;
        for (size_t i = 0; i < n; ++i) {
            double x;
            if (single) {
                uint32_t u = 0;
                for (int k = 0; k < 4; ++k) u |= uint32_t(buf[4 * i + k]) << (8 * k);
                float y;
                std::memcpy(&y, &u, 4);
                x = y;
            } else {
                uint64_t u = 0;
                for (int k = 0; k < 8; ++k) u |= uint64_t(buf[8 * i + k]) << (8 * k);
                std::memcpy(&x, &u, 8);
            }
            (comp < 0 ? v[i] : v[2 * i + comp]) = x;
        }
    }
};

}  // namespace

int tqsb_plan_save_tables(tqsb_plan* p, const char* path, int* classes_out) {
    if (!p || !path) return set_error(TQSB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(p->mu);
    const std::string where(path);
    // every resident class (union over devices, first holder wins), in key order
    std::map<int, std::pair<Device*, int>> owner;
    for (auto& dp : p->devs)
        for (const auto& [key, slot] : dp->slot_of) owner.emplace(key, std::make_pair(dp.get(), slot));
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return set_error(TQSB_EIO, where + ": cannot open for writing");
    TqskWriter w{f};
    const bool single = p->cfg.precision == TQSB_PRECISION_SINGLE;
    w.raw("TQSK", 4);
    w.u32(uint32_t(p->cfg.window));
    w.u32(uint32_t(p->period));
    w.u32(single ? 0u : 1u);
    w.f64(p->cfg.spatial_decay);
    w.f64(p->cfg.frequency_exponent);
    w.u64(tqsb_pattern_digest(p->opaque.data(), p->period));
    w.u32(uint32_t(owner.size()));
    const size_t K = p->wt.K;
    std::vector<double> b, c, dv(K);
    for (const auto& [key, hold] : owner) {
        Device* d = hold.first;
        const ClassTab& t = d->tabs[hold.second];
        const size_t L = size_t(t.local);
        b.resize(K * L * 2);
        c.resize(K * K * 2);
        if (cudaSetDevice(d->id) != cudaSuccess ||
            cudaMemcpy(b.data(), t.b64, sizeof(double) * b.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(c.data(), t.c64, sizeof(double) * c.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(dv.data(), t.d64, sizeof(double) * K, cudaMemcpyDeviceToHost) != cudaSuccess) {
            std::fclose(f);
            return set_error(TQSB_ECUDA, where + ": table download failed");
        }
        w.u32(uint32_t(key / p->period));
        w.u32(uint32_t(key % p->period));
        w.u32(uint32_t(L));
        w.plane(b.data(), K * L, 0, single);
        w.plane(b.data(), K * L, 1, single);
        w.plane(c.data(), K * K, 0, single);
        w.plane(c.data(), K * K, 1, single);
        w.plane(dv.data(), K, -1, single);
    }
    const bool closed = std::fclose(f) == 0;
    if (!w.ok || !closed) return set_error(TQSB_EIO, where + ": write failed");
    if (classes_out) *classes_out = int(owner.size());
    return TQSB_OK;
}

int tqsb_plan_load_tables(tqsb_plan* p, const char* path, int* classes_out) {
    if (!p || !path) return set_error(TQSB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(p->mu);
    const std::string where(path);
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return set_error(TQSB_EIO, where + ": cannot open for reading");
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
    TqskReader r{f};
    char magic[4] = {};
    r.raw(magic, 4);
    if (!r.ok || std::memcmp(magic, "TQSK", 4) != 0)
        return set_error(TQSB_EIO, where + ": not a TQSK kernel cache");
    const int window = int(r.le(4)), period = int(r.le(4));
    const bool single = r.le(4) == 0;
    const double decay = r.f64(), expo = r.f64();
    const uint64_t digest = r.le(8);
    const uint32_t n = uint32_t(r.le(4));
    if (!r.ok) return set_error(TQSB_EIO, where + ": truncated header");
    const bool plan_single = p->cfg.precision == TQSB_PRECISION_SINGLE;
    if (window != p->cfg.window || period != p->period || single != plan_single ||
        digest != tqsb_pattern_digest(p->opaque.data(), p->period) ||
        decay != p->cfg.spatial_decay || expo != p->cfg.frequency_exponent)
        return set_error(TQSB_EIO, where + ": kernel cache does not match the current configuration");
    const size_t K = size_t(window) * window;
    int installed = 0;
    std::vector<double> b, c, dv(K);
    for (uint32_t i = 0; i < n; ++i) {
        const int row = int(r.le(4)), col = int(r.le(4));
        const size_t L = size_t(r.le(4));
        if (!r.ok || L > K || row < 0 || col < 0 || row >= period || col >= period)
            return set_error(TQSB_EIO, where + ": corrupt class record");
        b.assign(K * L * 2, 0.0);
        c.assign(K * K * 2, 0.0);
        r.plane(b.data(), K * L, 0, single);
        r.plane(b.data(), K * L, 1, single);
        r.plane(c.data(), K * K, 0, single);
        r.plane(c.data(), K * K, 1, single);
        r.plane(dv.data(), K, -1, single);
        if (!r.ok) return set_error(TQSB_EIO, where + ": truncated class payload");
        const int key = row * period + col;
        if (local_system(p->opaque, period, row, col, p->cfg).L != int(L))
            return set_error(TQSB_EIO, where + ": corrupt class record");
        for (auto& dp : p->devs) {
            Device* d = dp.get();
            if (d->slot_of.count(key)) continue;  // already resident: the first insert wins
            CUDA_TRY(cudaSetDevice(d->id));
            ClassBuild cb;
            TQSB_TRY(alloc_class(p, d, p->cfg, key, row, col, &cb));
            CUDA_TRY(cudaMemcpyAsync(cb.b64, b.data(), sizeof(double) * b.size(),
                                     cudaMemcpyHostToDevice, d->stream));
            CUDA_TRY(cudaMemcpyAsync(cb.c64, c.data(), sizeof(double) * c.size(),
                                     cudaMemcpyHostToDevice, d->stream));
            CUDA_TRY(cudaMemcpyAsync(cb.d64, dv.data(), sizeof(double) * K, cudaMemcpyHostToDevice,
                                     d->stream));
            // the planes are the cache; the fp32 product tables are derived on first use;
            // the transposed B of the batched L-JSDE kernel is rebuilt from the loaded B
            int launches = 0;
            const int rc = launch_tables_transpose(&cb, 1, window, cb.local, d->stream, &launches);
            if (rc != 0)
                return set_error(TQSB_ECUDA, std::string("table transpose: ") +
                                                 cudaGetErrorString(cudaError_t(rc)));
            CUDA_TRY(cudaStreamSynchronize(d->stream));  // b/c/dv are reused next record
        }
        ++installed;
    }
    if (classes_out) *classes_out = installed;
    return TQSB_OK;
}

int tqsb_plan_block_trace(tqsb_plan* p, int orow, int ocol, const double* y_local, int* picks,
                          double* gd, double* window_out, int* n_out) {
    if (!p || !y_local || !picks || !gd || !n_out) return set_error(TQSB_EINVAL, "null argument");
    if (orow < 0 || ocol < 0) return set_error(TQSB_EINVAL, "window origin must be non-negative");
    std::lock_guard<std::mutex> lk(p->mu);
    Device* d = p->devs[0].get();
    const int W = p->cfg.window, B = p->cfg.block;
    const int key = (orow % p->period) * p->period + (ocol % p->period);
    std::map<int, std::pair<int, int>> rep{{key, {orow, ocol}}};
    int created = 0, launches = 0;
    Derived* dv = nullptr;
    TQSB_TRY(ensure_classes(p, d, p->cfg, {key}, rep, &created, &launches));
    TQSB_TRY(ensure_derived(p, d, p->cfg, &dv, &launches));
    // a frame holding y_local at the window's cells (gather_local_values order)
    const int r0 = (orow + 1) / 2, r1 = (orow + W - 2) / 2;
    const int c0 = (ocol + 1) / 2, c1 = (ocol + W - 2) / 2;
    const int fr = (orow + W) / 2 + 1, fc = (ocol + W) / 2 + 1;
    std::vector<double> frame(size_t(fr) * fc, 0.0);
    int m = 0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) frame[size_t(r) * fc + c] = y_local[m++];
    const int lead = (W - B) / 2;
    Task t{orow + lead, ocol + lead, orow, ocol};
    WorkItem wi{d->slot_of.at(key), 0, 1, 0};
    const int iters = std::max(1, p->cfg.max_iterations);
    CUDA_TRY(cudaSetDevice(d->id));
    char* buf = nullptr;
    const size_t out_n = size_t(B) * (t.block_col + B);
    const size_t bytes = sizeof(double) * frame.size() + sizeof(double) * out_n + sizeof(Task) +
                         sizeof(WorkItem) + sizeof(int) * iters + sizeof(double) * 2 * iters +
                         sizeof(double) * W * W + sizeof(int) + 1024;
    CUDA_TRY(cudaMalloc(&buf, bytes));
    size_t off = 0;
    auto take = [&](size_t n) {
        char* q = buf + off;
        off = align_up(off + n, 64);
        return q;
    };
    double* d_frame = reinterpret_cast<double*>(take(sizeof(double) * frame.size()));
    double* d_out = reinterpret_cast<double*>(take(sizeof(double) * out_n));
    Task* d_task = reinterpret_cast<Task*>(take(sizeof(Task)));
    WorkItem* d_item = reinterpret_cast<WorkItem*>(take(sizeof(WorkItem)));
    int* d_picks = reinterpret_cast<int*>(take(sizeof(int) * iters));
    double* d_gd = reinterpret_cast<double*>(take(sizeof(double) * 2 * iters));
    double* d_win = reinterpret_cast<double*>(take(sizeof(double) * W * W));
    int* d_n = reinterpret_cast<int*>(take(sizeof(int)));
    cudaMemcpy(d_frame, frame.data(), sizeof(double) * frame.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_task, &t, sizeof(Task), cudaMemcpyHostToDevice);
    cudaMemcpy(d_item, &wi, sizeof(WorkItem), cudaMemcpyHostToDevice);
    cudaMemset(d_n, 0, sizeof(int));
    SolveArgs a = base_args(p, d, p->cfg, dv);
    a.frame = d_frame;
    a.frame_rows = fr;
    a.frame_cols = fc;
    a.frame_row0 = 0;
    a.frame_pitch = fc;
    a.out = d_out;
    a.out_row0 = t.block_row;
    a.out_rows = t.block_row + B;
    a.out_cols = t.block_col + B;
    a.tasks = d_task;
    a.items = d_item;
    a.n_items = 1;
    a.n_tasks = 1;
    a.task_cls = nullptr;  // the single item's class
    a.trace_picks = d_picks;
    a.trace_gd = d_gd;
    a.trace_window = window_out ? d_win : nullptr;
    a.trace_n = d_n;
    int rc = launch(p->cfg, d, a, d->stream, p->wt.NS);
    if (rc) {
        cudaFree(buf);
        return rc;
    }
    cudaError_t e = cudaStreamSynchronize(d->stream);
    if (e != cudaSuccess) {
        cudaFree(buf);
        return set_error(TQSB_ECUDA, std::string("trace: ") + cudaGetErrorString(e));
    }
    int n = 0;
    cudaMemcpy(&n, d_n, sizeof(int), cudaMemcpyDeviceToHost);
    *n_out = n;
    cudaMemcpy(picks, d_picks, sizeof(int) * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(gd, d_gd, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost);
    if (window_out) cudaMemcpy(window_out, d_win, sizeof(double) * W * W, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    return TQSB_OK;
}

// ---------------------------------------------------------------------------
// host helpers: input side and test support
// ---------------------------------------------------------------------------
int tqsb_generate_pattern(uint64_t seed, int period, int block, uint8_t* opaque_out) {
    if (!opaque_out) return set_error(TQSB_EINVAL, "null argument");
    if (period < 4 || period % 2 != 0)
        return set_error(TQSB_EINVAL, "pattern period must be even and >= 4");
    if (block < 1 || period % block != 0)
        return set_error(TQSB_EINVAL, "pattern period must be divisible by the target block size");
    std::mt19937_64 gen(seed);
    const size_t n = size_t(period / 2) * (period / 2);
    for (size_t i = 0; i < n; ++i) opaque_out[i] = static_cast<uint8_t>(gen() & 3u);
    return TQSB_OK;
}

int tqsb_simulate(const double* image, int rows, int cols, const uint8_t* opaque, int period,
                  double* frame_out) {
    if (!image || !opaque || !frame_out) return set_error(TQSB_EINVAL, "null argument");
    if (rows % 2 != 0 || cols % 2 != 0) return set_error(TQSB_EINVAL, "image dimensions must be even");
    if (period <= 0) return set_error(TQSB_EINVAL, "invalid pattern");
    const int pc = period / 2, fr = rows / 2, fc = cols / 2;
    const double third = 1.0 / 3.0;
    for (int r = 0; r < fr; ++r)
        for (int c = 0; c < fc; ++c) {
            const int q = opaque[size_t(r % pc) * pc + c % pc];
            double acc = 0.0;
            for (int quad = 0; quad < 4; ++quad)
                if (quad != q)
                    acc += third * image[size_t(2 * r + quad / 2) * cols + 2 * c + quad % 2];
            frame_out[size_t(r) * fc + c] = acc;
        }
    return TQSB_OK;
}

// Smooth synthetic test scene: linear ramp + 6 plane waves + 5 Gaussian bumps +
// 2 logistic edges, rescaled to [0.02, 0.98]; parameters drawn in that order from
// mt19937_64(seed) through uniform_real_distribution(0,1)
// (the generator of tests/support/synthetic.cpp:9-80).
int tqsb_synthetic_image(int rows, int cols, uint64_t seed, double* out) {
    if (!out || rows < 1 || cols < 1) return set_error(TQSB_EINVAL, "invalid image shape");
    const SceneParams sp = scene_params(rows, cols, seed);
    const double two_pi = 6.283185307179586;
    double vmin = 1e300, vmax = -1e300;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            double v = sp.ramp_r * r / rows + sp.ramp_c * c / cols;
            for (const auto& wv : sp.wave) v += wv[3] * std::sin(two_pi * (wv[0] * r + wv[1] * c) + wv[2]);
            for (const auto& bp : sp.bump) {
                const double dy = r - bp[0], dx = c - bp[1];
                v += bp[3] * std::exp(-(dy * dy + dx * dx) / (2.0 * bp[2] * bp[2]));
            }
            for (const auto& ed : sp.edge)
                v += ed[3] / (1.0 + std::exp(-(ed[0] * r + ed[1] * c - ed[2]) / 2.5));
            out[size_t(r) * cols + c] = v;
            vmin = std::min(vmin, v);
            vmax = std::max(vmax, v);
        }
    const double span = vmax > vmin ? vmax - vmin : 1.0;
    for (size_t i = 0; i < size_t(rows) * cols; ++i) out[i] = 0.02 + 0.96 * (out[i] - vmin) / span;
    return TQSB_OK;
}

int tqsb_synthetic_image_device(int device, int rows, int cols, uint64_t seed, double* d_out,
                                void* stream) {
    if (!d_out || rows < 1 || cols < 1) return set_error(TQSB_EINVAL, "invalid image shape");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
        return set_error(TQSB_ENODEV, "no CUDA device (the library has no CPU fallback)");
    CUDA_TRY(cudaSetDevice(device));
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int max_parts = 4 * sms;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* parts = nullptr;
    CUDA_TRY(cudaMallocAsync(&parts, sizeof(double) * 2 * max_parts, s));
    const int rc = launch_scene(scene_params(rows, cols, seed), rows, cols, d_out, parts, max_parts,
                                stream, sms);
    CUDA_TRY(cudaFreeAsync(parts, s));
    if (rc != 0) return set_error(TQSB_ECUDA, std::string("scene: ") + cudaGetErrorString(cudaError_t(rc)));
    return TQSB_OK;
}

int tqsb_plan_simulate_device(tqsb_plan* p, const double* d_image, int rows, int cols,
                              double* d_frame, void* stream) {
    if (!p || !d_image || !d_frame) return set_error(TQSB_EINVAL, "null argument");
    if (rows < 2 || cols < 2 || rows % 2 != 0 || cols % 2 != 0)
        return set_error(TQSB_EINVAL, "image dimensions must be even");
    Device* d = p->devs[0].get();
    CUDA_TRY(cudaSetDevice(d->id));
    const int rc = launch_simulate(d_image, rows, cols, d->d_opaque, p->period, d_frame, stream,
                                   d->num_sms);
    if (rc != 0)
        return set_error(TQSB_ECUDA, std::string("simulate: ") + cudaGetErrorString(cudaError_t(rc)));
    return TQSB_OK;
}

double tqsb_psnr(const double* reference, const double* estimate, long long n) {
    if (!reference || !estimate || n <= 0) return std::numeric_limits<double>::quiet_NaN();
    return psnr_impl(reference, estimate, n);
}

void* tqsb_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
        set_error(TQSB_ENOMEM, "cudaHostAlloc failed");
        return nullptr;
    }
    return p;
}

void tqsb_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int tqsb_probe_peaks(int device, double* fp32_tflops, double* smem_tbps) {
    if (tqsb_device_count() < 1) return set_error(TQSB_ENODEV, "no CUDA device available");
    const int rc = probe_peaks(device, fp32_tflops, smem_tbps);
    if (rc) return set_error(TQSB_ECUDA, cudaGetErrorString(cudaError_t(rc)));
    return TQSB_OK;
}

} // extern "C"

// error reporting shared with io.cpp / tqsk handling (same thread-local message)
int tqsb_internal_set_error(int code, const std::string& msg) { return set_error(code, msg); }

namespace tqsb {
// synthetic.cpp:9-30 -- the scene's random parameters, in the reference's draw order
SceneParams scene_params(int rows, int cols, uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    const double two_pi = 6.283185307179586;
    SceneParams sp{};
    sp.ramp_r = U(gen) * 2.0 - 1.0;
    sp.ramp_c = U(gen) * 2.0 - 1.0;
    for (auto& wv : sp.wave) {
        wv[0] = (U(gen) * 6.0 + 0.5) / rows;
        wv[1] = (U(gen) * 6.0 + 0.5) / cols;
        wv[2] = U(gen) * two_pi;
        wv[3] = U(gen) * 0.5 + 0.1;
    }
    const double short_side = std::min(rows, cols);
    for (auto& bp : sp.bump) {
        bp[0] = U(gen) * rows;
        bp[1] = U(gen) * cols;
        bp[2] = (U(gen) * 0.12 + 0.04) * short_side;
        bp[3] = (U(gen) * 2.0 - 1.0) * 0.8;
    }
    for (auto& ed : sp.edge) {
        const double theta = U(gen) * two_pi;
        ed[0] = std::sin(theta);
        ed[1] = std::cos(theta);
        ed[2] = U(gen) * (rows + cols) * 0.5;
        ed[3] = (U(gen) * 2.0 - 1.0) * 0.6;
    }
    return sp;
}
}  // namespace tqsb
