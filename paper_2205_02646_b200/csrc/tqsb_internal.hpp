// tqsb_internal.hpp -- shared between the host orchestration (plan.cpp) and the
// CUDA translation units (tables.cu, solve_f32.cu, solve_f64.cu). No CUDA types
// here so plan.cpp compiles with plain g++.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdlib>

namespace tqsb {

constexpr int kMaxWindowF32 = 32;  // fp32 product kernel: a warp-row per window row/col;
                                  // larger windows run on the generic fp64 kernel
#ifndef TQSB_WARPS_F32
#define TQSB_WARPS_F32 16
#endif
constexpr int kWarpsF32 = TQSB_WARPS_F32;  // warps per CTA of the fp32 solve kernel (1 CTA/SM)
constexpr int kWarpsF32Heavy = 12;  // ... for its register-heavy instantiations (solve_f32.cu)
constexpr int kWarpsF64 = 4;    // warps per CTA of the fp64 parity kernel
constexpr int kSbufStride = 36; // floats per lane in the element-score buffer (conflict-free STS.128)

// One target block: top-left output pixel and clamped window origin
// (BlockTask, pipeline.cpp:54-58), plus its class slot in the plan.
struct Task {
    int block_row, block_col, origin_row, origin_col;
};

// A run of consecutive class-sorted tasks handled by one CTA pass.
struct WorkItem {
    int cls;    // class slot (index into the ClassTab array)
    int start;  // first task
    int count;  // number of tasks
    int pad;
};

// Device-resident tables of one offset class (the KernelSet analogue,
// rljsde.hpp:34-52), all pointers into device memory of one GPU.
struct ClassTab {
    // fp32 product tables (rank order)
    const float* cpack;   // K_pad columns x (K_pad/2) float4: C'[s,u] = s_s * C[s,u]
    const float* scale;   // K_pad: s_r = sqrt(q/D) (NaN where D <= 0 or padding)
    const float* fac;     // K_pad: gamma / (s_u * D_u)
    const float* mask32;  // W*W: w_m/3 at transparent pixels of included cells, else 0
    // fp64 parity tables (reference order)
    const double* b64;    // K*L complex interleaved, k-major [k*L+m]
    const double* c64;    // K*K complex interleaved, column-major [uk*K+sk]
    const double* d64;    // K
    const int* cells;     // L x (cell frame row offset, cell frame col offset) vs window origin
    const double* w64;    // L spatial weights (basis.cpp:75-88; L-JSDE residual update)
    const double* bt64;   // L*K complex interleaved, m-major [m*K+k]: B transposed for the
                          // batched L-JSDE kernel (stored in the build's T scratch)
    int local;            // L
    int pad;
};

// Per-window constants (class independent), device pointers.
struct WindowConsts {
    const int* perm;       // K_pad: rank -> flat k (or -1 for padding ranks)
    const int* src;        // K_pad: rank -> half-spectrum buffer index, bit 30 = conjugate
    const float* unit32;   // 2*W: (cos, sin) of 2*pi*k/W, the FourierTable (basis.cpp:15-26)
    const double* unit64;  // 2*W
    const double* q64;     // K: frequency_weights (basis.cpp:99-106)
};

struct SolveArgs {
    const double* frame;   // device frame (full frame, or a row band starting at frame_row0)
    int frame_rows;        // rows of the UNPADDED full frame (clamping implements pad_frame)
    int frame_cols;
    int frame_row0;        // first frame row held at frame[0]
    int frame_pitch;       // elements per frame row in the buffer
    double* out;           // output rows starting at out_row0
    int out_row0;
    int out_rows;          // rows of the unpadded output image (M); crop beyond
    int out_cols;          // N (also the pitch)
    const Task* tasks;
    const WorkItem* items;
    int n_items;
    const int* task_cls;   // class slot per task (warp-level dynamic scheduling)
    int n_tasks;
    int* counter;          // next task (zeroed before each launch)
    const ClassTab* tabs;
    WindowConsts wc;
    int window, block, iterations;
    double step;
    int clip;
    int hot;               // C' columns in the TMEM tier (fp32)
    int early_stop;        // L-JSDE energy stop (ljsde.cpp:178-183)
    double early_stop_scale;
    // tracing (single-block diagnostics): when trace_picks != nullptr, block 0
    // records picks (flat k), gd (re,im) and the full window synthesis.
    int* trace_picks;
    double* trace_gd;
    double* trace_window;
    int* trace_n;
    // streamed completion (fp32 kernel, warp-level scheduling): when non-null, task_cls
    // entries carry a chunk index above kTaskClsBits and every finished block bumps
    // progress[chunk] (device memory, release at GPU scope after the block's output
    // stores), which a copy stream waits on (cuStreamWaitValue32) to move finished
    // output rows to the host while the kernel runs
    int* progress;
};
constexpr int kTaskClsBits = 20;  // task_cls = class slot | chunk << kTaskClsBits
// the fp32 kernel has a streamed instantiation for NS == 16 slots (W = 23..32) and
// B*B <= 32 kept pixels (B <= 5): the product configurations
constexpr bool solve_f32_streams(int n_slots, int block_px) { return n_slots == 16 && block_px <= 32; }

// test hook (env TQSB_FORCE_GLOBAL_STATE=1): the fp64 / L-JSDE kernels keep their
// per-block state in global memory even when it fits in shared memory, so the
// large-window path (W >= 68) is exercised at sizes the CPU reference finishes quickly
inline bool force_global_state() {
    const char* v = std::getenv("TQSB_FORCE_GLOBAL_STATE");
    return v && v[0] == '1';
}

// ---- launchers (defined in the .cu files); return cudaError_t as int ----
int launch_solve_f32(const SolveArgs& a, int n_slots, void* stream, int num_sms);
int launch_solve_f64(const SolveArgs& a, void* stream, int num_sms);
int launch_solve_f64r(const SolveArgs& a, void* stream, int num_sms);  // register-resident, W <= 32
int launch_solve_ljsde(const SolveArgs& a, void* stream, int num_sms);
int solve_f32_max_hot(int n_slots, int device);

// Per-class build descriptor for the batched table kernels (tables.cu).
struct ClassBuild {
    int local;                 // L
    const short* px;           // L*6: (eta, gamma) of the 3 transparent pixels per cell
    const double* w;           // L spatial weights (host-computed, basis.cpp:75-88)
    double* t64;               // K*L*2 (re, im interleaved), k-major
    double* b64;               // K*L*2
    double* c64;               // K*K*2, column-major [uk*K+sk]
    double* d64;               // K
    float* cpack;              // K_pad * K_pad/2 * 4 (null: fp64-only plan)
    float* scale;              // K_pad
    float* fac;                // K_pad
};
// fp64 planes (t64, b64, c64, d64) of n classes; round_single stores B, C, D rounded
// to float (the reference's Precision::Single).
int launch_tables_build(const void* host_descs, int n, int window, const double* unit64,
                        int max_local, void* stream, int* launches, int round_single);
// B transposed to m-major into the (then dead) T scratch of n classes (the batched L-JSDE
// kernel's coalesced layout); part of launch_tables_build, separately after a TQSK load
int launch_tables_transpose(const void* host_descs, int n, int window, int max_local, void* stream,
                            int* launches);
// fp32 product tables (scale, fac, cpack) of n classes from their resident fp64
// planes, for one (q = frequency weights, step width gamma).
int launch_tables_derive(const void* host_descs, int n, int window, int k_pad, double step,
                         const double* q64, const int* perm, void* stream, int* launches);

int probe_peaks(int device, double* fp32_tflops, double* smem_tbps);

// synthetic scene parameters (tests/support/synthetic.cpp:9-80), drawn on the host
struct SceneParams {
    double ramp_r, ramp_c;
    double wave[6][4];  // fr, fc, phase, amp
    double bump[5][4];  // r, c, radius, amp
    double edge[2][4];  // nr, nc, offset, amp
};
SceneParams scene_params(int rows, int cols, uint64_t seed);  // plan.cpp

// sensor.cu: device readout and scene generation (grid-stride, HBM-bound)
int launch_simulate(const double* d_img, int rows, int cols, const uint8_t* d_opaque, int period,
                    double* d_frame, void* stream, int num_sms);
int launch_scene(const SceneParams& sp, int rows, int cols, double* d_out, double* d_parts,
                 int max_parts, void* stream, int num_sms);

} // namespace tqsb
