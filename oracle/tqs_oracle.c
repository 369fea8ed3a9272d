/* oracle/tqs_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's RL-JSDE reconstruction path, used as the CPU checker for the CUDA
 * product path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it (built by oracle/Makefile into oracle/liboracle.so).
 *
 * Parity pin: every function below is checked against the unmodified reference
 * library (oracle/_ref, built from /root/reference/proj by oracle/build_ref.sh)
 * in tests/test_oracle.py and against the committed fixtures in tests/golden/
 * (made by tests/golden/make_golden.py from oracle/_ref). Citations are
 * /root/reference/proj/<file>:<line>.
 *
 * Arithmetic follows the reference's operation order term by term so that, at
 * the same compiler contraction setting, results are bitwise equal; the tests
 * state the tolerance they actually rely on.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* mt19937_64 (the published Matsumoto-Nishimura 64-bit generator; the        */
/* reference uses std::mt19937_64, grid.cpp:20-23, synthetic.cpp:10).         */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} or_mt64;

void or_mt64_seed(or_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t or_mt64_next(or_mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* std::uniform_real_distribution<double>(0,1) over mt19937_64 as libstdc++
 * evaluates it (generate_canonical with one 64-bit draw: x / 2^64, clamped
 * below 1), the generator behind synthetic.cpp:11. */
double or_uniform01(or_mt64* g) {
    double r = (double)or_mt64_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

/* ------------------------------------------------------------------------- */
/* Patterns, measurement, local systems (grid.hpp / grid.cpp)                */
/* ------------------------------------------------------------------------- */

/* generate_pattern, grid.cpp:8-26: low two bits of each draw, row-major over
 * the (P/2)^2 tile. Returns -1 on the reference's invalid_argument cases. */
int or_generate_pattern(uint64_t seed, int period, int block, uint8_t* opaque) {
    if (period < 4 || period % 2 != 0) return -1;
    if (block < 1 || period % block != 0) return -1;
    or_mt64 g;
    or_mt64_seed(&g, seed);
    const int pc = period / 2;
    for (int i = 0; i < pc * pc; ++i) opaque[i] = (uint8_t)(or_mt64_next(&g) & 3u);
    return 0;
}

/* QuadrantPattern::quadrant, grid.hpp:28-33 */
static uint8_t quadrant(const uint8_t* opaque, int period, long r, long c) {
    const int pc = period / 2;
    const long rr = ((r % pc) + pc) % pc, cc = ((c % pc) + pc) % pc;
    return opaque[rr * pc + cc];
}

/* transparent_offsets, grid.cpp:31-42: the three open quadrants, row-major */
static void transparent_offsets(uint8_t opq, int off[3][2]) {
    int n = 0;
    for (int dr = 0; dr < 2; ++dr)
        for (int dc = 0; dc < 2; ++dc) {
            if (dr * 2 + dc == opq) continue;
            off[n][0] = dr;
            off[n][1] = dc;
            ++n;
        }
}

/* simulate_measurement, grid.cpp:46-66 */
int or_simulate(const double* image, int rows, int cols, const uint8_t* opaque, int period,
                double* frame) {
    if (rows % 2 || cols % 2) return -1;
    const double third = 1.0 / 3.0;
    const int fr = rows / 2, fc = cols / 2;
    for (int r = 0; r < fr; ++r)
        for (int c = 0; c < fc; ++c) {
            int off[3][2];
            transparent_offsets(quadrant(opaque, period, r, c), off);
            double y = 0.0;
            for (int t = 0; t < 3; ++t)
                y += third * image[(size_t)(2 * r + off[t][0]) * cols + 2 * c + off[t][1]];
            frame[(size_t)r * fc + c] = y;
        }
    return 0;
}

/* first/last fully contained cell, grid.cpp:70-71 */
static int first_full_cell(int o) { return (o + 1) / 2; }
static int last_full_cell(int o, int w) { return (o + w - 2) / 2; }

/* extract_local_matrix, grid.cpp:75-102: per included cell m (row-major) the
 * cell's local top-left (cellEta, cellGamma) and its 3 transparent pixels.
 * px[m*6 + 2t + {0,1}] = (eta, gamma). Returns L. */
int or_local_matrix(const uint8_t* opaque, int period, int orow, int ocol, int window,
                    int* cell_eta, int* cell_gamma, int* px) {
    const int r0 = first_full_cell(orow), r1 = last_full_cell(orow, window);
    const int c0 = first_full_cell(ocol), c1 = last_full_cell(ocol, window);
    int m = 0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) {
            const int ce = 2 * r - orow, cg = 2 * c - ocol;
            if (cell_eta) {
                int off[3][2];
                transparent_offsets(quadrant(opaque, period, r, c), off);
                cell_eta[m] = ce;
                cell_gamma[m] = cg;
                for (int t = 0; t < 3; ++t) {
                    px[m * 6 + 2 * t] = ce + off[t][0];
                    px[m * 6 + 2 * t + 1] = cg + off[t][1];
                }
            }
            ++m;
        }
    return m;
}

/* gather_local_values, grid.cpp:104-114 */
int or_gather(const double* frame, int frame_cols, int orow, int ocol, int window, double* y) {
    const int r0 = first_full_cell(orow), r1 = last_full_cell(orow, window);
    const int c0 = first_full_cell(ocol), c1 = last_full_cell(ocol, window);
    int m = 0;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) y[m++] = frame[(size_t)r * frame_cols + c];
    return m;
}

/* ------------------------------------------------------------------------- */
/* Basis and weights (basis.cpp)                                             */
/* ------------------------------------------------------------------------- */

/* FourierTable, basis.cpp:15-26: exact +-1 on the axes, upper half the exact
 * conjugate of the lower half. */
void or_unit_table(int window, double* re, double* im) {
    const double pi = 3.14159265358979323846;
    re[0] = 1.0; im[0] = 0.0;
    re[window / 2] = -1.0; im[window / 2] = 0.0;
    for (int k = 1; k < window / 2; ++k) {
        const double a = 2.0 * pi * k / window;
        re[k] = cos(a); im[k] = sin(a);
        re[window - k] = re[k]; im[window - k] = -im[k];
    }
}

/* spatial_weight, basis.cpp:75-80 */
double or_spatial_weight(int cell_eta, int cell_gamma, int window, double decay) {
    const double center = (window - 1) / 2.0;
    const double dr = (cell_eta + 0.5) - center, dc = (cell_gamma + 0.5) - center;
    return pow(decay, sqrt(dr * dr + dc * dc));
}

/* frequency_weights, basis.cpp:90-106 (k = sigma*W + rho) */
void or_frequency_weights(int window, double exponent, double* q) {
    const int half = window / 2;
    const double sqrt2 = 1.41421356237309504880;
    for (int s = 0; s < window; ++s)
        for (int r = 0; r < window; ++r) {
            const int cs = s <= half ? s : window - s, cr = r <= half ? r : window - r;
            const double radius = sqrt((double)cs * cs + (double)cr * cr);
            const double maxr = sqrt2 * half * (1.0 + 1e-6);
            q[s * window + r] = pow(1.0 - radius / maxr, exponent);
        }
}

/* ------------------------------------------------------------------------- */
/* RL-JSDE tables (rljsde.cpp:22-102)                                        */
/* ------------------------------------------------------------------------- */

/* build_transform (rljsde.cpp:22-48) + fill_planes (50-102) for one window
 * origin. B, T: k-major [k*L+m]; C: column-major [uk*K+sk], lower triangle
 * accumulated, upper mirrored as the exact conjugate; D = Re diag C. All
 * outputs double (fp64 accumulation); the reference's Single storage is the
 * float rounding of these (rljsde.cpp:70-73, 90-99). Returns L, or -1. */
int or_tables(const uint8_t* opaque, int period, int orow, int ocol, int window, double decay,
              double* b_re, double* b_im, double* c_re, double* c_im, double* d, double* w_out) {
    const int W = window, K = W * W;
    const int L = or_local_matrix(opaque, period, orow, ocol, W, NULL, NULL, NULL);
    int* ce = malloc(sizeof(int) * L);
    int* cg = malloc(sizeof(int) * L);
    int* px = malloc(sizeof(int) * 6 * L);
    double* ure = malloc(sizeof(double) * W);
    double* uim = malloc(sizeof(double) * W);
    double* w = malloc(sizeof(double) * L);
    double* tre = malloc(sizeof(double) * (size_t)K * L);
    double* tim = malloc(sizeof(double) * (size_t)K * L);
    or_local_matrix(opaque, period, orow, ocol, W, ce, cg, px);
    or_unit_table(W, ure, uim);
    for (int m = 0; m < L; ++m) w[m] = or_spatial_weight(ce[m], cg[m], W, decay);
    const double third = 1.0 / 3.0;
    for (int s = 0; s < W; ++s)
        for (int r = 0; r < W; ++r) {
            const size_t k = (size_t)s * W + r;
            for (int m = 0; m < L; ++m) {
                double re = 0.0, im = 0.0;
                for (int t = 0; t < 3; ++t) {
                    const int idx = (px[m * 6 + 2 * t] * s + px[m * 6 + 2 * t + 1] * r) % W;
                    re += third * ure[idx];
                    im -= third * uim[idx];
                }
                tre[k * L + m] = re;
                tim[k * L + m] = im;
            }
        }
    for (size_t i = 0; i < (size_t)K * L; ++i) {
        b_re[i] = w[i % L] * tre[i];
        b_im[i] = w[i % L] * tim[i];
    }
    for (int uk = 0; uk < K; ++uk) {
        const double* uRe = tre + (size_t)uk * L;
        const double* uIm = tim + (size_t)uk * L;
        for (int sk = uk; sk < K; ++sk) {
            const double* sRe = b_re + (size_t)sk * L;
            const double* sIm = b_im + (size_t)sk * L;
            double ar = 0.0, ai = 0.0;
            for (int m = 0; m < L; ++m) {
                ar += sRe[m] * uRe[m] + sIm[m] * uIm[m];
                ai += sIm[m] * uRe[m] - sRe[m] * uIm[m];
            }
            c_re[(size_t)uk * K + sk] = ar;
            c_im[(size_t)uk * K + sk] = ai;
            if (sk != uk) {
                c_re[(size_t)sk * K + uk] = ar;
                c_im[(size_t)sk * K + uk] = -ai;
            }
        }
        d[uk] = c_re[(size_t)uk * K + uk];
    }
    if (w_out) memcpy(w_out, w, sizeof(double) * L);
    free(ce); free(cg); free(px); free(ure); free(uim); free(w); free(tre); free(tim);
    return L;
}

/* ------------------------------------------------------------------------- */
/* Block solve (rljsde.cpp:122-182) and synthesis (basis.cpp:52-73)          */
/* ------------------------------------------------------------------------- */

/* One RL-JSDE block on fp64 tables. picks/gd (optional) receive the greedy
 * path; win (W*W) the real synthesis over the full window, summed over the
 * active coefficients in first-touch order like synthesize_real. Returns the
 * number of completed iterations. */
int or_block(int window, int L, const double* b_re, const double* b_im, const double* c_re,
             const double* c_im, const double* d, const double* q, const double* y,
             int iterations, double step, int* picks, double* gd, double* win) {
    const int W = window, K = W * W;
    double* RRe = malloc(sizeof(double) * K);
    double* RIm = malloc(sizeof(double) * K);
    double* cre = calloc(K, sizeof(double));
    double* cim = calloc(K, sizeof(double));
    int* active = malloc(sizeof(int) * K);
    uint8_t* touched = calloc(K, 1);
    int nactive = 0, done = 0;
    for (int k = 0; k < K; ++k) { /* init, rljsde.cpp:127-138 */
        double re = 0.0, im = 0.0;
        for (int m = 0; m < L; ++m) {
            re += b_re[(size_t)k * L + m] * y[m];
            im += b_im[(size_t)k * L + m] * y[m];
        }
        RRe[k] = re;
        RIm[k] = im;
    }
    for (int it = 0; it < iterations; ++it) {
        int best = -1; /* selection, rljsde.cpp:144-158; basis.hpp:90-92 */
        double bs = 0.0;
        for (int k = 0; k < K; ++k) {
            if (d[k] <= 0.0) continue;
            const double s = q[k] * (RRe[k] * RRe[k] + RIm[k] * RIm[k]) / d[k];
            if (best < 0 || s > bs) { best = k; bs = s; }
        }
        if (best < 0) break;
        const int u = best; /* update, rljsde.cpp:160-172 */
        const double gr = step * (RRe[u] / d[u]), gi = step * (RIm[u] / d[u]);
        cre[u] += gr;
        cim[u] += gi;
        if (!touched[u]) { touched[u] = 1; active[nactive++] = u; }
        const double* colRe = c_re + (size_t)u * K;
        const double* colIm = c_im + (size_t)u * K;
        for (int s = 0; s < K; ++s) {
            const double cr = colRe[s], ci = colIm[s];
            RRe[s] -= gr * cr - gi * ci;
            RIm[s] -= gr * ci + gi * cr;
        }
        if (picks) picks[it] = u;
        if (gd) { gd[2 * it] = gr; gd[2 * it + 1] = gi; }
        done = it + 1;
    }
    if (win) { /* synthesize_real, basis.cpp:52-73 */
        double ure[256], uim[256];
        or_unit_table(W, ure, uim);
        memset(win, 0, sizeof(double) * K);
        for (int a = 0; a < nactive; ++a) {
            const int f = active[a], s = f / W, r = f % W;
            const double c0 = cre[f], c1 = cim[f];
            for (int e = 0; e < W; ++e)
                for (int g = 0; g < W; ++g) {
                    const int idx = (e * s + g * r) % W;
                    win[e * W + g] += c0 * ure[idx] - c1 * uim[idx];
                }
        }
    }
    free(RRe); free(RIm); free(cre); free(cim); free(active); free(touched);
    return done;
}

/* ------------------------------------------------------------------------- */
/* Orchestration (pipeline.cpp:62-185)                                       */
/* ------------------------------------------------------------------------- */

/* validate_config, pipeline.cpp:27-42 (threads replaced by nothing here) */
int or_validate(int window, int block, int iterations, double step, int period) {
    if (window < 2 || window % 2 != 0) return -1;
    if (block < 1 || window % block != 0) return -1;
    if ((window - block) % 2 != 0) return -1;
    if (period % block != 0) return -1;
    if (iterations < 0) return -1;
    if (step <= 0.0 || step > 1.0) return -1;
    return 0;
}

static int gcd_i(int a, int b) { while (b) { int t = a % b; a = b; b = t; } return a; }
static int lcm_i(int a, int b) { return a / gcd_i(a, b) * b; }
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Block enumeration and class census, pipeline.cpp:84-106 (classes = window
 * origin mod P, rljsde.cpp:12-17). out: [blocks, classesTotal, classesInterior].
 * task (optional, 5 ints per block): blockRow, blockCol, originRow, originCol,
 * interior. Returns 0 or -1. */
int or_census(int frame_rows, int frame_cols, int window, int block, int period, long long* out,
              int* task) {
    const int M = 2 * frame_rows, N = 2 * frame_cols, step = lcm_i(block, 2);
    const int padM = (M + step - 1) / step * step, padN = (N + step - 1) / step * step;
    if (padM < window || padN < window) return -1;
    const int lead = (window - block) / 2;
    uint8_t* all = calloc((size_t)period * period, 1);
    uint8_t* inter = calloc((size_t)period * period, 1);
    long long n = 0, ca = 0, ci = 0;
    for (int br = 0; br + block <= padM; br += block)
        for (int bc = 0; bc + block <= padN; bc += block) {
            const int wr = br - lead, wc = bc - lead;
            const int orr = clampi(wr, 0, padM - window), oc = clampi(wc, 0, padN - window);
            const int interior = orr == wr && oc == wc;
            const int key = (orr % period) * period + (oc % period);
            if (!all[key]) { all[key] = 1; ++ca; }
            if (interior && !inter[key]) { inter[key] = 1; ++ci; }
            if (task) {
                int* t = task + 5 * n;
                t[0] = br; t[1] = bc; t[2] = orr; t[3] = oc; t[4] = interior;
            }
            ++n;
        }
    out[0] = n; out[1] = ca; out[2] = ci;
    free(all); free(inter);
    return 0;
}

/* reconstruct (pipeline.cpp:62-185) for Algorithm::Rljsde, single thread, fp64
 * tables: pad (44-52, 69-82), enumerate (84-106), per-class tables (127-133),
 * per-block solve and B x B placement with optional clip (140-167), crop (170).
 * out: (2*frame_rows) x (2*frame_cols). Returns blocks processed or -1. */
long long or_reconstruct(const double* frame, int frame_rows, int frame_cols,
                         const uint8_t* opaque, int period, int window, int block,
                         int iterations, double step, double decay, double exponent, int clip,
                         double* out) {
    if (or_validate(window, block, iterations, step, period) || frame_rows < 1 || frame_cols < 1)
        return -1;
    const int W = window, K = W * W, B = block;
    const int M = 2 * frame_rows, N = 2 * frame_cols, stp = lcm_i(B, 2);
    const int padM = (M + stp - 1) / stp * stp, padN = (N + stp - 1) / stp * stp;
    if (padM < W || padN < W) return -1;
    const int fr = padM / 2, fc = padN / 2;
    double* pf = malloc(sizeof(double) * (size_t)fr * fc);
    for (int r = 0; r < fr; ++r)
        for (int c = 0; c < fc; ++c) {
            const int sr = r < frame_rows - 1 ? r : frame_rows - 1;
            const int sc = c < frame_cols - 1 ? c : frame_cols - 1;
            pf[(size_t)r * fc + c] = frame[(size_t)sr * frame_cols + sc];
        }
    long long cen[3];
    or_census(fr, fc, W, B, period, cen, NULL);
    const long long nb = cen[0];
    int* task = malloc(sizeof(int) * 5 * (size_t)nb);
    or_census(fr, fc, W, B, period, cen, task);
    double* q = malloc(sizeof(double) * K);
    or_frequency_weights(W, exponent, q);
    const int P2 = period * period;
    double** tabs = calloc((size_t)P2, sizeof(double*));
    int* Ls = calloc((size_t)P2, sizeof(int));
    double* canvas = malloc(sizeof(double) * (size_t)padM * padN);
    double* y = malloc(sizeof(double) * (size_t)K);
    double* win = malloc(sizeof(double) * (size_t)K);
    for (long long i = 0; i < nb; ++i) {
        const int* t = task + 5 * i;
        const int key = (t[2] % period) * period + (t[3] % period);
        if (!tabs[key]) {
            const int L = or_local_matrix(opaque, period, t[2], t[3], W, NULL, NULL, NULL);
            const size_t KL = (size_t)K * L, KK = (size_t)K * K;
            double* mem = malloc(sizeof(double) * (2 * KL + 2 * KK + K));
            or_tables(opaque, period, t[2], t[3], W, decay, mem, mem + KL, mem + 2 * KL,
                      mem + 2 * KL + KK, mem + 2 * KL + 2 * KK, NULL);
            tabs[key] = mem;
            Ls[key] = L;
        }
        const int L = Ls[key];
        const size_t KL = (size_t)K * L, KK = (size_t)K * K;
        const double* mem = tabs[key];
        or_gather(pf, fc, t[2], t[3], W, y);
        or_block(W, L, mem, mem + KL, mem + 2 * KL, mem + 2 * KL + KK, mem + 2 * KL + 2 * KK, q,
                 y, iterations, step, NULL, NULL, win);
        const int rw = t[0] - t[2], cw = t[1] - t[3];
        for (int r = 0; r < B; ++r)
            for (int c = 0; c < B; ++c) {
                double v = win[(rw + r) * W + cw + c];
                if (clip) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                canvas[(size_t)(t[0] + r) * padN + t[1] + c] = v;
            }
    }
    for (int r = 0; r < M; ++r)
        memcpy(out + (size_t)r * N, canvas + (size_t)r * padN, sizeof(double) * N);
    for (int i = 0; i < P2; ++i) free(tabs[i]);
    free(tabs); free(Ls); free(canvas); free(y); free(win); free(q); free(task); free(pf);
    return nb;
}

/* psnr, pipeline.cpp:221-233 (returns +inf when identical) */
double or_psnr(const double* ref, const double* est, long long n) {
    double sum = 0.0;
    for (long long i = 0; i < n; ++i) {
        const double d = ref[i] - est[i];
        sum += d * d;
    }
    const double mse = sum / (double)n;
    if (mse == 0.0) return INFINITY;
    return -10.0 * log10(mse);
}

/* ------------------------------------------------------------------------- */
/* Test-image generator (tests/support/synthetic.cpp:9-80)                    */
/* ------------------------------------------------------------------------- */
int or_synthetic_image(int rows, int cols, uint64_t seed, double* img) {
    or_mt64 g;
    or_mt64_seed(&g, seed);
    const double tau = 6.283185307179586;
    const double gr = or_uniform01(&g) * 2.0 - 1.0;
    const double gc = or_uniform01(&g) * 2.0 - 1.0;
    double wv[6][4], bl[5][4], ed[2][4];
    for (int i = 0; i < 6; ++i) {
        wv[i][0] = (or_uniform01(&g) * 6.0 + 0.5) / rows;
        wv[i][1] = (or_uniform01(&g) * 6.0 + 0.5) / cols;
        wv[i][2] = or_uniform01(&g) * tau;
        wv[i][3] = or_uniform01(&g) * 0.5 + 0.1;
    }
    const int mn = rows < cols ? rows : cols;
    for (int i = 0; i < 5; ++i) {
        bl[i][0] = or_uniform01(&g) * rows;
        bl[i][1] = or_uniform01(&g) * cols;
        bl[i][2] = (or_uniform01(&g) * 0.12 + 0.04) * mn;
        bl[i][3] = (or_uniform01(&g) * 2.0 - 1.0) * 0.8;
    }
    for (int i = 0; i < 2; ++i) {
        const double ang = or_uniform01(&g) * tau;
        ed[i][0] = sin(ang);
        ed[i][1] = cos(ang);
        ed[i][2] = or_uniform01(&g) * (rows + cols) * 0.5;
        ed[i][3] = (or_uniform01(&g) * 2.0 - 1.0) * 0.6;
    }
    double lo = 1e300, hi = -1e300;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            double v = gr * r / rows + gc * c / cols;
            for (int i = 0; i < 6; ++i)
                v += wv[i][3] * sin(tau * (wv[i][0] * r + wv[i][1] * c) + wv[i][2]);
            for (int i = 0; i < 5; ++i) {
                const double dr = r - bl[i][0], dc = c - bl[i][1];
                v += bl[i][3] * exp(-(dr * dr + dc * dc) / (2.0 * bl[i][2] * bl[i][2]));
            }
            for (int i = 0; i < 2; ++i)
                v += ed[i][3] / (1.0 + exp(-(ed[i][0] * r + ed[i][1] * c - ed[i][2]) / 2.5));
            img[(size_t)r * cols + c] = v;
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
    const double span = hi > lo ? hi - lo : 1.0;
    for (size_t i = 0; i < (size_t)rows * cols; ++i) img[i] = 0.02 + 0.96 * (img[i] - lo) / span;
    return 0;
}
