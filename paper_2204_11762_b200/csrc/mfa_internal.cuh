// Internal declarations of libmfa (not part of the C ABI).
//
// Device layout of a model:
//   Q        bricked row quads (kernels.cuh): the entry of (i, j, k) holds the
//            quad (P[k][j][i], P[k][j][i+1], P[k][j][i+2], P[k][j][i+3]) -- for
//            p <= 3 together with the quad of row j+1 (a 32-byte row PAIR, one
//            256-bit load) -- with zeros past the grid; or Bezier blocks.
//   per axis span tables (span s = knot interval [U[p+s], U[p+s+1]]):
//     coef   float[nsp][REC]: power-basis coefficients of the p+1 non-zero
//            basis functions on span s in the local coordinate
//            t = (u - U[p+s]) / h_s in [0,1]:  N_{s+a}(t) = sum_m coef[a][m] t^m
//     invh   float[nsp]  1/h_s (0 for zero-length spans)
//     kh,kl  float[nsp+1] knots U[p..n] as an fp32 pair (kh + kl == U exactly
//            up to 2^-48 relative)
//     kfx    int64[nsp+1] knots U[p..n] in fixed point, 2^62 per unit
//     bucket int32[M]   bucket b covers [b/M, (b+1)/M): the last span whose
//            left knot is <= b/M (start of a short linear search)
//   interior (uniform axes): coefficients of the first interior span, passed
//            as kernel parameters so the FMAs read them from the constant bank.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>

#include "../../include/mfa.h"

// Device bounds checks for debug builds (compute-sanitizer is unavailable on
// this pool): build with MFA_EXTRA_NVCC_FLAGS=-DMFA_DEBUG_BOUNDS.
#ifdef MFA_DEBUG_BOUNDS
#include <cstdio>
#define MFA_DCHECK(c)                                                            \
    do {                                                                         \
        if (!(c)) {                                                              \
            printf("MFA_DCHECK failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);  \
            __trap();                                                            \
        }                                                                        \
    } while (0)
#else
#define MFA_DCHECK(c) \
    do {              \
    } while (0)
#endif

// render span records and the tracker that reads them must agree (model.cu
// writes the records, kernels.cuh reads them): defined here, for every TU
#ifndef MFA_NU_SHIFTCMP   // 1: span crossings tested on the shifted 32-bit offset d = (F - lo) >> dshift
#define MFA_NU_SHIFTCMP 1    //    against the span width in the same units (wsh, from the record): C5 +2.1 %
#endif
#ifndef MFA_SPAN_REC16   // 16-byte render span records (one 128-bit load per crossing instead of 256-bit)
#define MFA_SPAN_REC16 1
#endif
static_assert(!MFA_SPAN_REC16 || MFA_NU_SHIFTCMP, "16-byte span records carry wsh (MFA_NU_SHIFTCMP)");

#ifndef MFA_SUPERTILE   // full-frame work order: supertiles of MFA_SUPERTILE x MFA_SUPERTILE 16x16 tiles
#define MFA_SUPERTILE 2
#endif

namespace mfa {

constexpr int kMaxP = MFA_MAX_DEGREE;
constexpr int kMaxViewsPerLaunch = 64;
constexpr int kUniFracBits = 40;   // uniform axes: span-unit fixed point, 24.40
constexpr int kNonUniFracBits = 62; // non-uniform axes: parameter fixed point, 2.62
constexpr int kBrickLog = 4;        // bricks of 16x16x16 spans
constexpr int kBrick = 1 << kBrickLog;
constexpr int kQueueSlots = 256;    // persistent-kernel work counters (one per in-flight launch)
#ifndef MFA_MACRO_LOG
#define MFA_MACRO_LOG 1
#endif
constexpr int kMacroLog = MFA_MACRO_LOG;   // macro blocks of 2^3 span triples (transparent-block skip; 4^3: -3 %, 8^3: -9 %)
__host__ __device__ constexpr int bez_row(int p) { return p == 1 ? 2 : 4; }  // floats per stored block row
// Grouped Bezier layout (kBezierG, p = 3): blocks of 4 consecutive w-spans
// are interleaved by 32-byte sector -- group ((sw >> 2) * S1 + sv) * S0 + su is
// 8 lines of 128 B, line j holding sector j (block rows 2j, 2j+1) of its 4
// blocks -- so lanes of a warp that reload vertically neighbouring blocks in
// the same instruction share L1 lines (wavefronts).  kBezier: one contiguous
// block per span triple.
// group shape (experiment MFA_BEZ_GSHAPE): log2 extents (u, v, w) of the 4-block group
// 0 = (0,0,2) 4 w-spans, 1 = (0,1,1), 2 = (1,0,1), 3 = (2,0,0) 4 u-spans, 4 = (1,1,0)
#ifndef MFA_BEZ_GSHAPE
#define MFA_BEZ_GSHAPE 2
#endif
constexpr int kGLu = MFA_BEZ_GSHAPE == 2 || MFA_BEZ_GSHAPE == 4 ? 1 : (MFA_BEZ_GSHAPE == 3 ? 2 : 0);
constexpr int kGLv = MFA_BEZ_GSHAPE == 1 || MFA_BEZ_GSHAPE == 4 ? 1 : 0;
constexpr int kGLw = 2 - kGLu - kGLv;
// grouped block (su, sv, sw): its offset in 32-byte units = (group << 5) | slot
// (T = int in the render kernel: mfa_model_create keeps it below 2^31)
__host__ __device__ constexpr int bez_groups(int S, int l) { return (S + (1 << l) - 1) >> l; }
// S0g = bez_groups(S0, kGLu), S1g = bez_groups(S1, kGLv) (BezGrid carries both)
template <typename T = long long>
__host__ __device__ inline T bez_group_key(int S0g, int S1g, int su, int sv, int sw) {
    const T g = ((T)(sw >> kGLw) * S1g + (sv >> kGLv)) * S0g + (su >> kGLu);
    const int slot = (((sw & ((1 << kGLw) - 1)) << kGLv | (sv & ((1 << kGLv) - 1))) << kGLu) | (su & ((1 << kGLu) - 1));
    return (g << 5) | slot;
}
// float offset of block (su, sv, sw) (its sector 0) in the block array
__host__ __device__ inline long long bez_block_offset(int p, bool grouped, int S0, int S1, int su, int sv, int sw) {
    if (grouped) return bez_group_key(bez_groups(S0, kGLu), bez_groups(S1, kGLv), su, sv, sw) << 3;
    return (((long long)sw * S1 + sv) * S0 + su) * (long long)((p + 1) * (p + 1) * bez_row(p));
}
// floats between consecutive 32-byte sectors of one p = 3 block
__host__ __device__ constexpr int bez_sec(bool grouped) { return grouped ? 32 : 8; }
// blocks to allocate (grouped: whole groups)
__host__ __device__ inline long long bez_alloc_blocks(bool grouped, long long S0, long long S1, long long S2) {
    if (!grouped) return S0 * S1 * S2;
    auto up = [](long long n, int l) { return ((n + (1 << l) - 1) >> l) << l; };
    return up(S0, kGLu) * up(S1, kGLv) * up(S2, kGLw);
}

// float4 per brick entry: p <= 3 stores row PAIRS (rows j and j+1 of a quad
// column, 32 bytes: one 256-bit load fetches two rows), p >= 4 single quads
// (32-byte octets of one row measured 18% slower on C4: DESIGN.md §9)
__host__ __device__ constexpr int quad_f4(int p) { return p <= 3 ? 2 : 1; }
__host__ __device__ constexpr bool quad_pairs(int p) { return p <= 3; }

// brick entry extents for degree p (see kernels.cuh)
__host__ __device__ constexpr int brick_eu(int p) { return kBrick + (p == 4 ? 1 : (p == 5 ? 4 : 0)); }
__host__ __device__ constexpr int brick_ev(int p) { return kBrick + p; }

__host__ __device__ constexpr int rec_floats(int p) { return (((p + 1) * (p + 1)) + 3) / 4 * 4; }

struct AxisTables {
    const float* coef = nullptr;      // [nsp][rec_floats(p)]
    const float* invh = nullptr;      // [nsp]
    const float* kh = nullptr;        // [nsp+1]
    const float* kl = nullptr;        // [nsp+1]
    const long long* kfx = nullptr;   // [nsp+1]
    const int* bucket = nullptr;      // [M]
    const longlong4* srec = nullptr;  // [nsp] render span records {lo, hi (2^62 fixed point), bits(invh), bits(tsc)}
    int nsp = 0;                      // n - p (number of knot spans incl. zero-length)
    int M = 0;                        // bucket count
    int ic_lo = 0, ic_hi = -1;        // uniform: spans [ic_lo, ic_hi] use the interior constants
    int uniform = 0;
    int dshift = 0;                   // see kernels.cuh nu_span
    long long hmin_fx = 0;            // smallest span width in 2^62 fixed point (0 with repeated knots)
    float S = 0.f;                    // uniform: number of spans as float
};

enum Layout { kQuads = 0, kBezier = 1, kBricks = 2, kBezierG = 3 };   // kBezierG: grouped Bezier blocks (p = 3)
__host__ __device__ constexpr bool is_bez(int layout) { return layout == kBezier || layout == kBezierG; }

// plain haloed bricks (kBricks, p <= 3): one fp32 per control point, bricks
// of 16^3 spans with the p halo points on the high side, rows padded to a
// multiple of 4 floats (16-byte aligned): (16+p rounded up to 4) x (16+p)^2
// floats per brick, <= 1.86 x the grid (C5: 1.85 x)
__host__ __device__ constexpr int pbrick_eu(int p) { return ((kBrick + p + 3) / 4) * 4; }
__host__ __device__ constexpr int pbrick_ev(int p) { return kBrick + p; }

struct Model {
    int device = 0;
    int p = 0;
    int layout = kQuads;           // kBezier: per-span-triple Bernstein blocks (p <= 3); kBricks: plain haloed bricks
    int64_t n[3] = {0, 0, 0};
    int uniform[3] = {0, 0, 0};
    float vmin = 0.f, vmax = 0.f;
    float4* Q = nullptr;           // bricked row quads (kQuads) or Bezier blocks (kBezier)
    int64_t q_f4 = 0;              // size of Q in float4
    int nb[3] = {0, 0, 0};         // bricks per axis
    unsigned int* queue = nullptr; // kQueueSlots work counters
    AxisTables ax[3];
    void* table_mem = nullptr;   // one allocation for all axis tables
    int64_t device_bytes = 0;
    // Bezier layout: value bounds per macro block of kMacro^3 span triples (the
    // Bernstein convex hull: min / max coefficient, order-preserving uint
    // encoding), for NEXT-1's transparent-block skip (shading = 3)
    unsigned int* mmx = nullptr;   // [n_macro][2]
    int mm[3] = {0, 0, 0};         // macro blocks per axis
    int64_t model_bytes = 0;       // the fp32 control grid the caller passed (n_u n_v n_w * 4)
    double create_ms = 0.0;        // wall time of mfa_model_create (validation, upload, relayout, tables)

    // persistent-kernel work counters: a slot is owned by one launch until
    // its completion event fires; another launch on the SAME stream may reuse
    // it (stream order); more than kQueueSlots renders in flight on distinct
    // streams are refused (acquire_queue_slot)
    struct QueueSlot {
        cudaEvent_t done = nullptr;
        cudaStream_t stream = nullptr;
        bool used = false;
        bool pending = false;
    };
    mutable std::mutex slot_mu;
    mutable QueueSlot slots[kQueueSlots];

    // mfa_render_host resources, created on first use and reused (one
    // host-buffer render at a time per model: host_mu)
    struct HostRes {
        cudaStream_t copy = nullptr;
        cudaEvent_t rendered[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
        void* stage[2] = {nullptr, nullptr};
        size_t stage_bytes = 0;
        float* tf = nullptr;           // 1024 x 4 fp32
        unsigned long long* cnt = nullptr;
    };
    mutable std::mutex host_mu;
    mutable HostRes host;
};

// queue-slot ownership (render.cu): index of a free slot for a launch on st,
// or -1 if every slot is held by an unfinished launch on another stream
int acquire_queue_slot(const Model* m, cudaStream_t st);
void release_queue_slot(const Model* m, int slot, cudaStream_t st);   // records the completion event
void free_model_resources(Model* m);                                  // slot events, render_host resources
void* scratch_alloc(size_t bytes, cudaStream_t st);                   // stream-ordered, default pool (model.cu)
size_t hessian_workspace_bytes(const Model* m, int64_t n);             // hessian.cu

// Power-basis coefficients of the p+1 non-zero basis functions on knot span
// i (local t = (u - U_i)/h, u = U_i + h t): P[r][m] = coefficient of t^m of
// N_{i-p+r,p}.  Cox-de Boor recursion on polynomials in t, fp64.
__host__ __device__ inline void span_poly(const double* __restrict__ U, int p, int i, double (&P)[kMaxP + 1][kMaxP + 1]) {
    const double Ui = U[i], h = U[i + 1] - U[i];
    double Nx[kMaxP + 1][kMaxP + 1];
    for (int r = 0; r <= kMaxP; ++r)
        for (int m = 0; m <= kMaxP; ++m) P[r][m] = 0.0;
    P[0][0] = 1.0;  // level 0: N_{i,0} = 1 on the span
    for (int k = 1; k <= p; ++k) {
        for (int r = 0; r <= k; ++r) {
            for (int m = 0; m <= kMaxP; ++m) Nx[r][m] = 0.0;
            const int j = i - k + r;
            if (r >= 1) {  // (u - U_j)/(U_{j+k} - U_j) * N_{j,k-1}; N_{j,k-1} is old function r-1
                const double den = U[j + k] - U[j];
                const double c0 = (Ui - U[j]) / den, c1 = h / den;
                for (int m = 0; m < k; ++m) {
                    Nx[r][m] += c0 * P[r - 1][m];
                    Nx[r][m + 1] += c1 * P[r - 1][m];
                }
            }
            if (r <= k - 1) {  // (U_{j+k+1} - u)/(U_{j+k+1} - U_{j+1}) * N_{j+1,k-1}; old function r
                const double den = U[j + k + 1] - U[j + 1];
                const double c0 = (U[j + k + 1] - Ui) / den, c1 = -h / den;
                for (int m = 0; m < k; ++m) {
                    Nx[r][m] += c0 * P[r][m];
                    Nx[r][m + 1] += c1 * P[r][m];
                }
            }
        }
        for (int r = 0; r <= k; ++r)
            for (int m = 0; m <= kMaxP; ++m) P[r][m] = Nx[r][m];
    }
}

// error plumbing
void set_error(const std::string& msg);
mfa_status fail(mfa_status st, const std::string& msg);
mfa_status cuda_fail(cudaError_t e, const char* what);
mfa_status check_device(const Model* m);
mfa_status validate_knots(int d, int p, int64_t n, const double* U, int* uniform);

// kernel launchers (defined in eval.cu / render.cu)
mfa_status launch_eval(const Model* m, int64_t n, const float* u, const float* v, const float* w,
                       float* value, float* du, float* dv, float* dw,
                       unsigned long long* n_err, cudaStream_t st, void* ws = nullptr, size_t ws_bytes = 0);
size_t eval_workspace_bytes(const Model* m, int64_t n);
// spatial binning of a point batch (eval.cu): records (u, v, w, index bits) in
// bin order, and pos[i] = sorted position of point i; needs bin_workspace_bytes
struct BinnedPoints {
    float4* rec;
    int* pos;
    const unsigned* counts;   // points per bin (nbins + 1: the last bin holds points outside [0,1]^3)
    const unsigned* cursor;   // after the scatter: end of bin b at cursor[b * stride]
    int stride;
    int nb[3];
    int nbins;
};
size_t bin_workspace_bytes(const Model* m, int64_t n);
// binning pays only when the model does not stay in L2: a model of at most
// kBinModelBytes is gathered directly in input order (C2, 56 MB of Bezier
// blocks: 24 G vs 10 G points/s binned; C3 quads, 722 MB: 6.4 vs 13.1)
constexpr int64_t kBinModelBytes = 64ll << 20;
inline bool bin_worthwhile(const Model* m, int64_t n) {
    return n >= ((int64_t)1 << 16) && n < ((int64_t)1 << 31) && m->device_bytes > kBinModelBytes;
}
BinnedPoints bin_points(const Model* m, int64_t n, const float* u, const float* v, const float* w, void* ws,
                        cudaStream_t st);
mfa_status launch_render(const Model* m, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                         const mfa_render_params* prm, const mfa_tiles* tiles, void* out,
                         unsigned long long* samples, cudaStream_t st, const mfa_render_ext* ext = nullptr);

}  // namespace mfa
