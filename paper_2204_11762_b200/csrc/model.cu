// libmfa: model ingest, error plumbing, tile unpack (K4)
// and the host-buffer render driver.
//
// mfa_model_create validates the knot vectors, copies the fp32
// control grid, and builds on the device
//   * the row-quad layout Q (K1 relayout kernel),
//   * per-axis span tables: the power-basis coefficients of the p+1 non-zero
//     basis functions on every knot span, derived from the Cox-de Boor
//     recursion in fp64 and stored in fp32, plus knot tables
//     for span search (fp32 pairs, 2^62 fixed point, buckets),
//   * the value range [min P, max P] and a finiteness check.
#include <cuda_fp16.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "mfa_internal.cuh"

namespace mfa {

constexpr double kBezSmallModelBytes = 64.0 * 1024 * 1024;   // AUTO layout: uniform models up to this use Bezier blocks

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

mfa_status fail(mfa_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

mfa_status cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return e == cudaErrorMemoryAllocation ? MFA_ERR_OOM : MFA_ERR_CUDA;
}

mfa_status check_device(const Model* m) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev != m->device)
        return fail(MFA_ERR_DEVICE, "model lives on device " + std::to_string(m->device) +
                                        " but device " + std::to_string(dev) + " is current");
    return MFA_OK;
}

// ---------------------------------------------------------------------------
// K1: bricked row-quad relayout.  Brick (bx,by,bz) entry (lu,lv,lw) holds the
// quad (P[k][j][i..i+3]) of i = 16 bx + lu, j = 16 by + lv, k = 16 bz + lw
// (zeros outside the grid).  One thread per entry.
// ---------------------------------------------------------------------------
__global__ void relayout_bricks_kernel(const float* __restrict__ P, float4* __restrict__ Q, int nu, int nv,
                                       int nw, int nbx, int nby, int EU, int EV, int EW, int64_t total, int pairs) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bsz = (int64_t)EU * EV * EW;
        const int64_t brick = idx / bsz;
        int rem = (int)(idx - brick * bsz);
        const int lu = rem % EU;
        rem /= EU;
        const int lv = rem % EV;
        const int lw = rem / EV;
        const int bx = (int)(brick % nbx);
        const int by = (int)((brick / nbx) % nby);
        const int bz = (int)(brick / ((int64_t)nbx * nby));
        const int i = bx * kBrick + lu, j = by * kBrick + lv, k = bz * kBrick + lw;
        auto quad = [&](int jj) {
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            if (jj < nv && k < nw) {
                const float* r = P + ((int64_t)k * nv + jj) * nu;
                if (i < nu) q.x = r[i];
                if (i + 1 < nu) q.y = r[i + 1];
                if (i + 2 < nu) q.z = r[i + 2];
                if (i + 3 < nu) q.w = r[i + 3];
            }
            return q;
        };
        if (pairs == 1) {   // p <= 3: rows j and j+1 side by side (one 256-bit load, kernels.cuh load_slab)
            Q[2 * idx] = quad(j);
            Q[2 * idx + 1] = quad(j + 1);
        } else {
            Q[idx] = quad(j);
        }
    }
}

// K1c: plain haloed bricks (kBricks, p <= 3).  Brick (bx,by,bz) float
// (lu,lv,lw) = P[k][j][i] of i = 16 bx + lu, j = 16 by + lv, k = 16 bz + lw
// (zeros outside the grid and in the row padding).  One thread per float.
__global__ void relayout_plain_kernel(const float* __restrict__ P, float* __restrict__ Q, int nu, int nv, int nw,
                                      int nbx, int nby, int EU, int EV, int64_t total) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bsz = (int64_t)EU * EV * EV;
        const int64_t brick = idx / bsz;
        int rem = (int)(idx - brick * bsz);
        const int lu = rem % EU;
        rem /= EU;
        const int lv = rem % EV;
        const int lw = rem / EV;
        const int bx = (int)(brick % nbx);
        const int by = (int)((brick / nbx) % nby);
        const int bz = (int)(brick / ((int64_t)nbx * nby));
        const int i = bx * kBrick + lu, j = by * kBrick + lv, k = bz * kBrick + lw;
        Q[idx] = (lu < EV && i < nu && j < nv && k < nw) ? P[((int64_t)k * nv + j) * nu + i] : 0.f;
    }
}

// Order-preserving float <-> uint mapping for atomic min/max.
__device__ __forceinline__ unsigned int f2ord(float f) {
    unsigned int u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
static inline float ord2f(unsigned int u) {
    unsigned int b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &b, 4);
    return f;
}

__global__ void minmax_kernel(const float* __restrict__ P, int64_t n, unsigned int* out /*min,max,nonfinite*/) {
    unsigned int lo = 0xffffffffu, hi = 0u, bad = 0u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float x = P[i];
        if (!isfinite(x)) { bad++; continue; }
        unsigned int o = f2ord(x);
        lo = min(lo, o);
        hi = max(hi, o);
    }
    for (int s = 16; s > 0; s >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, s));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, s));
        bad += __shfl_xor_sync(0xffffffffu, bad, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out + 0, lo);
        atomicMax(out + 1, hi);
        if (bad) atomicAdd(out + 2, bad);
    }
}

// ---------------------------------------------------------------------------
// K0: span tables.  One thread per knot span s (knot index i = p + s).
// The p+1 non-zero basis functions on [U_i, U_{i+1}) are polynomials in the
// local coordinate t = (u - U_i)/h.  They follow from the Cox-de Boor
// recursion  N_{j,k} = (u-U_j)/(U_{j+k}-U_j) N_{j,k-1}
//                    + (U_{j+k+1}-u)/(U_{j+k+1}-U_{j+1}) N_{j+1,k-1}
// applied to polynomials in t (u = U_i + h t), in fp64.
// ---------------------------------------------------------------------------
__global__ void span_tables_kernel(const double* __restrict__ U, int p, int nsp, int rec,
                                   float* __restrict__ coef, float* __restrict__ invh) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsp) return;
    const int i = p + s;
    const double h = U[i + 1] - U[i];
    float* out = coef + (int64_t)s * rec;
    for (int q = 0; q < rec; ++q) out[q] = 0.f;
    if (!(h > 0.0)) {
        invh[s] = 0.f;
        return;
    }
    invh[s] = (float)(1.0 / h);
    double P[kMaxP + 1][kMaxP + 1];
    span_poly(U, p, i, P);
    for (int a = 0; a <= p; ++a)
        for (int m = 0; m <= p; ++m) out[a * (p + 1) + m] = (float)P[a][m];
}

// Render span records (non-uniform axes): one 32-byte record per span with
// the bounds [lo, hi) in 2^62 fixed point (hi of the last span = INT64_MAX),
// 1/h and the offset scale 2^(dshift-62)/h, so a span crossing is one sector
// load (kernels.cuh nu_load).
__global__ void span_rec_kernel(const long long* __restrict__ kfx, const float* __restrict__ invh, int nsp,
                                float dscale, int dshift, longlong4* __restrict__ rec) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsp) return;
    const float ih = invh[s];
#if MFA_NU_SHIFTCMP   // {lo, ceil(width / 2^dshift) (INT_MAX for the last span), bits(1/h), bits(tsc)}
    const long long w = s + 1 < nsp ? kfx[s + 1] - kfx[s] : -1;
    const long long second = w < 0 ? 0x7fffffffLL : (w + (1LL << dshift) - 1) >> dshift;
#else
    const long long second = s + 1 < nsp ? kfx[s + 1] : 0x7fffffffffffffffLL;
#endif
#if MFA_SPAN_REC16   // {lo, wsh | bits(1/h) << 32}: the kernels derive tsc = (1/h) * dscale
    reinterpret_cast<longlong2*>(rec)[s] =
        make_longlong2(kfx[s], (long long)(((unsigned long long)(unsigned)__float_as_int(ih) << 32) |
                                           (unsigned long long)(unsigned)second));
#else
    rec[s] = make_longlong4(kfx[s], second,
                            (long long)(unsigned)__float_as_int(ih),
                            (long long)(unsigned)__float_as_int(ih * dscale));
#endif
}

// Bezier extraction operator of span s: N_{s+a}(t) = sum_j D[a][j] B_j(t) with
// the Bernstein polynomials B_j(t) = C(p,j) t^j (1-t)^(p-j).  From the power
// form: t^m = sum_{j>=m} C(j,m)/C(p,m) B_j(t).  All D >= 0 (convex weights).
__device__ double binom_d(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

__global__ void bezier_tables_kernel(const double* __restrict__ U, int p, int nsp, double* __restrict__ D) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsp) return;
    const int i = p + s;
    double* out = D + (int64_t)s * (p + 1) * (p + 1);
    for (int q = 0; q < (p + 1) * (p + 1); ++q) out[q] = 0.0;
    if (!(U[i + 1] - U[i] > 0.0)) return;
    double P[kMaxP + 1][kMaxP + 1];
    span_poly(U, p, i, P);
    for (int a = 0; a <= p; ++a)
        for (int j = 0; j <= p; ++j) {
            double acc = 0.0;
            for (int m = 0; m <= j; ++m) acc += binom_d(j, m) / binom_d(p, m) * P[a][m];
            out[a * (p + 1) + j] = acc;
        }
}

// K1b: Bezier blocks.  Block (su,sv,sw) holds the (p+1)^3 Bernstein
// coefficients of the spline on that span triple:
//   Z[l][k][j] = sum_{c,b,a} Dw[c][l] Dv[b][k] Du[a][j] P[sw+c][sv+b][su+a]
// (sum-factorised, fp64), stored as rows of bez_row(p) floats, j fastest.
__global__ void init_minmax_kernel(unsigned* __restrict__ mmx, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        mmx[2 * i] = 0xffffffffu;   // ordered min: starts at the largest key
        mmx[2 * i + 1] = 0u;
    }
}

template <int P, bool G = false>
__global__ void bezier_blocks_kernel(const float* __restrict__ Pg, int nu, int nv, const double* __restrict__ Du,
                                     const double* __restrict__ Dv, const double* __restrict__ Dw, int Su, int Sv,
                                     int64_t nblocks, float* __restrict__ out, unsigned* __restrict__ mmx, int mm0,
                                     int mm1) {
    constexpr int Q = P + 1, R = bez_row(P);
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nblocks;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int su = (int)(idx % Su);
        const int sv = (int)((idx / Su) % Sv);
        const int sw = (int)(idx / ((int64_t)Su * Sv));
        const double* du = Du + (int64_t)su * Q * Q;
        const double* dv = Dv + (int64_t)sv * Q * Q;
        const double* dw = Dw + (int64_t)sw * Q * Q;
        double X[Q][Q][Q], Y[Q][Q][Q];
        for (int c = 0; c < Q; ++c)
            for (int b = 0; b < Q; ++b) {
                const float* row = Pg + ((int64_t)(sw + c) * nv + (sv + b)) * nu + su;
                double g[Q];
                for (int a = 0; a < Q; ++a) g[a] = (double)row[a];
                for (int j = 0; j < Q; ++j) {
                    double acc = 0.0;
                    for (int a = 0; a < Q; ++a) acc += du[a * Q + j] * g[a];
                    X[c][b][j] = acc;
                }
            }
        for (int c = 0; c < Q; ++c)
            for (int k = 0; k < Q; ++k)
                for (int j = 0; j < Q; ++j) {
                    double acc = 0.0;
                    for (int b = 0; b < Q; ++b) acc += dv[b * Q + k] * X[c][b][j];
                    Y[c][k][j] = acc;
                }
        float* o = out + bez_block_offset(P, G, Su, Sv, su, sv, sw);
        float lo = INFINITY, hi = -INFINITY;
        for (int l = 0; l < Q; ++l)
            for (int k = 0; k < Q; ++k) {
                // row (l, k) = the (l * Q + k)-th R-float row; 32-byte sector = 8 / R rows
                const int row = l * Q + k;
                float* orow = G ? o + (row >> 1) * bez_sec(G) + (row & 1) * R : o + row * R;
                for (int j = 0; j < Q; ++j) {
                    double acc = 0.0;
                    for (int c = 0; c < Q; ++c) acc += dw[c * Q + l] * Y[c][k][j];
                    const float f = (float)acc;
                    orow[j] = f;
                    lo = fminf(lo, f);
                    hi = fmaxf(hi, f);
                }
                for (int j = Q; j < R; ++j) orow[j] = 0.f;
            }
        // macro-block value bounds (the spline on a span triple lies in the
        // convex hull of its Bernstein coefficients)
        const int64_t mi = ((int64_t)(sw >> kMacroLog) * mm1 + (sv >> kMacroLog)) * mm0 + (su >> kMacroLog);
        atomicMin(mmx + 2 * mi, f2ord(lo));
        atomicMax(mmx + 2 * mi + 1, f2ord(hi));
    }
}

__global__ void knot_tables_kernel(const double* __restrict__ U, int p, int nsp, float* __restrict__ kh,
                                   float* __restrict__ kl, long long* __restrict__ kfx, int M,
                                   int* __restrict__ bucket) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t <= nsp) {
        const double u = U[p + t];
        const float hi = (float)u;
        kh[t] = hi;
        kl[t] = (float)(u - (double)hi);
        kfx[t] = llrint(ldexp(u, kNonUniFracBits));
    }
    if (t < M) {
        // last span s in [0, nsp-1] with U[p+s] <= t/M
        const double x = (double)t / (double)M;
        int lo = 0, hi = nsp - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (U[p + mid] <= x) lo = mid; else hi = mid - 1;
        }
        bucket[t] = lo;
    }
}

// ---------------------------------------------------------------------------
// K4: scatter packed 16x16 tiles into images.
// ---------------------------------------------------------------------------
__global__ void unpack_tiles_kernel(const void* __restrict__ packed, int in_fp16, const int* __restrict__ tiles,
                                    int64_t n_tiles, int n_views, int W, int H, float4* __restrict__ img) {
    const int64_t t = blockIdx.x;
    if (t >= n_tiles) return;
    const int view = tiles[3 * t], tx = tiles[3 * t + 1], ty = tiles[3 * t + 2];
    // padding units (view = -1) and malformed entries are skipped (no store outside the image)
    if (view < 0 || view >= n_views || tx < 0 || ty < 0 || tx >= (W + MFA_TILE - 1) / MFA_TILE ||
        ty >= (H + MFA_TILE - 1) / MFA_TILE)
        return;
    const int px = threadIdx.x & 15, py = threadIdx.x >> 4;
    const int x = tx * MFA_TILE + px, y = ty * MFA_TILE + py;
    if (x >= W || y >= H) return;
    const int64_t src = t * (MFA_TILE * MFA_TILE) + threadIdx.x;
    float4 v;
    if (in_fp16) {
        const __half2* p = reinterpret_cast<const __half2*>(packed) + 2 * src;
        float2 a = __half22float2(p[0]), b = __half22float2(p[1]);
        v = make_float4(a.x, a.y, b.x, b.y);
    } else {
        v = reinterpret_cast<const float4*>(packed)[src];
    }
    img[((int64_t)view * H + y) * W + x] = v;
}

}  // namespace mfa

using namespace mfa;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" const char* mfa_last_error(void) { return g_err.c_str(); }

extern "C" const char* mfa_version(void) { return "mfa-b200 0.1 sm_100a"; }

mfa_status mfa::validate_knots(int d, int p, int64_t n, const double* U, int* uniform) {
    const char* ax = d == 0 ? "u" : (d == 1 ? "v" : "w");
    const int64_t len = n + p + 1;
    for (int64_t i = 0; i < len; ++i)
        if (!isfinite(U[i]))
            return fail(MFA_ERR_KNOTS, std::string("knots[") + ax + "][" + std::to_string(i) + "] is not finite");
    for (int64_t i = 0; i + 1 < len; ++i)
        if (U[i + 1] < U[i])
            return fail(MFA_ERR_KNOTS, std::string("knots[") + ax + "] decreases at index " + std::to_string(i + 1));
    for (int i = 0; i <= p; ++i) {
        if (U[i] != 0.0)
            return fail(MFA_ERR_KNOTS, std::string("knots[") + ax + "][" + std::to_string(i) +
                                           "] must be 0 (clamped, first p+1 knots)");
        if (U[len - 1 - i] != 1.0)
            return fail(MFA_ERR_KNOTS, std::string("knots[") + ax + "][" + std::to_string(len - 1 - i) +
                                           "] must be 1 (clamped, last p+1 knots)");
    }
    int64_t run = 1;
    for (int64_t i = p + 2; i < n; ++i) {  // interior knots U[p+1..n-1]
        run = (U[i] == U[i - 1]) ? run + 1 : 1;
        if (run > p)
            return fail(MFA_ERR_KNOTS, std::string("knots[") + ax + "] interior multiplicity > degree at index " +
                                           std::to_string(i));
    }
    if (n > p + 1 && (U[p + 1] == 0.0 || U[n - 1] == 1.0))
        return fail(MFA_ERR_KNOTS, std::string("knots[") + ax + "] interior knot equals an end knot");
    const int64_t S = n - p;
    int uni = 1;
    for (int64_t k = 1; k < S && uni; ++k)
        if (U[p + k] != (double)k / (double)S) uni = 0;
    *uniform = uni;
    return MFA_OK;
}

extern "C" mfa_status mfa_model_create_ex(const int32_t degree[3], const int64_t nctrl[3],
                                          const double* const knots[3], const float* ctrl, int32_t ctrl_on_device,
                                          const mfa_model_options* opt, mfa_stream stream, mfa_model* out) {
    const auto t_create = std::chrono::steady_clock::now();
    if (!out) return fail(MFA_ERR_INVALID_ARG, "out is NULL");
    const int want_layout = opt ? opt->layout : MFA_LAYOUT_AUTO;
    if (want_layout < MFA_LAYOUT_AUTO || want_layout > MFA_LAYOUT_BEZIER_GROUPED)
        return fail(MFA_ERR_INVALID_ARG, "options.layout out of range");
    *out = nullptr;
    if (!degree || !nctrl || !knots || !ctrl) return fail(MFA_ERR_INVALID_ARG, "NULL argument");
    const int p = degree[0];
    if (degree[1] != p || degree[2] != p)
        return fail(MFA_ERR_UNSUPPORTED, "this build requires equal degrees on all axes");
    if (p < 1 || p > MFA_MAX_DEGREE)
        return fail(MFA_ERR_UNSUPPORTED, "degree " + std::to_string(p) + " outside the compiled set 1..5");
    for (int d = 0; d < 3; ++d) {
        if (!knots[d]) return fail(MFA_ERR_INVALID_ARG, "knots[" + std::to_string(d) + "] is NULL");
        if (nctrl[d] < p + 1)
            return fail(MFA_ERR_INVALID_ARG, "nctrl[" + std::to_string(d) + "] < degree+1");
        if (nctrl[d] > (1 << 20))
            return fail(MFA_ERR_UNSUPPORTED, "nctrl[" + std::to_string(d) + "] > 2^20");
    }
    int uniform[3];
    for (int d = 0; d < 3; ++d) {
        mfa_status st = validate_knots(d, p, nctrl[d], knots[d], &uniform[d]);
        if (st != MFA_OK) return st;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Model* m = new Model();
    m->p = p;
    for (int d = 0; d < 3; ++d) {
        m->n[d] = nctrl[d];
        m->uniform[d] = uniform[d];
    }
    cudaError_t e = cudaGetDevice(&m->device);
    if (e != cudaSuccess) { delete m; return cuda_fail(e, "cudaGetDevice"); }

    const int64_t nu = nctrl[0], nv = nctrl[1], nw = nctrl[2];
    const int64_t npts = nu * nv * nw;
    float* Pdev = nullptr;
    float* Pown = nullptr;
    double* Udev = nullptr;
    unsigned int* mm = nullptr;
    auto cleanup = [&](mfa_status s) {
        if (Pown) cudaFree(Pown);
        if (Udev) cudaFree(Udev);
        if (mm) cudaFree(mm);
        if (s != MFA_OK) {
            if (m->mmx) cudaFree(m->mmx);
            if (m->Q) cudaFree(m->Q);
            if (m->queue) cudaFree(m->queue);
            if (m->table_mem) cudaFree(m->table_mem);
            delete m;
        }
        return s;
    };
    if (ctrl_on_device) {
        Pdev = const_cast<float*>(ctrl);
    } else {
        if ((e = cudaMalloc(&Pown, npts * sizeof(float))) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc ctrl"));
        if ((e = cudaMemcpyAsync(Pown, ctrl, npts * sizeof(float), cudaMemcpyHostToDevice, st)) != cudaSuccess)
            return cleanup(cuda_fail(e, "copy ctrl"));
        Pdev = Pown;
    }
    // finiteness + value range
    if ((e = cudaMalloc(&mm, 3 * sizeof(unsigned int))) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc"));
    unsigned int init[3] = {0xffffffffu, 0u, 0u};
    cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, st);
    minmax_kernel<<<1184, 256, 0, st>>>(Pdev, npts, mm);
    if ((e = cudaMalloc(&m->queue, kQueueSlots * sizeof(unsigned int))) != cudaSuccess)
        return cleanup(cuda_fail(e, "cudaMalloc queue"));
    cudaMemsetAsync(m->queue, 0, kQueueSlots * sizeof(unsigned int), st);

    // axis tables: one allocation
    const int rec = rec_floats(p);
    size_t off[3][7];
    size_t total = 0;
    int Mb[3];
    auto bump = [&](size_t bytes) {
        size_t o = total;
        total += (bytes + 255) & ~(size_t)255;
        return o;
    };
    for (int d = 0; d < 3; ++d) {
        const int nsp = (int)(nctrl[d] - p);
        int M = 1;
        while (M < 4 * nsp) M <<= 1;
        Mb[d] = M;
        off[d][0] = bump(sizeof(float) * rec * nsp);        // coef
        off[d][1] = bump(sizeof(float) * nsp);              // invh
        off[d][2] = bump(sizeof(float) * (nsp + 1));        // kh
        off[d][3] = bump(sizeof(float) * (nsp + 1));        // kl
        off[d][4] = bump(sizeof(long long) * (nsp + 1));    // kfx
        off[d][5] = bump(sizeof(int) * M);                  // bucket
        off[d][6] = bump(sizeof(longlong4) * nsp);          // span records
    }
    size_t uoff[3];
    size_t utotal = 0;
    for (int d = 0; d < 3; ++d) {
        uoff[d] = utotal;
        utotal += sizeof(double) * (nctrl[d] + p + 1);
    }
    if ((e = cudaMalloc(&m->table_mem, total)) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc tables"));
    if ((e = cudaMalloc(&Udev, utotal)) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc knots"));
    m->device_bytes += total;
    char* base = (char*)m->table_mem;
    for (int d = 0; d < 3; ++d) {
        const int nsp = (int)(nctrl[d] - p);
        double* Ud = (double*)((char*)Udev + uoff[d]);
        cudaMemcpyAsync(Ud, knots[d], sizeof(double) * (nctrl[d] + p + 1), cudaMemcpyHostToDevice, st);
        AxisTables& A = m->ax[d];
        A.coef = (float*)(base + off[d][0]);
        A.invh = (float*)(base + off[d][1]);
        A.kh = (float*)(base + off[d][2]);
        A.kl = (float*)(base + off[d][3]);
        A.kfx = (long long*)(base + off[d][4]);
        A.bucket = (int*)(base + off[d][5]);
        A.nsp = nsp;
        A.M = Mb[d];
        {   // smallest shift with (max span width * 2^62) >> shift < 2^23
            double hmax = 0.0;
            for (int64_t i = p; i < nctrl[d]; ++i) hmax = std::max(hmax, knots[d][i + 1] - knots[d][i]);
            int sh = 0;
            while (sh < 62 && ldexp(hmax, kNonUniFracBits - sh) >= 8388607.0) ++sh;
            A.dshift = sh;
            long long hm = 0x7fffffffffffffffLL;   // the kfx of knot_tables_kernel, on the host
            for (int64_t i = p; i < nctrl[d]; ++i)
                hm = std::min(hm, llrint(ldexp(knots[d][i + 1], kNonUniFracBits)) - llrint(ldexp(knots[d][i], kNonUniFracBits)));
            A.hmin_fx = hm;
        }
        A.uniform = uniform[d];
        A.S = (float)nsp;
        span_tables_kernel<<<(nsp + 127) / 128, 128, 0, st>>>(Ud, p, nsp, rec, (float*)A.coef, (float*)A.invh);
        const int nt = std::max(nsp + 1, Mb[d]);
        knot_tables_kernel<<<(nt + 255) / 256, 256, 0, st>>>(Ud, p, nsp, (float*)A.kh, (float*)A.kl,
                                                             (long long*)A.kfx, Mb[d], (int*)A.bucket);
        A.srec = (longlong4*)(base + off[d][6]);
        span_rec_kernel<<<(nsp + 127) / 128, 128, 0, st>>>((const long long*)A.kfx, (const float*)A.invh, nsp,
                                                           ldexpf(1.0f, A.dshift - kNonUniFracBits), A.dshift,
                                                           (longlong4*)A.srec);
        // uniform interior spans [p-1, S-p] share one polynomial set
        A.ic_lo = p - 1;
        A.ic_hi = nsp - p;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return cleanup(cuda_fail(e, "model ingest kernels"));
    for (int d = 0; d < 3; ++d) {
        AxisTables& A = m->ax[d];
        if (!(A.uniform && A.ic_hi >= A.ic_lo)) {
            A.ic_lo = 0;
            A.ic_hi = -1;
        }
    }

    // ---- control-point layout ----------------------------
    const bool nonuni = !(uniform[0] && uniform[1] && uniform[2]);
    // AUTO: Bezier blocks for non-uniform models, and for uniform ones whose
    // blocks fit in a fraction of L2 (small models: every reload is an L2 hit)
    const double bez_bytes = 4.0 * (p + 1) * (p + 1) * (p + 1) * (double)(nctrl[0] - p) * (nctrl[1] - p) * (nctrl[2] - p);
    const bool want_bez = want_layout == MFA_LAYOUT_BEZIER || want_layout == MFA_LAYOUT_BEZIER_GROUPED;
    bool bez = want_bez || (want_layout == MFA_LAYOUT_AUTO && p <= 3 && (nonuni || bez_bytes <= kBezSmallModelBytes));
    if (bez && p > 3) return cleanup(fail(MFA_ERR_UNSUPPORTED, "Bezier-block layout needs degree <= 3"));
    if (want_layout == MFA_LAYOUT_BEZIER_GROUPED && p != 3)
        return cleanup(fail(MFA_ERR_UNSUPPORTED, "grouped Bezier layout needs degree 3"));
    // AUTO takes the grouped blocks at p = 3 (C5 render +6 %, bit-identical)
    const bool grouped = bez && p == 3 && want_layout != MFA_LAYOUT_BEZIER;
    if (want_layout == MFA_LAYOUT_BRICKS && p > 3)
        return cleanup(fail(MFA_ERR_UNSUPPORTED, "plain-brick layout needs degree <= 3"));
    // 32-bit block index (render cache key; grouped layout: the offset in 32-byte units)
    if (bez && bez_alloc_blocks(grouped, nctrl[0] - p, nctrl[1] - p, nctrl[2] - p) * (grouped ? 8 : 1) >=
                   ((int64_t)1 << 31)) {
        if (want_bez)
            return cleanup(fail(MFA_ERR_UNSUPPORTED, "Bezier-block layout needs < 2^31 span triples"));
        bez = false;
    }
    if (bez) {
        const int64_t S0 = nctrl[0] - p, S1 = nctrl[1] - p, S2 = nctrl[2] - p;
        const int64_t nblk = S0 * S1 * S2;
        const int64_t nblk_alloc = bez_alloc_blocks(grouped, S0, S1, S2);   // grouped layout: whole groups
        const int64_t bfl = (int64_t)(p + 1) * (p + 1) * bez_row(p);      // floats per block
        e = cudaMalloc(&m->Q, nblk_alloc * bfl * sizeof(float));
        if (e != cudaSuccess) {
            m->Q = nullptr;
            if (want_bez) return cleanup(cuda_fail(e, "cudaMalloc Bezier blocks"));
            cudaGetLastError();   // AUTO: fall back to the quad layout
            bez = false;
        } else {
            double* D = nullptr;
            const int64_t q2 = (int64_t)(p + 1) * (p + 1);
            if ((e = cudaMalloc(&D, sizeof(double) * q2 * (S0 + S1 + S2))) != cudaSuccess)
                return cleanup(cuda_fail(e, "cudaMalloc extraction"));
            double* Dax[3] = {D, D + q2 * S0, D + q2 * (S0 + S1)};
            for (int d = 0; d < 3; ++d) {
                const int nsp = (int)(nctrl[d] - p);
                bezier_tables_kernel<<<(nsp + 127) / 128, 128, 0, st>>>((const double*)((char*)Udev + uoff[d]), p, nsp,
                                                                       Dax[d]);
            }
            float* out = reinterpret_cast<float*>(m->Q);
            const int64_t Sd[3] = {S0, S1, S2};
            for (int d = 0; d < 3; ++d) m->mm[d] = (int)((Sd[d] + (1 << kMacroLog) - 1) >> kMacroLog);
            const int64_t nmac = (int64_t)m->mm[0] * m->mm[1] * m->mm[2];
            if ((e = cudaMalloc(&m->mmx, sizeof(unsigned) * 2 * nmac)) != cudaSuccess)
                return cleanup(cuda_fail(e, "cudaMalloc macro bounds"));
            init_minmax_kernel<<<(unsigned)std::min<int64_t>((nmac + 255) / 256, 4096), 256, 0, st>>>(m->mmx, nmac);
            m->device_bytes += sizeof(unsigned) * 2 * nmac;
            switch (p) {
                case 1: bezier_blocks_kernel<1><<<4736, 128, 0, st>>>(Pdev, (int)nu, (int)nv, Dax[0], Dax[1], Dax[2], (int)S0, (int)S1, nblk, out, m->mmx, m->mm[0], m->mm[1]); break;
                case 2: bezier_blocks_kernel<2><<<4736, 128, 0, st>>>(Pdev, (int)nu, (int)nv, Dax[0], Dax[1], Dax[2], (int)S0, (int)S1, nblk, out, m->mmx, m->mm[0], m->mm[1]); break;
                default: (grouped ? bezier_blocks_kernel<3, true> : bezier_blocks_kernel<3, false>)<<<4736, 128, 0, st>>>(Pdev, (int)nu, (int)nv, Dax[0], Dax[1], Dax[2], (int)S0, (int)S1, nblk, out, m->mmx, m->mm[0], m->mm[1]); break;
            }
            cudaStreamSynchronize(st);
            cudaFree(D);
            m->device_bytes += nblk_alloc * bfl * (int64_t)sizeof(float);
            m->q_f4 = nblk_alloc * bfl / 4;
            m->layout = grouped ? kBezierG : kBezier;
        }
    }
    if (!bez && want_layout == MFA_LAYOUT_BRICKS) {   // plain haloed bricks (<= 1.86 x the grid)
        for (int d = 0; d < 3; ++d) m->nb[d] = (int)((nctrl[d] - p + kBrick - 1) / kBrick);
        const int EU = pbrick_eu(p), EV = pbrick_ev(p);
        const int64_t fl = (int64_t)m->nb[0] * m->nb[1] * m->nb[2] * EU * EV * EV;   // floats
        if ((e = cudaMalloc(&m->Q, fl * sizeof(float) + 32)) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc Q"));
        relayout_plain_kernel<<<4736, 256, 0, st>>>(Pdev, reinterpret_cast<float*>(m->Q), (int)nu, (int)nv, (int)nw,
                                                     m->nb[0], m->nb[1], EU, EV, fl);
        cudaMemsetAsync(reinterpret_cast<float*>(m->Q) + fl, 0, 32, st);   // the 8-float row window may read past the end
        m->device_bytes += fl * (int64_t)sizeof(float) + 32;
        m->q_f4 = (fl + 8) / 4;
        m->layout = kBricks;
    } else if (!bez) {   // bricked row quads
        for (int d = 0; d < 3; ++d) m->nb[d] = (int)((nctrl[d] - p + kBrick - 1) / kBrick);
        const int EU = brick_eu(p), EV = brick_ev(p), EW = brick_ev(p);
        const int64_t qn = (int64_t)m->nb[0] * m->nb[1] * m->nb[2] * EU * EV * EW;   // entries
        const int f4 = quad_f4(p);
        if ((e = cudaMalloc(&m->Q, qn * f4 * sizeof(float4))) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc Q"));
        relayout_bricks_kernel<<<4736, 256, 0, st>>>(Pdev, m->Q, (int)nu, (int)nv, (int)nw, m->nb[0], m->nb[1], EU, EV,
                                                      EW, qn, quad_pairs(p) ? 1 : 0);
        m->device_bytes += qn * f4 * (int64_t)sizeof(float4);
        m->q_f4 = qn * f4;
        m->layout = kQuads;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return cleanup(cuda_fail(e, "layout kernels"));
    unsigned int hmm[3];
    if ((e = cudaMemcpyAsync(hmm, mm, sizeof(hmm), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return cleanup(cuda_fail(e, "copy range"));
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cleanup(cuda_fail(e, "model ingest"));
    if (hmm[2] != 0)
        return cleanup(fail(MFA_ERR_DOMAIN, std::to_string(hmm[2]) + " non-finite control values"));
    m->vmin = ord2f(hmm[0]);
    m->vmax = ord2f(hmm[1]);
    m->model_bytes = npts * (int64_t)sizeof(float);
    m->create_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_create).count();
    cleanup(MFA_OK);
    *out = reinterpret_cast<mfa_model>(m);
    return MFA_OK;
}

extern "C" mfa_status mfa_model_create(const int32_t degree[3], const int64_t nctrl[3], const double* const knots[3],
                                       const float* ctrl, int32_t ctrl_on_device, mfa_stream stream,
                                       mfa_model* out) {
    return mfa_model_create_ex(degree, nctrl, knots, ctrl, ctrl_on_device, nullptr, stream, out);
}

extern "C" mfa_status mfa_model_info(mfa_model h, mfa_model_desc* out) {
    if (!h || !out) return fail(MFA_ERR_INVALID_ARG, "NULL argument");
    const Model* m = reinterpret_cast<const Model*>(h);
    for (int d = 0; d < 3; ++d) {
        out->degree[d] = m->p;
        out->nctrl[d] = m->n[d];
        out->uniform[d] = m->uniform[d];
    }
    out->v_min = m->vmin;
    out->v_max = m->vmax;
    out->device_bytes = m->device_bytes;
    out->device = m->device;
    out->layout = m->layout == kBezier    ? MFA_LAYOUT_BEZIER
                  : m->layout == kBezierG ? MFA_LAYOUT_BEZIER_GROUPED
                  : m->layout == kBricks  ? MFA_LAYOUT_BRICKS
                                          : MFA_LAYOUT_QUADS;
    out->model_bytes = m->model_bytes;
    out->create_ms = m->create_ms;
    return MFA_OK;
}

extern "C" mfa_status mfa_model_destroy(mfa_model h) {
    if (!h) return MFA_OK;
    Model* m = reinterpret_cast<Model*>(h);
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != m->device) cudaSetDevice(m->device);
    free_model_resources(m);
    if (m->Q) cudaFree(m->Q);
    if (m->mmx) cudaFree(m->mmx);
    if (m->queue) cudaFree(m->queue);
    if (m->table_mem) cudaFree(m->table_mem);
    if (cur != m->device && cur >= 0) cudaSetDevice(cur);
    delete m;
    return MFA_OK;
}

extern "C" mfa_status mfa_eval_batch(mfa_model h, int64_t n, const float* u, const float* v, const float* w,
                                     float* value, float* du, float* dv, float* dw,
                                     unsigned long long* n_domain_errors, mfa_stream stream) {
    if (!h) return fail(MFA_ERR_INVALID_ARG, "model is NULL");
    if (n < 0) return fail(MFA_ERR_INVALID_ARG, "n < 0");
    if (n == 0) return MFA_OK;
    if (!u || !v || !w || !value) return fail(MFA_ERR_INVALID_ARG, "u, v, w and value are required");
    const int ng = (du != nullptr) + (dv != nullptr) + (dw != nullptr);
    if (ng != 0 && ng != 3) return fail(MFA_ERR_INVALID_ARG, "du, dv, dw must be all NULL or all non-NULL");
    const Model* m = reinterpret_cast<const Model*>(h);
    mfa_status s = check_device(m);
    if (s != MFA_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if (bin_worthwhile(m, n)) {
        // the binned path with stream-ordered scratch (no caller workspace)
        const size_t bytes = eval_workspace_bytes(m, n);
        void* ws = scratch_alloc(bytes, st);
        if (ws) {
            s = launch_eval(m, n, u, v, w, value, du, dv, dw, n_domain_errors, st, ws, bytes);
            cudaFreeAsync(ws, st);
            return s;
        }
    }
    return launch_eval(m, n, u, v, w, value, du, dv, dw, n_domain_errors, st);
}

// Stream-ordered scratch for the calls without a caller workspace
// (mfa_eval_batch, mfa_eval_hessian): cudaMallocAsync from the device's
// default memory pool, whose release threshold is raised once per device (to
// 8 GiB, as the encoder's) so freed blocks stay cached for the next call (no
// cudaMalloc / sync on the hot path).  NULL if the pool cannot serve it (the caller then runs the
// unbinned kernels).
void* mfa::scratch_alloc(size_t bytes, cudaStream_t st) {
    static std::mutex mu;
    static uint64_t warmed = 0;   // bit per device ordinal < 64
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 64 && !(warmed >> dev & 1)) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = 8ULL << 30;   // keep up to 8 GiB cached (the encoder's keep_pool uses the same)
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            warmed |= (uint64_t)1 << dev;
        }
    }
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

extern "C" size_t mfa_eval_workspace_bytes(mfa_model h, int64_t n) {
    if (!h || n < 0) return 0;
    return eval_workspace_bytes(reinterpret_cast<const Model*>(h), n);
}

extern "C" mfa_status mfa_eval_batch_ws(mfa_model h, int64_t n, const float* u, const float* v, const float* w,
                                        float* value, float* du, float* dv, float* dw,
                                        unsigned long long* n_domain_errors, void* workspace,
                                        size_t workspace_bytes, mfa_stream stream) {
    if (!h) return fail(MFA_ERR_INVALID_ARG, "model is NULL");
    if (n < 0) return fail(MFA_ERR_INVALID_ARG, "n < 0");
    if (n == 0) return MFA_OK;
    if (!u || !v || !w || !value) return fail(MFA_ERR_INVALID_ARG, "u, v, w and value are required");
    const int ng = (du != nullptr) + (dv != nullptr) + (dw != nullptr);
    if (ng != 0 && ng != 3) return fail(MFA_ERR_INVALID_ARG, "du, dv, dw must be all NULL or all non-NULL");
    const Model* m = reinterpret_cast<const Model*>(h);
    if (workspace && workspace_bytes < eval_workspace_bytes(m, n))
        return fail(MFA_ERR_INVALID_ARG, "workspace smaller than mfa_eval_workspace_bytes()");
    mfa_status s = check_device(m);
    if (s != MFA_OK) return s;
    return launch_eval(m, n, u, v, w, value, du, dv, dw, n_domain_errors, (cudaStream_t)stream, workspace,
                       workspace_bytes);
}

static mfa_status validate_render(const Model* m, int32_t n_views, const mfa_camera* cams,
                                  const mfa_render_params* prm) {
    if (n_views < 1) return fail(MFA_ERR_INVALID_ARG, "n_views < 1");
    if (!cams || !prm) return fail(MFA_ERR_INVALID_ARG, "cams and prm are required");
    for (int v = 0; v < n_views; ++v) {
        const mfa_camera& c = cams[v];
        if (c.width < 1 || c.height < 1) return fail(MFA_ERR_INVALID_ARG, "camera " + std::to_string(v) + ": size < 1");
        if (c.width != cams[0].width || c.height != cams[0].height)
            return fail(MFA_ERR_INVALID_ARG, "all views of one call must share width and height");
        if (!(c.fov_y_deg >= 0.0 && c.fov_y_deg < 180.0))
            return fail(MFA_ERR_INVALID_ARG, "camera " + std::to_string(v) + ": fov_y_deg outside [0,180)");
        if (c.fov_y_deg == 0.0 && !(c.ortho_half_height > 0.0))
            return fail(MFA_ERR_INVALID_ARG, "camera " + std::to_string(v) + ": ortho_half_height <= 0");
        double f[3] = {c.look_at[0] - c.eye[0], c.look_at[1] - c.eye[1], c.look_at[2] - c.eye[2]};
        double x[3] = {f[1] * c.up[2] - f[2] * c.up[1], f[2] * c.up[0] - f[0] * c.up[2], f[0] * c.up[1] - f[1] * c.up[0]};
        double lf = sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
        double lx = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
        if (!(lf > 0.0) || !(lx > 1e-12 * lf))
            return fail(MFA_ERR_INVALID_ARG, "camera " + std::to_string(v) + ": degenerate eye/look_at/up");
    }
    for (int d = 0; d < 3; ++d)
        if (!(prm->box_max[d] > prm->box_min[d])) return fail(MFA_ERR_INVALID_ARG, "box_max <= box_min");
    if (!(prm->step > 0.0)) return fail(MFA_ERR_INVALID_ARG, "step <= 0");
    {   // the per-ray sample count must fit an int: box diagonal / step < 2^30
        double d2 = 0.0;
        for (int d = 0; d < 3; ++d) d2 += (prm->box_max[d] - prm->box_min[d]) * (prm->box_max[d] - prm->box_min[d]);
        if (!(sqrt(d2) / prm->step < 1073741824.0))
            return fail(MFA_ERR_INVALID_ARG, "step too small: box diagonal / step must stay below 2^30 samples");
    }
    (void)m;
    return MFA_OK;
}

extern "C" mfa_status mfa_render(mfa_model h, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                                 const mfa_render_params* prm, const mfa_tiles* tiles, void* rgba_out,
                                 unsigned long long* samples_out, mfa_stream stream) {
    return mfa_render_ex(h, n_views, cams, tf, prm, nullptr, tiles, rgba_out, samples_out, stream);
}

extern "C" mfa_status mfa_render_field(mfa_model h, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                                       const mfa_render_params* prm, const mfa_field* field, const mfa_tiles* tiles,
                                       void* rgba_out, unsigned long long* samples_out, mfa_stream stream) {
    mfa_render_ext ext{field, 0, nullptr, nullptr, nullptr, 0, 0.0};
    return mfa_render_ex(h, n_views, cams, tf, prm, &ext, tiles, rgba_out, samples_out, stream);
}

extern "C" mfa_status mfa_render_ex(mfa_model h, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                                    const mfa_render_params* prm, const mfa_render_ext* ext, const mfa_tiles* tiles,
                                    void* rgba_out, unsigned long long* samples_out, mfa_stream stream) {
    if (!h) return fail(MFA_ERR_INVALID_ARG, "model is NULL");
    const mfa_field* field = ext ? ext->field : nullptr;
    if (field && (field->value_src || field->grad_src) &&
        !(field->kind == MFA_FIELD_GAUSSIAN_BEAM || field->kind == MFA_FIELD_MARSCHNER_LOBB))
        return fail(MFA_ERR_INVALID_ARG, "field: unknown kind");
    if (field && field->kind == MFA_FIELD_GAUSSIAN_BEAM && !(field->prm[3] > 0.0 && field->prm[4] > 0.0))
        return fail(MFA_ERR_INVALID_ARG, "field: Gaussian beam needs sigma > 0 and R > 0");
    if (ext && ext->n_lights) {
        if (ext->n_lights < 0 || ext->n_lights > MFA_MAX_LIGHTS)
            return fail(MFA_ERR_INVALID_ARG, "n_lights must be in [0, MFA_MAX_LIGHTS]");
        if (!ext->light_dir || !ext->light_intensity) return fail(MFA_ERR_INVALID_ARG, "light arrays are NULL");
        for (int l = 0; l < ext->n_lights; ++l) {
            const double* L = ext->light_dir + 3 * l;
            const double n2 = L[0] * L[0] + L[1] * L[1] + L[2] * L[2];
            if (!(n2 > 0.0) || !isfinite(n2) || !isfinite(ext->light_intensity[l]))
                return fail(MFA_ERR_INVALID_ARG, "light " + std::to_string(l) + ": zero or non-finite direction/intensity");
        }
    }
    if (ext && ext->curv_n && (ext->curv_n < 2 || !ext->curv_rgba || !(ext->curv_range > 0.0)))
        return fail(MFA_ERR_INVALID_ARG, "curvature TF: need curv_n >= 2, a table and curv_range > 0");
    const Model* m = reinterpret_cast<const Model*>(h);
    mfa_status s = validate_render(m, n_views, cams, prm);
    if (s != MFA_OK) return s;
    if (!tf || !tf->rgba || tf->n_entries < 2 || tf->n_entries > 1024 || !(tf->v_hi > tf->v_lo))
        return fail(MFA_ERR_INVALID_ARG, "tf: need rgba, 2 <= n_entries <= 1024, v_hi > v_lo");
    if (tiles && (tiles->n_tiles < 0 || (tiles->n_tiles > 0 && !tiles->tiles)))
        return fail(MFA_ERR_INVALID_ARG, "tiles: bad n_tiles / tiles pointer");
    if (tiles && tiles->n_tiles == 0) return MFA_OK;   // an empty tile list is valid (nothing to do)
    if (!rgba_out) return fail(MFA_ERR_INVALID_ARG, "rgba_out is NULL");
    if ((s = check_device(m)) != MFA_OK) return s;
    return launch_render(m, n_views, cams, tf, prm, tiles, rgba_out, samples_out, (cudaStream_t)stream, ext);
}

extern "C" mfa_status mfa_enable_peer_access(int32_t peer_device) {
    int cur = -1, can = 0;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (peer_device == cur) return MFA_OK;
    if ((e = cudaDeviceCanAccessPeer(&can, cur, peer_device)) != cudaSuccess) return cuda_fail(e, "cudaDeviceCanAccessPeer");
    if (!can) return fail(MFA_ERR_DEVICE, "device " + std::to_string(cur) + " cannot access peer " + std::to_string(peer_device));
    e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return MFA_OK;
    }
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "cudaDeviceEnablePeerAccess");
}

extern "C" mfa_status mfa_ipc_open(const void* handle, void** base_out) {
    if (!handle || !base_out) return fail(MFA_ERR_INVALID_ARG, "mfa_ipc_open: NULL handle or base_out");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    *base_out = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

extern "C" mfa_status mfa_ipc_alloc(size_t bytes, void** ptr_out, void* handle_out) {
    if (!ptr_out || !handle_out || bytes == 0) return fail(MFA_ERR_INVALID_ARG, "mfa_ipc_alloc: NULL output or 0 bytes");
    *ptr_out = nullptr;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(MFA_ERR_OOM, std::string("mfa_ipc_alloc: cudaMalloc: ") + cudaGetErrorString(e));
    }
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, p)) != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    std::memcpy(handle_out, &h, sizeof h);
    *ptr_out = p;
    return MFA_OK;
}

extern "C" mfa_status mfa_ipc_free(void* ptr) {
    if (!ptr) return fail(MFA_ERR_INVALID_ARG, "mfa_ipc_free: NULL");
    const cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "cudaFree");
}

extern "C" mfa_status mfa_ipc_close(void* base) {
    if (!base) return fail(MFA_ERR_INVALID_ARG, "mfa_ipc_close: NULL base");
    const cudaError_t e = cudaIpcCloseMemHandle(base);
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

extern "C" mfa_status mfa_unpack_tiles(const void* packed, int32_t in_fp16, const int32_t* tiles, int64_t n_tiles,
                                       int32_t n_views, int32_t width, int32_t height, float* image_out,
                                       mfa_stream stream) {
    if (n_tiles < 0 || n_views < 1 || width < 1 || height < 1) return fail(MFA_ERR_INVALID_ARG, "bad sizes");
    if (n_tiles == 0) return MFA_OK;
    if (!packed || !tiles || !image_out) return fail(MFA_ERR_INVALID_ARG, "NULL pointer");
    unpack_tiles_kernel<<<(unsigned)n_tiles, MFA_TILE * MFA_TILE, 0, (cudaStream_t)stream>>>(
        packed, in_fp16, tiles, n_tiles, n_views, width, height, reinterpret_cast<float4*>(image_out));
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "unpack_tiles launch");
}

// mfa_render_host / mfa_render_host_views: per view, render into one of two
// model-owned staging buffers on the caller's stream while the copy stream
// moves the previous view to the host (D2H of view v overlaps the render of
// view v+1).  The staging buffers, events, copy stream, TF and counter are
// created on first use and reused (Model::host, one host-buffer render per
// model at a time).
static mfa_status render_host_impl(const Model* m, int32_t n_views, const mfa_camera* cams, const float* tf_rgba_host,
                                   int32_t tf_n_entries, float v_lo, float v_hi, const mfa_render_params* prm,
                                   void* const* dst, unsigned long long* samples_host, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(m->host_mu);
    Model::HostRes& H = m->host;
    const size_t px = (size_t)cams[0].width * cams[0].height;
    const size_t view_bytes = px * (prm->out_fp16 ? 8 : 16);
    cudaError_t e;
    // each resource on its own: a call that failed half way (out of memory)
    // leaves the rest to the next one
    if (!H.copy && (e = cudaStreamCreateWithFlags(&H.copy, cudaStreamNonBlocking)) != cudaSuccess) {
        H.copy = nullptr;
        return cuda_fail(e, "stream");
    }
    for (int i = 0; i < 2; ++i) {
        if (!H.rendered[i] && (e = cudaEventCreateWithFlags(&H.rendered[i], cudaEventDisableTiming)) != cudaSuccess) {
            H.rendered[i] = nullptr;
            return cuda_fail(e, "event");
        }
        if (!H.copied[i] && (e = cudaEventCreateWithFlags(&H.copied[i], cudaEventDisableTiming)) != cudaSuccess) {
            H.copied[i] = nullptr;
            return cuda_fail(e, "event");
        }
    }
    if (!H.tf && (e = cudaMalloc((void**)&H.tf, sizeof(float) * 4 * 1024)) != cudaSuccess) {
        H.tf = nullptr;
        return cuda_fail(e, "tf");
    }
    if (!H.cnt && (e = cudaMalloc((void**)&H.cnt, sizeof(unsigned long long))) != cudaSuccess) {
        H.cnt = nullptr;
        return cuda_fail(e, "count");
    }
    if (H.stage_bytes < view_bytes) {
        cudaStreamSynchronize(H.copy);
        for (int i = 0; i < 2; ++i) {
            if (H.stage[i]) cudaFree(H.stage[i]);
            H.stage[i] = nullptr;
        }
        H.stage_bytes = 0;
        for (int i = 0; i < 2; ++i)
            if ((e = cudaMalloc(&H.stage[i], view_bytes)) != cudaSuccess) return cuda_fail(e, "staging");
        H.stage_bytes = view_bytes;
    }
    // the previous call's copies are complete (it synchronised); order this
    // call's uploads after the caller's earlier work on st
    cudaMemcpyAsync(H.tf, tf_rgba_host, sizeof(float) * 4 * tf_n_entries, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(H.cnt, 0, sizeof(unsigned long long), st);
    mfa_tf tf{H.tf, tf_n_entries, v_lo, v_hi};
    mfa_status s = MFA_OK;
    for (int v = 0; v < n_views; ++v) {
        const int b = v & 1;
        if (v >= 2) cudaStreamWaitEvent(st, H.copied[b], 0);  // staging buffer b free again
        s = launch_render(m, 1, cams + v, &tf, prm, nullptr, H.stage[b], H.cnt, st);
        if (s != MFA_OK) break;
        cudaEventRecord(H.rendered[b], st);
        cudaStreamWaitEvent(H.copy, H.rendered[b], 0);
        cudaMemcpyAsync(dst[v], H.stage[b], view_bytes, cudaMemcpyDeviceToHost, H.copy);
        cudaEventRecord(H.copied[b], H.copy);
    }
    if (s == MFA_OK && samples_host) {
        cudaStreamWaitEvent(st, H.copied[(n_views - 1) & 1], 0);
        cudaMemcpyAsync(samples_host, H.cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    }
    cudaStreamSynchronize(H.copy);
    cudaStreamSynchronize(st);
    if (s == MFA_OK && (e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "render_host");
    return s;
}

static mfa_status render_host_check(mfa_model h, int32_t n_views, const mfa_camera* cams, const float* tf_rgba_host,
                                    int32_t tf_n_entries, float v_lo, float v_hi, const mfa_render_params* prm,
                                    const void* dst) {
    if (!h) return fail(MFA_ERR_INVALID_ARG, "model is NULL");
    const Model* m = reinterpret_cast<const Model*>(h);
    mfa_status s = validate_render(m, n_views, cams, prm);
    if (s != MFA_OK) return s;
    if (!tf_rgba_host || tf_n_entries < 2 || tf_n_entries > 1024 || !(v_hi > v_lo) || !dst)
        return fail(MFA_ERR_INVALID_ARG, "tf / rgba_host");
    return check_device(m);
}

extern "C" mfa_status mfa_render_host(mfa_model h, int32_t n_views, const mfa_camera* cams, const float* tf_rgba_host,
                                      int32_t tf_n_entries, float v_lo, float v_hi, const mfa_render_params* prm,
                                      void* rgba_host, unsigned long long* samples_host, mfa_stream stream) {
    mfa_status s = render_host_check(h, n_views, cams, tf_rgba_host, tf_n_entries, v_lo, v_hi, prm, rgba_host);
    if (s != MFA_OK) return s;
    const size_t view_bytes = (size_t)cams[0].width * cams[0].height * (prm->out_fp16 ? 8 : 16);
    std::vector<void*> dst((size_t)n_views);
    for (int v = 0; v < n_views; ++v) dst[v] = (char*)rgba_host + v * view_bytes;
    return render_host_impl(reinterpret_cast<const Model*>(h), n_views, cams, tf_rgba_host, tf_n_entries, v_lo, v_hi,
                            prm, dst.data(), samples_host, (cudaStream_t)stream);
}

extern "C" mfa_status mfa_render_host_views(mfa_model h, int32_t n_views, const mfa_camera* cams,
                                            const float* tf_rgba_host, int32_t tf_n_entries, float v_lo, float v_hi,
                                            const mfa_render_params* prm, void* const* rgba_host_views,
                                            unsigned long long* samples_host, mfa_stream stream) {
    mfa_status s = render_host_check(h, n_views, cams, tf_rgba_host, tf_n_entries, v_lo, v_hi, prm, rgba_host_views);
    if (s != MFA_OK) return s;
    for (int v = 0; v < n_views; ++v)
        if (!rgba_host_views[v]) return fail(MFA_ERR_INVALID_ARG, "rgba_host_views[" + std::to_string(v) + "] is NULL");
    return render_host_impl(reinterpret_cast<const Model*>(h), n_views, cams, tf_rgba_host, tf_n_entries, v_lo, v_hi,
                            prm, rgba_host_views, samples_host, (cudaStream_t)stream);
}
