// MFA encoder: least-squares fit of the control points
// of a tensor-product B-spline to a structured grid, and the adaptive loop of
// Fig. 1 ("New control points and knots are added adaptively until all
// evaluated points in each span of knots are within the allowable maximum
// relative error of the original points ... knot spans that fall beyond the
// tolerance are subdivided, and MFA is recomputed").
//
// Fit (R-27): grid samples at uniform parameters t_j = j/(m-1) per axis; the
// least-squares solution of (N_w (x) N_v (x) N_u) c = q is separable,
// c = q x_u N_u^+ x_v N_v^+ x_w N_w^+ with N^+ = (N^T N)^{-1} N^T.  All on
// the device, hand-written (no cuBLAS):
//   K_fs  per sample j: span and the p+1 basis values (Cox-de Boor as power
//         polynomials per span, fp64) -- one thread per sample
//   K_fn  the banded normal matrix A = N^T N (bandwidth p), one thread per row
//         (samples in ascending order: deterministic sums)
//   K_fc  its banded Cholesky factor, one thread (n p^2 flops, sequential by
//         nature); a basis function without samples -> singular -> error
//   K_fm  the dense n x m operator N^+ = A^{-1} N^T: one thread per column j
//         (forward + backward banded substitution, p-wide register windows)
//   K_gemm the three axis passes as dense fp64 GEMMs over all grid lines (w
//         pass one GEMM, v pass a batch over the w slices, u pass one GEMM
//         with the operator transposed): 64x64 CTA tiles, 4x4 register tiles
//         per thread, k-slabs of 16 double-buffered in shared memory, DFMA on
//         the CUDA cores.  A dense operator costs 2 m n flops per line instead
//         of the banded solve's ~4 m p, but every line is independent; the
//         banded solve is a chain of 2n dependent steps per line.
//   fp32 <-> fp64 conversion kernels at the ends.
// Residual (adaptive loop): K_expand applies N along each axis (the spline
// at every grid sample, separable), K_err forms |v - q| / (max q - min q) and
// per-axis per-span maxima (atomicMax on the ordered bits of non-negative
// doubles); the host splits every span above e_max that holds >= 2(p+1) samples at
// its midpoint (R-28: every span keeps >= p+1 samples, so the normal equations
// stay regular), within the per-axis caps, and refits.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include <map>
#include <mutex>

#include "mfa_internal.cuh"

namespace mfa {

struct AxisFitDev {
    int m, n;
    const int* f;       // [m] first non-zero function at sample j (= local span)
    const double* B;    // [m][p+1] basis values N_{f_j + a}(t_j)
    const double* M;    // [n][m] dense N^+
};

// host: the knot span of parameter t (right-continuous; t = 1 -> last
// non-degenerate span); the adaptive loop's split rule counts samples per span
static int host_span(const double* U, int p, int n, double t) {
    if (t >= U[n]) {
        int i = n - 1;
        while (i > p && U[i] == U[n]) --i;
        return i;
    }
    int lo = p, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (t < U[mid]) hi = mid; else lo = mid;
    }
    return lo;
}

static std::vector<int> sample_spans(const double* U, int p, int n, int m) {
    std::vector<int> f(m);
    for (int j = 0; j < m; ++j) f[j] = host_span(U, p, n, (double)j / (double)(m - 1)) - p;
    return f;
}

// ---- K_fs: span and basis values of every sample ---------------------------
__global__ void fit_samples_kernel(const double* __restrict__ U, int p, int n, int m, int* __restrict__ f,
                                   double* __restrict__ B) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const double t = (double)j / (double)(m - 1);
    int span;
    if (t >= U[n]) {
        span = n - 1;
        while (span > p && U[span] == U[n]) --span;
    } else {
        int lo = p, hi = n;
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (t < U[mid]) hi = mid; else lo = mid;
        }
        span = lo;
    }
    double P[kMaxP + 1][kMaxP + 1];
    span_poly(U, p, span, P);
    const double x = (t - U[span]) / (U[span + 1] - U[span]);
    for (int a = 0; a <= p; ++a) {
        double v = P[a][p];
        for (int k = p - 1; k >= 0; --k) v = v * x + P[a][k];
        B[(size_t)j * (p + 1) + a] = v;
    }
    f[j] = span - p;
}

// first sample index j with f[j] >= key (f is nondecreasing in j)
__device__ __forceinline__ int lower_bound_f(const int* __restrict__ f, int m, int key) {
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (f[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// ---- K_fn: banded normal matrix Ab[r][k] = (N^T N)(r, r - k) ----------------
// entry (r, c = r - k) sums B[j][r - f_j] B[j][c - f_j] over the samples with
// f_j in [r - p, c], in ascending j (deterministic)
__global__ void fit_normal_kernel(const int* __restrict__ f, const double* __restrict__ B, int p, int n, int m,
                                  double* __restrict__ Ab) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    for (int k = 0; k <= p; ++k) {
        const int c = r - k;
        double acc = 0.0;
        if (c >= 0) {
            const int j1 = lower_bound_f(f, m, c + 1);
            for (int j = lower_bound_f(f, m, r - p); j < j1; ++j)
                acc += B[(size_t)j * (p + 1) + (r - f[j])] * B[(size_t)j * (p + 1) + (c - f[j])];
        }
        Ab[(size_t)r * (p + 1) + k] = acc;
    }
}

// ---- K_fc: banded Cholesky A = L L^T, L[i][k] = L(i, i - k) -----------------
// one thread per axis (blockIdx.x = axis: the three factorisations run
// concurrently); the last P rows of L stay in a register window and each row
// takes one reciprocal and one square root, so a row costs a few hundred
// cycles of dependent fp64 latency instead of a chain of global loads.
// status[axis] = -1 on success, else the first control point whose pivot failed
struct CholArgs {
    const double* Ab[3];
    double* L[3];
    int n[3];
    int* status;
};

template <int P>
__global__ void fit_cholesky_kernel(const CholArgs a) {
    if (threadIdx.x != 0) return;
    const int ax = blockIdx.x;
    const double* __restrict__ Ab = a.Ab[ax];
    double* __restrict__ L = a.L[ax];
    const int n = a.n[ax];
    // win[q][k] = L(i-1-q, i-1-q-k) for the previous P rows (q = 0 is row i-1);
    // inv[q] = 1 / L(i-1-q, i-1-q)
    double win[P][P + 1], inv[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
        inv[q] = 0.0;
#pragma unroll
        for (int k = 0; k <= P; ++k) win[q][k] = 0.0;
    }
    a.status[ax] = -1;
    for (int i = 0; i < n; ++i) {
        double row[P + 1];   // row[k] = L(i, i - k)
        // off-diagonal entries c = i - k, k = P .. 1 (ascending c)
#pragma unroll
        for (int k = P; k >= 1; --k) {
            row[k] = 0.0;
            if (i - k < 0) continue;
            double sum = Ab[(size_t)i * (P + 1) + k];
            const int q = k - 1;   // row c = i - k is window entry q
            // l = c - kk .. for l in [max(0, i - P), c - 1]: L(i, l) = row[i - l], L(c, l) = win[q][c - l]
#pragma unroll
            for (int j = P; j > k; --j) {   // l = i - j (ascending l), needs l >= 0 and l < c
                if (i - j >= 0) sum -= row[j] * win[q][j - k];
            }
            row[k] = sum * inv[q];
        }
        double d = Ab[(size_t)i * (P + 1)];
#pragma unroll
        for (int k = P; k >= 1; --k)
            if (i - k >= 0) d -= row[k] * row[k];
        if (!(d > 1e-14 * fmax(1.0, Ab[(size_t)i * (P + 1)]))) {
            a.status[ax] = i;
            return;
        }
        row[0] = sqrt(d);
#pragma unroll
        for (int k = 0; k <= P; ++k) L[(size_t)i * (P + 1) + k] = row[k];
#pragma unroll
        for (int q = P - 1; q > 0; --q) {
            inv[q] = inv[q - 1];
#pragma unroll
            for (int k = 0; k <= P; ++k) win[q][k] = win[q - 1][k];
        }
        inv[0] = 1.0 / row[0];
#pragma unroll
        for (int k = 0; k <= P; ++k) win[0][k] = row[k];
    }
}

// ---- K_fm: N^+ = A^{-1} N^T, one thread per column j --------------------------
// column j of N^T has p+1 entries B[j][a] at rows f_j + a; forward substitution
// from row f_j (rows above are 0), then backward over all rows; a p-wide
// window of the latest results stays in registers
template <int P>
__global__ void fit_pinv_kernel(const int* __restrict__ f, const double* __restrict__ B, const double* __restrict__ L,
                                int n, int m, double* __restrict__ M) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int fj = f[j];
    for (int i = 0; i < fj; ++i) M[(size_t)i * m + j] = 0.0;
    double win[P + 1];   // win[q] = y_{i-1-q}
#pragma unroll
    for (int q = 0; q <= P; ++q) win[q] = 0.0;
    for (int i = fj; i < n; ++i) {
        double sum = (i - fj <= P) ? B[(size_t)j * (P + 1) + (i - fj)] : 0.0;
        // L(i, l) for l = i-P .. i-1 (ascending l, as the row-wise host order)
#pragma unroll
        for (int q = P - 1; q >= 0; --q) {
            const int l = i - 1 - q;
            if (l >= fj) sum -= L[(size_t)i * (P + 1) + (i - l)] * win[q];
        }
        const double y = sum / L[(size_t)i * (P + 1)];
#pragma unroll
        for (int q = P; q > 0; --q) win[q] = win[q - 1];
        win[0] = y;
        M[(size_t)i * m + j] = y;
    }
#pragma unroll
    for (int q = 0; q <= P; ++q) win[q] = 0.0;   // win[q] = x_{i+1+q}
    for (int i = n - 1; i >= 0; --i) {
        double sum = M[(size_t)i * m + j];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const int l = i + 1 + q;
            if (l < n) sum -= L[(size_t)l * (P + 1) + (l - i)] * win[q];
        }
        const double x = sum / L[(size_t)i * (P + 1)];
#pragma unroll
        for (int q = P; q > 0; --q) win[q] = win[q - 1];
        win[0] = x;
        M[(size_t)i * m + j] = x;
    }
}

__global__ void f32_to_f64_kernel(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (double)a[i];
}

__global__ void f64_to_f32_kernel(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

// the spline along one axis at the grid samples: out_j = sum_a N_{f_j+a}(t_j) in_{f_j+a}
template <int P>
__global__ void __launch_bounds__(128) expand_axis_kernel(const double* __restrict__ X, double* __restrict__ Y,
                                                          const AxisFitDev ax, int64_t n_outer, int64_t inner) {
    const int64_t total = n_outer * ax.m * inner;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t in = idx % inner;
        const int64_t rest = idx / inner;
        const int j = (int)(rest % ax.m);
        const int64_t o = rest / ax.m;
        const int f = __ldg(ax.f + j);
        const double* x = X + (o * ax.n + f) * inner + in;
        double v = 0.0;
#pragma unroll
        for (int a = 0; a <= P; ++a) v = fma(__ldg(ax.B + j * (P + 1) + a), x[a * inner], v);
        Y[idx] = v;
    }
}

__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }

// relative errors at the samples: per-axis per-span maxima, global max, sum of squares
__global__ void grid_error_kernel(const double* __restrict__ V, const float* __restrict__ Q, int mu, int mv, int mw,
                                  double inv_range, const int* __restrict__ fu, const int* __restrict__ fv,
                                  const int* __restrict__ fw, unsigned long long* __restrict__ eu,
                                  unsigned long long* __restrict__ ev, unsigned long long* __restrict__ ew,
                                  unsigned long long* __restrict__ emax, double* __restrict__ esq, int S0, int S1,
                                  int nspan_total) {
    // per-CTA span maxima in shared memory (one global atomic per span per CTA)
    // when the three span tables fit, else straight to global memory
    extern __shared__ unsigned long long smax[];
    const bool local = nspan_total > 0;
    unsigned long long *su = smax, *sv = smax + S0, *sw = smax + S0 + S1;
    if (local)
        for (int b = threadIdx.x; b < nspan_total; b += blockDim.x) smax[b] = 0ULL;
    __syncthreads();
    const int64_t total = (int64_t)mu * mv * mw;
    double sq = 0.0, mx = 0.0;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % mu);
        const int j = (int)((idx / mu) % mv);
        const int k = (int)(idx / ((int64_t)mu * mv));
        const double e = fabs(V[idx] - (double)Q[idx]) * inv_range;
        sq += e * e;
        mx = fmax(mx, e);
        const unsigned long long eb = dbits(e);
        if (local) {
            atomicMax(su + __ldg(fu + i), eb);
            atomicMax(sv + __ldg(fv + j), eb);
            atomicMax(sw + __ldg(fw + k), eb);
        } else {
            atomicMax(eu + __ldg(fu + i), eb);
            atomicMax(ev + __ldg(fv + j), eb);
            atomicMax(ew + __ldg(fw + k), eb);
        }
    }
    __syncthreads();
    if (local)
        for (int b = threadIdx.x; b < nspan_total; b += blockDim.x)
            if (smax[b]) atomicMax(eu + b, smax[b]);   // eu, ev, ew are contiguous like smax
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(esq, sq);
        atomicMax(emax, dbits(mx));
    }
}

// value range of the grid (ordered-bits min / max in out[0..1]) and the
// number of non-finite samples (out[2], as an unsigned long long)
__global__ void range_kernel(const float* __restrict__ Q, int64_t n, double* __restrict__ out /*min,max,bad*/) {
    double lo = INFINITY, hi = -INFINITY;
    unsigned bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float q = Q[i];
        bad += !isfinite(q);
        lo = fmin(lo, (double)q);
        hi = fmax(hi, (double)q);
    }
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(reinterpret_cast<unsigned long long*>(out) + 2, (unsigned long long)bad);
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {   // ordered-bits trick: negate for the minimum of possibly negative values
        const unsigned long long blo = dbits(lo), bhi = dbits(hi);
        atomicMin(reinterpret_cast<unsigned long long*>(out) + 0,
                  (blo & 0x8000000000000000ULL) ? ~blo : (blo | 0x8000000000000000ULL));
        atomicMax(reinterpret_cast<unsigned long long*>(out) + 1,
                  (bhi & 0x8000000000000000ULL) ? ~bhi : (bhi | 0x8000000000000000ULL));
    }
}

static double ord_to_double(unsigned long long u) {
    const unsigned long long b = (u & 0x8000000000000000ULL) ? (u & 0x7fffffffffffffffULL) : ~u;
    double d;
    memcpy(&d, &b, 8);
    return d;
}

// one axis' device tables (one stream-ordered allocation; the pool makes
// repeated fits cheap)
struct AxisDevMem {
    void* mem = nullptr;
    AxisFitDev d{};
    void release(cudaStream_t st) {
        if (mem) cudaFreeAsync(mem, st);
        mem = nullptr;
    }
};

// the operators of the three axes on the device: samples, normal matrix,
// Cholesky (one launch for all axes), N^+ (K_fs, K_fn, K_fc, K_fm);
// synchronises once to report a singular fit
static mfa_status build_axes_dev(const int m[3], const int n[3], int p, const double* const U_host[3],
                                 AxisDevMem (&D)[3], cudaStream_t st) {
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    CholArgs ca;
    int* status = nullptr;
    cudaError_t e;
    int* f[3];
    double* B[3];
    double* M[3];
    for (int d = 0; d < 3; ++d) {
        const size_t nu = sizeof(double) * (n[d] + p + 1), nf = sizeof(int) * m[d],
                     nb = sizeof(double) * (size_t)m[d] * (p + 1), nab = sizeof(double) * (size_t)n[d] * (p + 1),
                     nm = sizeof(double) * (size_t)n[d] * m[d];
        if ((e = cudaMallocAsync(&D[d].mem, up(nu) + up(nf) + up(nb) + 2 * up(nab) + up(nm) + 256, st)) != cudaSuccess)
            return cuda_fail(e, "fit tables");
        char* b = (char*)D[d].mem;
        double* U = (double*)b;
        f[d] = (int*)(b + up(nu));
        B[d] = (double*)(b + up(nu) + up(nf));
        double* Ab = (double*)(b + up(nu) + up(nf) + up(nb));
        double* L = (double*)(b + up(nu) + up(nf) + up(nb) + up(nab));
        M[d] = (double*)(b + up(nu) + up(nf) + up(nb) + 2 * up(nab));
        if (d == 0) status = (int*)(b + up(nu) + up(nf) + up(nb) + 2 * up(nab) + up(nm));
        cudaMemcpyAsync(U, U_host[d], nu, cudaMemcpyHostToDevice, st);
        fit_samples_kernel<<<(m[d] + 127) / 128, 128, 0, st>>>(U, p, n[d], m[d], f[d], B[d]);
        fit_normal_kernel<<<(n[d] + 127) / 128, 128, 0, st>>>(f[d], B[d], p, n[d], m[d], Ab);
        ca.Ab[d] = Ab;
        ca.L[d] = L;
        ca.n[d] = n[d];
    }
    ca.status = status;
    switch (p) {
        case 1: fit_cholesky_kernel<1><<<3, 32, 0, st>>>(ca); break;
        case 2: fit_cholesky_kernel<2><<<3, 32, 0, st>>>(ca); break;
        case 3: fit_cholesky_kernel<3><<<3, 32, 0, st>>>(ca); break;
        case 4: fit_cholesky_kernel<4><<<3, 32, 0, st>>>(ca); break;
        default: fit_cholesky_kernel<5><<<3, 32, 0, st>>>(ca); break;
    }
    for (int d = 0; d < 3; ++d) {
        const unsigned g = (unsigned)((m[d] + 127) / 128);
        switch (p) {
            case 1: fit_pinv_kernel<1><<<g, 128, 0, st>>>(f[d], B[d], ca.L[d], n[d], m[d], M[d]); break;
            case 2: fit_pinv_kernel<2><<<g, 128, 0, st>>>(f[d], B[d], ca.L[d], n[d], m[d], M[d]); break;
            case 3: fit_pinv_kernel<3><<<g, 128, 0, st>>>(f[d], B[d], ca.L[d], n[d], m[d], M[d]); break;
            case 4: fit_pinv_kernel<4><<<g, 128, 0, st>>>(f[d], B[d], ca.L[d], n[d], m[d], M[d]); break;
            default: fit_pinv_kernel<5><<<g, 128, 0, st>>>(f[d], B[d], ca.L[d], n[d], m[d], M[d]); break;
        }
    }
    int hs[3] = {-1, -1, -1};
    cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "fit operator");
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fit operator kernels");
    for (int d = 0; d < 3; ++d) {
        if (hs[d] >= 0)
            return fail(MFA_ERR_INVALID_ARG, std::string("fit: normal equations singular on axis ") + "uvw"[d] +
                                                 " at control point " + std::to_string(hs[d]) +
                                                 " (a basis function without samples: too many control points for the grid)");
        D[d].d = AxisFitDev{m[d], n[d], f[d], B[d], M[d]};
    }
    return MFA_OK;
}

// Keep the device's default stream-ordered pool from returning memory to the
// driver at every synchronisation, so repeated fits / refinement rounds reuse
// their scratch instead of re-mapping it (once per device).
static void keep_pool() {
    static std::mutex mu;
    static std::map<int, bool> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = 8ULL << 30;   // keep up to 8 GiB cached
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

static unsigned grid_for(int64_t work) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 127) / 128, (int64_t)sms * 16));
}

// ---- K_gemm: C[z][M][N] = A[z][M][K] . op(B)[z][K][N], fp64, row-major -----
// op(B) = B[K][N] (BT = false) or B^T with B stored [N][K] (BT = true).
// 128 x 64 tile per 256-thread CTA, each thread an 8 x 4 register tile (32
// DFMA per 6 shared-memory 16-byte loads); k-slabs of 16 staged through
// shared memory, double-buffered (the next slab's global loads are in flight
// while the current one is multiplied).  Batch z via blockIdx.z with element
// strides sa, sb, sc (0 = shared operand).
constexpr int kGM = 128, kGN = 64, kGK = 16;

template <bool BT>
__global__ void __launch_bounds__(256) dgemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                    double* __restrict__ C, int M, int N, int K, int64_t sa,
                                                    int64_t sb, int64_t sc) {
    extern __shared__ __align__(16) double gsm[];             // dynamic: 50 KB (opt-in above 48 KB)
    double (*As)[kGK][kGM + 2] = reinterpret_cast<double (*)[kGK][kGM + 2]>(gsm);                   // As[b][k][m]
    double (*Bs)[kGK][kGN + 2] = reinterpret_cast<double (*)[kGK][kGN + 2]>(gsm + 2 * kGK * (kGM + 2));   // Bs[b][k][n]
    const int z = blockIdx.z;
    A += z * sa;
    B += z * sb;
    C += z * sc;
    const int m0 = blockIdx.y * kGM, n0 = blockIdx.x * kGN;
    const int tid = threadIdx.x;
    const int tm = (tid / 16) * 8, tn = (tid % 16) * 4;
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    double ra[8], rb[4];
    auto load = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {   // A tile 128 (m) x 16 (k), k fastest in memory
            const int e = tid + 256 * q;
            const int am = e / kGK, ak = e % kGK;
            const int gm = m0 + am, gk = k0 + ak;
            ra[q] = (gm < M && gk < K) ? __ldg(A + (int64_t)gm * K + gk) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + 256 * q;
            if (BT) {   // B stored [N][K]: k fastest
                const int bn = e / kGK, bk = e % kGK;
                const int gn = n0 + bn, gk = k0 + bk;
                rb[q] = (gn < N && gk < K) ? __ldg(B + (int64_t)gn * K + gk) : 0.0;
            } else {    // B stored [K][N]: n fastest
                const int bk = e / kGN, bn = e % kGN;
                const int gn = n0 + bn, gk = k0 + bk;
                rb[q] = (gn < N && gk < K) ? __ldg(B + (int64_t)gk * N + gn) : 0.0;
            }
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = tid + 256 * q;
            As[buf][e % kGK][e / kGK] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + 256 * q;
            if (BT) Bs[buf][e % kGK][e / kGK] = rb[q];
            else Bs[buf][e / kGN][e % kGN] = rb[q];
        }
    };
    load(0);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += kGK) {
        const bool more = k0 + kGK < K;
        if (more) load(k0 + kGK);
#pragma unroll
        for (int k = 0; k < kGK; ++k) {
            double a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                const double2 t = *reinterpret_cast<const double2*>(&As[buf][k][tm + i]);
                a[i] = t.x;
                a[i + 1] = t.y;
            }
#pragma unroll
            for (int j = 0; j < 4; j += 2) {
                const double2 t = *reinterpret_cast<const double2*>(&Bs[buf][k][tn + j]);
                b[j] = t.x;
                b[j + 1] = t.y;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        if (more) {
            stash(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int gm = m0 + tm + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tn + j;
            if (gn < N) C[(int64_t)gm * N + gn] = acc[i][j];
        }
    }
}

static cudaError_t dgemm(bool bt, const double* A, const double* B, double* C, int M, int N, int K, int batch,
                         int64_t sa, int64_t sb, int64_t sc, cudaStream_t st) {
    const dim3 grid((unsigned)((N + kGN - 1) / kGN), (unsigned)((M + kGM - 1) / kGM), (unsigned)batch);
    const int smem = (int)(sizeof(double) * 2 * kGK * ((kGM + 2) + (kGN + 2)));
    if (bt) {
        cudaFuncSetAttribute(dgemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        dgemm_kernel<true><<<grid, 256, smem, st>>>(A, B, C, M, N, K, sa, sb, sc);
    } else {
        cudaFuncSetAttribute(dgemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        dgemm_kernel<false><<<grid, 256, smem, st>>>(A, B, C, M, N, K, sa, sb, sc);
    }
    return cudaGetLastError();
}

// the three axis passes (row-major):
//   w: T1[nw][mv*mu]  = M_w[nw][mw] . Q64[mw][mv*mu]
//   v: T2[k][nv][mu]  = M_v[nv][mv] . T1[k][mv][mu]      (batch over k < nw)
//   u: C64[nw*nv][nu] = T2[nw*nv][mu] . M_u^T             (M_u stored [nu][mu])
static mfa_status fit_all(const double* Q64, const AxisFitDev (&ax)[3], double* T1, double* T2, float* C32,
                          double* C64, cudaStream_t st) {
    const int mu = ax[0].m, mv = ax[1].m, mw = ax[2].m, nu = ax[0].n, nv = ax[1].n, nw = ax[2].n;
    cudaError_t e = dgemm(false, ax[2].M, Q64, T1, nw, mv * mu, mw, 1, 0, 0, 0, st);
    if (e == cudaSuccess)
        e = dgemm(false, ax[1].M, T1, T2, nv, mu, mv, nw, 0, (int64_t)mv * mu, (int64_t)nv * mu, st);
    if (e == cudaSuccess) e = dgemm(true, T2, ax[0].M, C64, nw * nv, nu, mu, 1, 0, 0, 0, st);
    if (e != cudaSuccess) return cuda_fail(e, "fit GEMM");
    const int64_t nc = (int64_t)nu * nv * nw;
    f64_to_f32_kernel<<<grid_for(nc), 128, 0, st>>>(C64, C32, nc);
    e = cudaGetLastError();
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "fit conversion");
}

template <int P>
static cudaError_t expand_all_t(const double* C64, const AxisFitDev (&ax)[3], double* T1, double* T2, double* V,
                                cudaStream_t st) {
    const int mu = ax[0].m, mv = ax[1].m, mw = ax[2].m, nv = ax[1].n, nw = ax[2].n;
    expand_axis_kernel<P><<<grid_for((int64_t)nw * nv * mu), 128, 0, st>>>(C64, T1, ax[0], (int64_t)nw * nv, 1);
    expand_axis_kernel<P><<<grid_for((int64_t)nw * mv * mu), 128, 0, st>>>(T1, T2, ax[1], nw, mu);
    expand_axis_kernel<P><<<grid_for((int64_t)mw * mv * mu), 128, 0, st>>>(T2, V, ax[2], 1, (int64_t)mv * mu);
    return cudaGetLastError();
}

static cudaError_t expand_all(int p, const double* C64, const AxisFitDev (&ax)[3], double* T1, double* T2, double* V,
                              cudaStream_t st) {
    switch (p) {
        case 1: return expand_all_t<1>(C64, ax, T1, T2, V, st);
        case 2: return expand_all_t<2>(C64, ax, T1, T2, V, st);
        case 3: return expand_all_t<3>(C64, ax, T1, T2, V, st);
        case 4: return expand_all_t<4>(C64, ax, T1, T2, V, st);
        default: return expand_all_t<5>(C64, ax, T1, T2, V, st);
    }
}

// scratch sized for the largest control counts the loop may reach
struct FitScratch {
    double *Q64 = nullptr, *T1 = nullptr, *T2 = nullptr, *C64 = nullptr, *V = nullptr;
    unsigned long long* err = nullptr;   // [nu + nv + nw spans] + max, then esq, range
    void release(cudaStream_t st) {
        for (void* p : {(void*)Q64, (void*)T1, (void*)T2, (void*)C64, (void*)V, (void*)err})
            if (p) cudaFreeAsync(p, st);
        Q64 = T1 = T2 = C64 = V = nullptr;
        err = nullptr;
    }
};

static mfa_status check_grid(const int64_t dims[3], const float* values, int p, const int64_t nctrl[3]) {
    if (!dims || !values || !nctrl) return fail(MFA_ERR_INVALID_ARG, "NULL argument");
    if (p < 1 || p > MFA_MAX_DEGREE) return fail(MFA_ERR_UNSUPPORTED, "degree outside 1..5");
    for (int d = 0; d < 3; ++d) {
        if (dims[d] < 2 || dims[d] > (1 << 20)) return fail(MFA_ERR_INVALID_ARG, "dims[d] must be in [2, 2^20]");
        if (nctrl[d] < p + 1) return fail(MFA_ERR_INVALID_ARG, "nctrl[d] < degree + 1");
        if (nctrl[d] > dims[d]) return fail(MFA_ERR_INVALID_ARG, "nctrl[d] > dims[d]: the fit would be singular");
    }
    return MFA_OK;
}

}  // namespace mfa

using namespace mfa;

extern "C" mfa_status mfa_fit_grid(const int64_t dims[3], const float* values, int32_t degree, const int64_t nctrl[3],
                                   const double* const knots[3], float* ctrl_out, double* ctrl_out64,
                                   mfa_stream stream) {
    mfa_status s = check_grid(dims, values, degree, nctrl);
    if (s != MFA_OK) return s;
    if (!knots || !ctrl_out) return fail(MFA_ERR_INVALID_ARG, "knots and ctrl_out are required");
    const int p = degree;
    for (int d = 0; d < 3; ++d) {
        int uni = 0;
        if (!knots[d]) return fail(MFA_ERR_INVALID_ARG, "knots[d] is NULL");
        if ((s = validate_knots(d, p, nctrl[d], knots[d], &uni)) != MFA_OK) return s;
    }
    cudaStream_t st = (cudaStream_t)stream;
    keep_pool();
    AxisDevMem D[3];
    FitScratch W;
    auto done = [&](mfa_status r) {
        cudaStreamSynchronize(st);
        for (auto& x : D) x.release(st);
        W.release(st);
        return r;
    };
    cudaError_t e;
    {   // non-finite samples would turn every control value NaN: refuse up front
        double* rng_dev = nullptr;
        if ((e = cudaMallocAsync(&rng_dev, 3 * sizeof(double), st)) != cudaSuccess) return done(cuda_fail(e, "fit scratch"));
        unsigned long long rb[3] = {~0ULL, 0ULL, 0ULL};
        cudaMemcpyAsync(rng_dev, rb, sizeof(rb), cudaMemcpyHostToDevice, st);
        range_kernel<<<grid_for(dims[0] * dims[1] * dims[2]), 128, 0, st>>>(values, dims[0] * dims[1] * dims[2], rng_dev);
        cudaMemcpyAsync(rb, rng_dev, sizeof(rb), cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(rng_dev, st);
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return done(cuda_fail(e, "fit range"));
        if (rb[2]) return done(fail(MFA_ERR_DOMAIN, std::to_string(rb[2]) + " non-finite grid values"));
    }
    {
        const int mm[3] = {(int)dims[0], (int)dims[1], (int)dims[2]}, nn[3] = {(int)nctrl[0], (int)nctrl[1], (int)nctrl[2]};
        if ((s = build_axes_dev(mm, nn, p, knots, D, st)) != MFA_OK) return done(s);
    }
    const int64_t mu = dims[0], mv = dims[1], mw = dims[2], nu = nctrl[0], nv = nctrl[1], nw = nctrl[2];
    if ((e = cudaMallocAsync(&W.Q64, sizeof(double) * mw * mv * mu, st)) != cudaSuccess) return done(cuda_fail(e, "fit scratch"));
    f32_to_f64_kernel<<<grid_for(mw * mv * mu), 128, 0, st>>>(values, W.Q64, mw * mv * mu);
    if ((e = cudaMallocAsync(&W.T1, sizeof(double) * nw * mv * mu, st)) != cudaSuccess) return done(cuda_fail(e, "fit scratch"));
    if ((e = cudaMallocAsync(&W.T2, sizeof(double) * nw * nv * mu, st)) != cudaSuccess) return done(cuda_fail(e, "fit scratch"));
    double* c64 = ctrl_out64;
    if (!c64) {
        if ((e = cudaMallocAsync(&W.C64, sizeof(double) * nw * nv * nu, st)) != cudaSuccess) return done(cuda_fail(e, "fit scratch"));
        c64 = W.C64;
    }
    const AxisFitDev ax[3] = {D[0].d, D[1].d, D[2].d};
    return done(fit_all(W.Q64, ax, W.T1, W.T2, ctrl_out, c64, st));
}

extern "C" mfa_status mfa_encode_grid(const int64_t dims[3], const float* values, const mfa_encode_config* cfg,
                                      double* const knots_out[3], float* ctrl_out, mfa_encode_result* res,
                                      double* round_log, mfa_stream stream) {
    if (!cfg || !knots_out || !ctrl_out || !res) return fail(MFA_ERR_INVALID_ARG, "NULL argument");
    const int p = cfg->degree;
    mfa_status s = check_grid(dims, values, p, cfg->nctrl_init);
    if (s != MFA_OK) return s;
    for (int d = 0; d < 3; ++d) {
        if (!knots_out[d]) return fail(MFA_ERR_INVALID_ARG, "knots_out[d] is NULL");
        if (cfg->max_ctrl[d] < cfg->nctrl_init[d]) return fail(MFA_ERR_INVALID_ARG, "max_ctrl[d] < nctrl_init[d]");
    }
    if (!(cfg->e_max >= 0.0) || cfg->max_rounds < 0) return fail(MFA_ERR_INVALID_ARG, "e_max >= 0, max_rounds >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t mu = dims[0], mv = dims[1], mw = dims[2], npts = mu * mv * mw;
    int64_t cap[3];
    for (int d = 0; d < 3; ++d) cap[d] = std::min<int64_t>(cfg->max_ctrl[d], dims[d]);
    // initial knots: clamped uniform with nctrl_init control points (R-28)
    std::vector<double> U[3];
    for (int d = 0; d < 3; ++d) {
        const int64_t n = cfg->nctrl_init[d], S = n - p;
        U[d].assign(p + 1, 0.0);
        for (int64_t k = 1; k < S; ++k) U[d].push_back((double)k / (double)S);
        U[d].insert(U[d].end(), p + 1, 1.0);
    }
    keep_pool();
    FitScratch W;
    AxisDevMem D[3];
    double* rng_dev = nullptr;
    auto done = [&](mfa_status r) {
        cudaStreamSynchronize(st);
        for (auto& x : D) x.release(st);
        W.release(st);
        if (rng_dev) cudaFreeAsync(rng_dev, st);
        return r;
    };
    cudaError_t e;
    const int64_t maxT1 = cap[2] * mv * mu, maxT2 = std::max(cap[2] * cap[1] * mu, cap[2] * mv * mu);
    if ((e = cudaMallocAsync(&W.T1, sizeof(double) * std::max(maxT1, cap[2] * cap[1] * mu), st)) != cudaSuccess)
        return done(cuda_fail(e, "encode scratch"));
    if ((e = cudaMallocAsync(&W.T2, sizeof(double) * std::max(maxT2, mw * mv * mu), st)) != cudaSuccess)
        return done(cuda_fail(e, "encode scratch"));
    if ((e = cudaMallocAsync(&W.C64, sizeof(double) * cap[0] * cap[1] * cap[2], st)) != cudaSuccess)
        return done(cuda_fail(e, "encode scratch"));
    if ((e = cudaMallocAsync(&W.V, sizeof(double) * npts, st)) != cudaSuccess) return done(cuda_fail(e, "encode scratch"));
    if ((e = cudaMallocAsync(&W.Q64, sizeof(double) * npts, st)) != cudaSuccess) return done(cuda_fail(e, "encode scratch"));
    f32_to_f64_kernel<<<grid_for(npts), 128, 0, st>>>(values, W.Q64, npts);
    const int64_t nerr = cap[0] + cap[1] + cap[2] + 2;
    if ((e = cudaMallocAsync(&W.err, sizeof(unsigned long long) * nerr, st)) != cudaSuccess)
        return done(cuda_fail(e, "encode scratch"));
    if ((e = cudaMallocAsync(&rng_dev, 3 * sizeof(double), st)) != cudaSuccess) return done(cuda_fail(e, "encode scratch"));
    unsigned long long rinit[3] = {~0ULL, 0ULL, 0ULL};
    cudaMemcpyAsync(rng_dev, rinit, sizeof(rinit), cudaMemcpyHostToDevice, st);
    range_kernel<<<grid_for(npts), 128, 0, st>>>(values, npts, rng_dev);
    unsigned long long rb[3];
    cudaMemcpyAsync(rb, rng_dev, sizeof(rb), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return done(cuda_fail(e, "encode range"));
    if (rb[2]) return done(fail(MFA_ERR_DOMAIN, std::to_string(rb[2]) + " non-finite grid values"));
    const double range = ord_to_double(rb[1]) - ord_to_double(rb[0]);
    const double inv_range = range > 0.0 ? 1.0 / range : 1.0;

    int rounds = 0;
    bool converged = false;
    double max_err = 0.0, rms = 0.0;
    for (;;) {
        int64_t n[3];
        for (int d = 0; d < 3; ++d) {
            n[d] = (int64_t)U[d].size() - p - 1;
            D[d].release(st);
        }
        {
            const int mm[3] = {(int)dims[0], (int)dims[1], (int)dims[2]}, nn[3] = {(int)n[0], (int)n[1], (int)n[2]};
            const double* const uu[3] = {U[0].data(), U[1].data(), U[2].data()};
            if ((s = build_axes_dev(mm, nn, p, uu, D, st)) != MFA_OK) return done(s);
        }
        const AxisFitDev ax[3] = {D[0].d, D[1].d, D[2].d};
        if ((s = fit_all(W.Q64, ax, W.T1, W.T2, ctrl_out, W.C64, st)) != MFA_OK) return done(s);
        if ((e = expand_all(p, W.C64, ax, W.T1, W.T2, W.V, st)) != cudaSuccess) return done(cuda_fail(e, "expand"));
        const int64_t S0 = n[0] - p, S1 = n[1] - p, S2 = n[2] - p;
        cudaMemsetAsync(W.err, 0, sizeof(unsigned long long) * nerr, st);
        unsigned long long *eu = W.err, *ev = eu + S0, *ew = ev + S1, *emax = ew + S2;
        double* esq = reinterpret_cast<double*>(emax + 1);
        const int nsp = (S0 + S1 + S2 <= 6144) ? (int)(S0 + S1 + S2) : 0;   // shared-memory span maxima
        grid_error_kernel<<<grid_for(npts), 128, sizeof(unsigned long long) * nsp, st>>>(
            W.V, values, (int)mu, (int)mv, (int)mw, inv_range, ax[0].f, ax[1].f, ax[2].f, eu, ev, ew, emax, esq,
            (int)S0, (int)S1, nsp);
        std::vector<unsigned long long> h(S0 + S1 + S2 + 2);
        cudaMemcpyAsync(h.data(), W.err, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return done(cuda_fail(e, "encode residual"));
        auto dv = [](unsigned long long b) {
            double x;
            memcpy(&x, &b, 8);
            return x;
        };
        max_err = dv(h[S0 + S1 + S2]);
        double sq;
        memcpy(&sq, &h[S0 + S1 + S2 + 1], 8);
        rms = sqrt(sq / (double)npts);
        if (round_log) {
            double* r = round_log + 5 * rounds;
            r[0] = (double)n[0];
            r[1] = (double)n[1];
            r[2] = (double)n[2];
            r[3] = max_err;
            r[4] = rms;
        }
        ++rounds;
        for (int d = 0; d < 3; ++d) res->nctrl[d] = n[d];
        if (max_err <= cfg->e_max) {
            converged = true;
            break;
        }
        if (rounds > cfg->max_rounds) break;
        // split every offending span holding >= 2 samples at its midpoint, within the caps
        bool split_any = false;
        const unsigned long long* hs[3] = {h.data(), h.data() + S0, h.data() + S0 + S1};
        for (int d = 0; d < 3; ++d) {
            const int64_t Sd = n[d] - p;
            std::vector<int> cnt(Sd, 0);
            for (int fj : sample_spans(U[d].data(), p, (int)n[d], (int)dims[d])) cnt[fj]++;
            std::vector<double> ins;
            for (int64_t sp = 0; sp < Sd; ++sp)
                if (dv(hs[d][sp]) > cfg->e_max && cnt[sp] >= 2 * (p + 1) && n[d] + (int64_t)ins.size() < cap[d])
                    ins.push_back(0.5 * (U[d][p + sp] + U[d][p + sp + 1]));
            if (!ins.empty()) {
                split_any = true;
                U[d].insert(U[d].end(), ins.begin(), ins.end());
                std::sort(U[d].begin(), U[d].end());
            }
        }
        if (!split_any) break;
    }
    for (int d = 0; d < 3; ++d) std::copy(U[d].begin(), U[d].end(), knots_out[d]);
    res->rounds = rounds;
    res->converged = converged ? 1 : 0;
    res->max_err = max_err;
    res->rms_err = rms;
    return done(MFA_OK);
}
