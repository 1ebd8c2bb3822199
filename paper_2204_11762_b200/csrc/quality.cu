// Image-quality metrics: MSE, PSNR and SSIM of a
// rendering against the ground-truth rendering "at the pixel level"
// (Tables 1-2).  Readings (R-22, after
// SPEC S:469-516): displayed colour = premultiplied RGB over black, 8-bit
// levels q = floor(255 clamp(x) + 1/2); MSE over pixels x 3 channels; PSNR =
// 10 log10(255^2 / MSE); SSIM on luma 0.299 R + 0.587 G + 0.114 B, 11x11
// Gaussian window (sigma 1.5), C1 = (0.01*255)^2, C2 = (0.03*255)^2, mean over
// the valid window positions.
//
// All arithmetic in fp64 (the quantisation is exact: 255 x of an fp32 x is
// exact in fp64), reductions in a fixed order (deterministic):
//   K_q  per pixel: levels, luma images, squared-difference partial sums, error map
//   K_s  per valid window: 5 windowed moments from a shared-memory tile, SSIM partials
//   K_r  one CTA: fixed-order tree of the partials -> (MSE, PSNR, mean SSIM)
#include <math.h>

#include <algorithm>

#include "mfa_internal.cuh"

namespace mfa {

#ifndef MFA_SSIM_SEP   // 1: separable SSIM window passes
#define MFA_SSIM_SEP 1
#endif
constexpr int kWin = 11;
constexpr int kQThreads = 256;
constexpr int kSTileX = 32, kSTileY = 8;   // SSIM outputs per CTA

struct GaussWin {
    double w[kWin * kWin];
};

static GaussWin make_window() {
    GaussWin g;
    double sum = 0.0;
    for (int i = 0; i < kWin; ++i)
        for (int j = 0; j < kWin; ++j) {
            const double di = i - kWin / 2, dj = j - kWin / 2;
            g.w[i * kWin + j] = exp(-(di * di + dj * dj) / (2.0 * 1.5 * 1.5));
            sum += g.w[i * kWin + j];
        }
    for (int k = 0; k < kWin * kWin; ++k) g.w[k] /= sum;
    return g;
}

__device__ __forceinline__ double level8(float x) {
    return floor(255.0 * (double)fminf(fmaxf(x, 0.f), 1.f) + 0.5);
}

template <int N>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < N / 32; ++k) r += sh[k];
    return r;
}

__global__ void __launch_bounds__(kQThreads) quality_pixels_kernel(const float4* __restrict__ a,
                                                                   const float4* __restrict__ b, int64_t n,
                                                                   double* __restrict__ ya, double* __restrict__ yb,
                                                                   float* __restrict__ err, double* __restrict__ part) {
    __shared__ double sh[kQThreads / 32];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kQThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kQThreads) {
        const float4 pa = a[i], pb = b[i];
        const double ar = level8(pa.x), ag = level8(pa.y), ab = level8(pa.z);
        const double br = level8(pb.x), bg = level8(pb.y), bb = level8(pb.z);
        ya[i] = 0.299 * ar + 0.587 * ag + 0.114 * ab;
        yb[i] = 0.299 * br + 0.587 * bg + 0.114 * bb;
        const double s = (ar - br) * (ar - br) + (ag - bg) * (ag - bg) + (ab - bb) * (ab - bb);  // exact integers
        if (err) err[i] = (float)sqrt(s);
        acc += s;
    }
    const double t = block_sum<kQThreads>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kSTileX* kSTileY) ssim_kernel(const double* __restrict__ ya,
                                                                const double* __restrict__ yb, int W, int H,
                                                                const GaussWin gw, double* __restrict__ part) {
    constexpr int TW = kSTileX + kWin - 1, TH = kSTileY + kWin - 1;
    __shared__ double sa[TH][TW], sb[TH][TW];
    __shared__ double sh[kSTileX * kSTileY / 32];
    const int ow = W - kWin + 1, oh = H - kWin + 1;
    const int x0 = blockIdx.x * kSTileX, y0 = blockIdx.y * kSTileY;
    for (int k = threadIdx.x; k < TW * TH; k += blockDim.x) {
        const int ty = k / TW, tx = k % TW;
        const int gx = min(x0 + tx, W - 1), gy = min(y0 + ty, H - 1);
        sa[ty][tx] = ya[(int64_t)gy * W + gx];
        sb[ty][tx] = yb[(int64_t)gy * W + gx];
    }
    __syncthreads();
    const int lx = threadIdx.x % kSTileX, ly = threadIdx.x / kSTileX;
    const int ox = x0 + lx, oy = y0 + ly;
    double v = 0.0;
    if (ox < ow && oy < oh) {
        double ma = 0.0, mb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
        for (int di = 0; di < kWin; ++di)
#pragma unroll
            for (int dj = 0; dj < kWin; ++dj) {
                const double w = gw.w[di * kWin + dj];
                const double A = sa[ly + di][lx + dj], B = sb[ly + di][lx + dj];
                ma += w * A;
                mb += w * B;
                saa += w * A * A;
                sbb += w * B * B;
                sab += w * A * B;
            }
        const double va = saa - ma * ma, vb = sbb - mb * mb, cab = sab - ma * mb;
        const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
        v = ((2.0 * ma * mb + C1) * (2.0 * cab + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2));
    }
    const double t = block_sum<kSTileX * kSTileY>(v, sh);
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// K_s, separable form (MFA_SSIM_SEP): the 11x11 Gaussian window is the outer
// product of the normalised 1-D window g (w_ij = g_i g_j exactly, up to fp64
// rounding), so the 5 moments are an 11-tap row pass into shared memory and
// an 11-tap column pass: 55 + 55 * 18/8 weighted terms per output instead of 605
struct GaussWin1 {
    double g[kWin];
};

static GaussWin1 make_window1() {
    GaussWin1 g;
    double sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
        const double di = i - kWin / 2;
        g.g[i] = exp(-(di * di) / (2.0 * 1.5 * 1.5));
        sum += g.g[i];
    }
    for (int i = 0; i < kWin; ++i) g.g[i] /= sum;
    return g;
}

__global__ void __launch_bounds__(kSTileX* kSTileY) ssim_sep_kernel(const double* __restrict__ ya,
                                                                    const double* __restrict__ yb, int W, int H,
                                                                    const GaussWin1 gw, double* __restrict__ part) {
    constexpr int TW = kSTileX + kWin - 1, TH = kSTileY + kWin - 1;
    __shared__ double sa[TH][TW], sb[TH][TW];
    __shared__ double hm[5][TH][kSTileX];
    __shared__ double sh[kSTileX * kSTileY / 32];
    const int ow = W - kWin + 1, oh = H - kWin + 1;
    const int x0 = blockIdx.x * kSTileX, y0 = blockIdx.y * kSTileY;
    for (int k = threadIdx.x; k < TW * TH; k += blockDim.x) {
        const int ty = k / TW, tx = k % TW;
        const int gx = min(x0 + tx, W - 1), gy = min(y0 + ty, H - 1);
        sa[ty][tx] = ya[(int64_t)gy * W + gx];
        sb[ty][tx] = yb[(int64_t)gy * W + gx];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < TH * kSTileX; k += blockDim.x) {   // row pass
        const int r = k / kSTileX, c = k % kSTileX;
        double ma = 0.0, mb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
#pragma unroll
        for (int dj = 0; dj < kWin; ++dj) {
            const double w = gw.g[dj];
            const double A = sa[r][c + dj], B = sb[r][c + dj];
            ma += w * A;
            mb += w * B;
            saa += w * A * A;
            sbb += w * B * B;
            sab += w * A * B;
        }
        hm[0][r][c] = ma;
        hm[1][r][c] = mb;
        hm[2][r][c] = saa;
        hm[3][r][c] = sbb;
        hm[4][r][c] = sab;
    }
    __syncthreads();
    const int lx = threadIdx.x % kSTileX, ly = threadIdx.x / kSTileX;
    const int ox = x0 + lx, oy = y0 + ly;
    double v = 0.0;
    if (ox < ow && oy < oh) {   // column pass
        double ma = 0.0, mb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
#pragma unroll
        for (int di = 0; di < kWin; ++di) {
            const double w = gw.g[di];
            ma += w * hm[0][ly + di][lx];
            mb += w * hm[1][ly + di][lx];
            saa += w * hm[2][ly + di][lx];
            sbb += w * hm[3][ly + di][lx];
            sab += w * hm[4][ly + di][lx];
        }
        const double va = saa - ma * ma, vb = sbb - mb * mb, cab = sab - ma * mb;
        const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
        v = ((2.0 * ma * mb + C1) * (2.0 * cab + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2));
    }
    const double t = block_sum<kSTileX * kSTileY>(v, sh);
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// one CTA of 1024 threads: strided partial sums, then a fixed-order tree
__global__ void __launch_bounds__(1024) quality_final_kernel(const double* __restrict__ pq, int nq,
                                                             const double* __restrict__ ps, int ns, int64_t npix,
                                                             int64_t nwin, double* __restrict__ out) {
    __shared__ double sq[1024], st[1024];
    double a = 0.0, b = 0.0;
    for (int k = threadIdx.x; k < nq; k += 1024) a += pq[k];
    for (int k = threadIdx.x; k < ns; k += 1024) b += ps[k];
    sq[threadIdx.x] = a;
    st[threadIdx.x] = b;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sq[threadIdx.x] += sq[threadIdx.x + o];
            st[threadIdx.x] += st[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const double s = sq[0], t = st[0];
    const double mse = s / (3.0 * (double)npix);
    out[0] = mse;
    out[1] = mse == 0.0 ? INFINITY : 10.0 * log10(255.0 * 255.0 / mse);
    out[2] = t / (double)nwin;
}

struct QualityPlan {
    int nq, sx, sy;
    size_t bytes, off_yb, off_pq, off_ps;
};

static QualityPlan plan_quality(int W, int H) {
    QualityPlan p;
    const int64_t n = (int64_t)W * H;
    p.nq = (int)std::min<int64_t>((n + kQThreads - 1) / kQThreads, 4 * 148);
    p.sx = (W - kWin + 1 + kSTileX - 1) / kSTileX;
    p.sy = (H - kWin + 1 + kSTileY - 1) / kSTileY;
    p.off_yb = sizeof(double) * n;
    p.off_pq = 2 * sizeof(double) * n;
    p.off_ps = p.off_pq + sizeof(double) * p.nq;
    p.bytes = p.off_ps + sizeof(double) * (size_t)p.sx * p.sy;
    return p;
}

}  // namespace mfa

using namespace mfa;

extern "C" size_t mfa_image_quality_workspace(int32_t width, int32_t height) {
    if (width < kWin || height < kWin) return 0;
    return plan_quality(width, height).bytes;
}

extern "C" mfa_status mfa_image_quality(int32_t width, int32_t height, const float* img_a, const float* img_b,
                                        float* err_map, void* workspace, size_t workspace_bytes, double* out3,
                                        mfa_stream stream) {
    if (!img_a || !img_b || !out3 || !workspace) return fail(MFA_ERR_INVALID_ARG, "NULL argument");
    if (width < kWin || height < kWin)
        return fail(MFA_ERR_INVALID_ARG, "image smaller than the 11x11 SSIM window");
    if ((int64_t)width * height > (int64_t)1 << 31) return fail(MFA_ERR_UNSUPPORTED, "image larger than 2^31 pixels");
    const QualityPlan p = plan_quality(width, height);
    if (workspace_bytes < p.bytes) return fail(MFA_ERR_INVALID_ARG, "workspace smaller than mfa_image_quality_workspace()");
    cudaStream_t st = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    double* ya = (double*)ws;
    double* yb = (double*)(ws + p.off_yb);
    double* pq = (double*)(ws + p.off_pq);
    double* ps = (double*)(ws + p.off_ps);
    const int64_t n = (int64_t)width * height;
    quality_pixels_kernel<<<p.nq, kQThreads, 0, st>>>(reinterpret_cast<const float4*>(img_a),
                                                      reinterpret_cast<const float4*>(img_b), n, ya, yb, err_map, pq);
#if MFA_SSIM_SEP
    static const GaussWin1 gw1 = make_window1();
    ssim_sep_kernel<<<dim3(p.sx, p.sy), kSTileX * kSTileY, 0, st>>>(ya, yb, width, height, gw1, ps);
#else
    static const GaussWin gw = make_window();
    ssim_kernel<<<dim3(p.sx, p.sy), kSTileX * kSTileY, 0, st>>>(ya, yb, width, height, gw, ps);
#endif
    const int64_t nwin = (int64_t)(width - kWin + 1) * (height - kWin + 1);
    quality_final_kernel<<<1, 1024, 0, st>>>(pq, p.nq, ps, p.sx * p.sy, n, nwin, out3);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "image quality kernels");
}
