// mfa_eval_batch kernel: per point a4 span -> a5 basis +
// derivatives -> a6 gather -> a7 contraction; value and parameter-space
// gradient (Algorithm 1 lines 6 and 9; "all derivatives
// along the three dimensions at once").  One point per thread, grid-stride,
// grid = a multiple of the SM count.
#include "kernels.cuh"

namespace mfa {

struct EvalArgs {
    const float4* Q;
    BrickGrid g;
    BezGrid bg;
    AxisArgs ax[3];
    const float* u;
    const float* v;
    const float* w;
    float* value;
    float* du;
    float* dv;
    float* dw;
    unsigned long long* n_err;
    int64_t n;
    const float4* rec;     // SORTED: points as (u, v, w, index bits), grouped by spatial bin
    float4* out4;          // SORTED: (value, du, dv, dw) at the sorted position (in place over rec)
    const int* pos;        // SORTED: sorted position of point i
    // binned Bezier eval (eval_cells_kernel): bin b holds records [end_b - cnt_b, end_b)
    const unsigned* bin_cnt;   // per bin (nbins + 1, the last for points outside [0,1]^3); NULL: grid-stride kernel
    const unsigned* bin_end;   // end of bin b at bin_end[b * bin_stride]
    int bin_stride;
    int nb[3];
    int nbins;
};

#ifndef MFA_EVAL_MINB     // resident 256-thread CTAs per SM the register budget is sized for
#define MFA_EVAL_MINB 1
#endif

// one point: value and parameter-space gradient (NaN and false outside [0,1]^3)
template <int P, int LAYOUT, bool UNI, bool GRAD>
__device__ __forceinline__ bool eval_point(const EvalArgs& args, const float (&q)[3], float& val, float& gu, float& gv,
                                           float& gw) {
    constexpr bool BEZ = is_bez(LAYOUT);
    constexpr int SEC = bez_sec(LAYOUT == kBezierG);
    gu = gv = gw = 0.f;
    if (!(q[0] >= 0.f && q[0] <= 1.f && q[1] >= 0.f && q[1] <= 1.f && q[2] >= 0.f && q[2] <= 1.f)) {
        val = gu = gv = gw = __int_as_float(0x7fc00000);
        return false;
    }
    int s[3];
    float t[3], sc[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        if (UNI) {
            uni_span_f32(q[d], args.ax[d].S, args.ax[d].nsp, s[d], t[d]);
            sc[d] = args.ax[d].S;
        } else {
            nonuni_span_f32(args.ax[d], q[d], s[d], t[d], sc[d]);
        }
    }
    if constexpr (BEZ) {
        const float4* base = bez_block<P, SEC>(args.Q, args.bg, s[0], s[1], s[2]);
        if (GRAD) {
            float r0[P + 1][P + 1];
            load_bslab<P, SEC>(base, r0);
            float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
            bernstein<P, false>(t[0], Bu);
            bernstein<P, true>(t[1], Bv);
            bernstein<P, false>(t[2], Bw);
            contract_vg_bez<P, SEC>(base, r0, Bu, Bv, Bw, val, gu, gv, gw);
        } else {
            float nb[P + 1][P + 1][P + 1];
            load_bblock<P, SEC>(base, nb);
            float Nu[P + 1], Nv[P + 1], Nw[P + 1];
            bernstein_value<P>(t[0], Nu);
            bernstein_value<P>(t[1], Nv);
            bernstein_value<P>(t[2], Nw);
            val = contract_v_cached<P>(nb, Nu, Nv, Nw);
        }
    } else if constexpr (LAYOUT == kBricks) {   // plain haloed bricks: the block into registers
        float nb[P + 1][P + 1][P + 1];
        load_pblock<P>(args.Q, plain_entry<P>(args.g, s[0], s[1], s[2]), nb);
        if (GRAD) {
            float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
            axis_basis<P, false>(args.ax[0], UNI, s[0], t[0], Bu);
            axis_basis<P, true>(args.ax[1], UNI, s[1], t[1], Bv);
            axis_basis<P, false>(args.ax[2], UNI, s[2], t[2], Bw);
            contract_vg_cached<P>(nb, Bu, Bv, Bw, val, gu, gv, gw);
        } else {
            float Nu[P + 1], Nv[P + 1], Nw[P + 1];
            axis_basis_value<P>(args.ax[0], UNI, s[0], t[0], Nu);
            axis_basis_value<P>(args.ax[1], UNI, s[1], t[1], Nv);
            axis_basis_value<P>(args.ax[2], UNI, s[2], t[2], Nw);
            val = contract_v_cached<P>(nb, Nu, Nv, Nw);
        }
    } else {
        const float4* base = args.Q + brick_entry<P>(args.g, s[0], s[1], s[2]);
        float r0[P + 1][P + 1];
        load_slab<P>(base, r0);   // issued before the basis so its latency overlaps it
        if (GRAD) {
            float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
            axis_basis<P, false>(args.ax[0], UNI, s[0], t[0], Bu);
            axis_basis<P, true>(args.ax[1], UNI, s[1], t[1], Bv);
            axis_basis<P, false>(args.ax[2], UNI, s[2], t[2], Bw);
            contract_vg<P>(base, r0, Bu, Bv, Bw, val, gu, gv, gw);
        } else {
            float Nu[P + 1], Nv[P + 1], Nw[P + 1];
            axis_basis_value<P>(args.ax[0], UNI, s[0], t[0], Nu);
            axis_basis_value<P>(args.ax[1], UNI, s[1], t[1], Nv);
            axis_basis_value<P>(args.ax[2], UNI, s[2], t[2], Nw);
            val = contract_v<P>(base, r0, Nu, Nv, Nw);
        }
    }
    if (GRAD) {
        gu *= sc[0];
        gv *= sc[1];
        gw *= sc[2];
    }
    return true;
}

template <int P, int LAYOUT, bool UNI, bool GRAD, bool SORTED>
__global__ void __launch_bounds__(256, MFA_EVAL_MINB) eval_kernel(const __grid_constant__ EvalArgs args) {
    unsigned errs = 0;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < args.n;
         it += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = it;
        float q[3];
        if constexpr (SORTED) {   // consecutive threads hold spatially close points
            const float4 r = __ldg(args.rec + it);
            q[0] = r.x;
            q[1] = r.y;
            q[2] = r.z;
            i = (int64_t)(unsigned)__float_as_int(r.w);
        } else {
            q[0] = __ldg(args.u + i);
            q[1] = __ldg(args.v + i);
            q[2] = __ldg(args.w + i);
        }
        float val, gu, gv, gw;
        if (!eval_point<P, LAYOUT, UNI, GRAD>(args, q, val, gu, gv, gw)) ++errs;
        if constexpr (SORTED) {   // one coalesced float4 at the sorted position
            args.out4[it] = make_float4(val, gu, gv, gw);
        } else {                  // SoA outputs at i
            args.value[i] = val;
            if (GRAD) {
                args.du[i] = gu;
                args.dv[i] = gv;
                args.dw[i] = gw;
            }
        }
    }
    if (args.n_err) {
        for (int o = 16; o > 0; o >>= 1) errs += __shfl_xor_sync(0xffffffffu, errs, o);
        if ((threadIdx.x & 31) == 0 && errs) atomicAdd(args.n_err, (unsigned long long)errs);
    }
}

// Binned points on the Bezier layout, one CTA per bin: the bin's records are
// re-ordered in shared memory by a counting sort on a cell key (kCellSub^3
// cells per bin, u fastest), so the lanes of a warp hold points of
// neighbouring cells and points in one span triple share its 256-byte block
// within one load instruction.  Results go back to the record's own slot
// (out4 over rec), which the gather reads.  (On the quad layouts the same
// sort is slower: C3 12.8 vs 13.1, C4 6.1 vs 6.75 G points/s.)
#ifndef MFA_EVAL_CELLS      // 1: binned Bezier eval sorts each bin into cells in shared memory
#define MFA_EVAL_CELLS 1
#endif
#ifndef MFA_EVAL_CELLS_QUADS   // experiment: the cell sort on the quad layouts too (C3 13.8 vs 14.2 G points/s: off)
#define MFA_EVAL_CELLS_QUADS 0
#endif
constexpr int kCellSub = 8;                        // cells per bin edge
constexpr int kCells = kCellSub * kCellSub * kCellSub;
#ifndef MFA_CELL_THREADS
#define MFA_CELL_THREADS 128
#endif
constexpr int kCellCap = 1024;                     // points per shared-memory piece
constexpr int kCellThreads = MFA_CELL_THREADS;

// Quad layout (p = 3, 32-byte row-pair entries, 4 u-neighbours per 128-byte
// line): an LDG.256 is served by the L1 data pipe in groups of 4 lanes, one
// wavefront per distinct 128-byte line in a group (tools/ubench: 2 lanes per
// line 16 wavefronts per warp, 4 lanes per line 8).  So the cell key is the
// point's line group (span w, span v, span u / 4) and each key gets whole
// 4-lane slots: the 4 lanes of a slot read the same line on all 8 row-pair
// loads.  Idle lanes of a partly filled slot skip the evaluation.
// Measured (C3, 2^24 points; tools/gpu_ab_lines.sh): global L1 wavefronts
// 109 M -> 84 M against the plain cell sort, but 1.57x the instructions (idle
// slot lanes, the span key, a second scan) and 2x the shared-memory
// wavefronts: 12.6 vs 13.9 G points/s for the unsorted-bin kernel, so it is
// off (kept as a measured experiment).
#ifndef MFA_EVAL_LINES
#define MFA_EVAL_LINES 0
#endif
constexpr int kLaneCap = 4 * kCellCap;             // worst case: one point per slot

template <int P, int LAYOUT>
constexpr bool eval_lines() { return MFA_EVAL_LINES && LAYOUT == kQuads && P == 3; }

// exclusive scan of kCells counts in place (f applied to each count first);
// returns the total.  All threads of the CTA call it.
template <typename F>
__device__ __forceinline__ unsigned cells_scan(unsigned* a, unsigned* wsum, F f) {
    constexpr int E = kCells / kCellThreads;
    unsigned c[E], tsum = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        c[e] = f(a[threadIdx.x * E + e]);
        tsum += c[e];
    }
    unsigned x = tsum;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    unsigned run = x - tsum, total = 0;
    for (int w = 0; w < kCellThreads / 32; ++w) {
        if (w < wid) run += wsum[w];
        total += wsum[w];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        a[threadIdx.x * E + e] = run;
        run += c[e];
    }
    __syncthreads();
    return total;
}

template <int P, int LAYOUT, bool UNI, bool GRAD>
__global__ void __launch_bounds__(kCellThreads) eval_cells_kernel(const __grid_constant__ EvalArgs args) {
    constexpr bool LINES = eval_lines<P, LAYOUT>();
    __shared__ float4 s_rec[kCellCap];
    __shared__ unsigned short s_ord[kCellCap];
    __shared__ unsigned short s_key[kCellCap];
    __shared__ unsigned s_hist[kCells];
    __shared__ unsigned s_kstart[LINES ? kCells : 1];
    __shared__ unsigned s_slot[LINES ? kCells : 1];
    __shared__ unsigned short s_lane[LINES ? kLaneCap : 1];
    __shared__ unsigned s_wsum[kCellThreads / 32];
    const int b = blockIdx.x;
    const unsigned cnt = __ldg(args.bin_cnt + b);
    const unsigned end = __ldg(args.bin_end + (size_t)b * args.bin_stride);
    const unsigned start = end - cnt;
    int bc[3] = {0, 0, 0};
    if (b < args.nbins) {
        bc[0] = b % args.nb[0];
        bc[1] = (b / args.nb[0]) % args.nb[1];
        bc[2] = b / (args.nb[0] * args.nb[1]);
    }
    int s0[3] = {0, 0, 0};   // LINES: spans of the bin's lower corner
    if constexpr (LINES) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const float q0 = (float)bc[d] / (float)args.nb[d];
            float t, h;
            if (UNI) uni_span_f32(q0, args.ax[d].S, args.ax[d].nsp, s0[d], t);
            else nonuni_span_f32(args.ax[d], q0, s0[d], t, h);
        }
    }
    unsigned errs = 0;
    for (unsigned piece = 0; piece < cnt; piece += kCellCap) {
        const int m = (int)min((unsigned)kCellCap, cnt - piece);
        for (int c = threadIdx.x; c < kCells; c += kCellThreads) s_hist[c] = 0;
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += kCellThreads) {
            const float4 r = __ldg(args.rec + start + piece + j);
            s_rec[j] = r;
            int key = 0;
            if (b < args.nbins) {   // the point's cell in its bin (points outside [0,1]^3 sit in bin nbins)
                const float q[3] = {r.x, r.y, r.z};
                int c[3];
                if constexpr (LINES) {   // line group: (span w, span v, span u / 4) relative to the bin corner
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        int sd;
                        float t, h;
                        if (UNI) uni_span_f32(q[d], args.ax[d].S, args.ax[d].nsp, sd, t);
                        else nonuni_span_f32(args.ax[d], q[d], sd, t, h);
                        c[d] = d == 0 ? (sd >> 2) - (s0[0] >> 2) : sd - s0[d];
                        c[d] = min(max(c[d], 0), kCellSub - 1);
                    }
                } else {
#pragma unroll
                    for (int d = 0; d < 3; ++d)
                        c[d] = min(max((int)((q[d] * (float)args.nb[d] - (float)bc[d]) * (float)kCellSub), 0), kCellSub - 1);
                }
                if constexpr (LAYOUT == kBezierG) {
                    // cells of one block group (the layout's 4-block group) consecutive, so
                    // neighbouring lanes read the same 128-byte lines
                    const int hi = (((c[2] >> kGLw) * (kCellSub >> kGLv) + (c[1] >> kGLv)) * (kCellSub >> kGLu)) + (c[0] >> kGLu);
                    const int lo = ((c[2] & ((1 << kGLw) - 1)) << (kGLv + kGLu)) | ((c[1] & ((1 << kGLv) - 1)) << kGLu) |
                                   (c[0] & ((1 << kGLu) - 1));
                    key = (hi << 2) | lo;
                } else {   // u fastest
                    key = (c[2] * kCellSub + c[1]) * kCellSub + c[0];
                }
            }
            s_key[j] = (unsigned short)key;
            atomicAdd(s_hist + key, 1u);
        }
        __syncthreads();
        int lanes = m;
        if constexpr (LINES) {
            for (int c = threadIdx.x; c < kCells; c += kCellThreads) s_slot[c] = s_hist[c];
            __syncthreads();
            lanes = 4 * (int)cells_scan(s_slot, s_wsum, [](unsigned x) { return (x + 3u) >> 2; });
            for (int j = threadIdx.x; j < lanes; j += kCellThreads) s_lane[j] = 0xffff;
        }
        cells_scan(s_hist, s_wsum, [](unsigned x) { return x; });
        if constexpr (LINES) {
            for (int c = threadIdx.x; c < kCells; c += kCellThreads) s_kstart[c] = s_hist[c];
            __syncthreads();
        }
        for (int j = threadIdx.x; j < m; j += kCellThreads) {
            const int key = s_key[j];
            const unsigned pos = atomicAdd(s_hist + key, 1u);
            if constexpr (LINES) s_lane[4 * s_slot[key] + (pos - s_kstart[key])] = (unsigned short)j;
            else s_ord[pos] = (unsigned short)j;
        }
        __syncthreads();
        for (int j = threadIdx.x; j < lanes; j += kCellThreads) {
            const int li = LINES ? (int)s_lane[j] : (int)s_ord[j];
            if (LINES && li == 0xffff) continue;
            const float4 r = s_rec[li];
            const float q[3] = {r.x, r.y, r.z};
            float val, gu, gv, gw;
            if (!eval_point<P, LAYOUT, UNI, GRAD>(args, q, val, gu, gv, gw)) ++errs;
            args.out4[start + piece + li] = make_float4(val, gu, gv, gw);
        }
        __syncthreads();
    }
    if (args.n_err) {
        for (int o = 16; o > 0; o >>= 1) errs += __shfl_xor_sync(0xffffffffu, errs, o);
        if ((threadIdx.x & 31) == 0 && errs) atomicAdd(args.n_err, (unsigned long long)errs);
    }
}

template <int P, int LAYOUT, bool UNI, bool GRAD, bool SORTED>
static cudaError_t launch_eval_s(const EvalArgs& a, cudaStream_t st) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (a.n + 255) / 256;
    const int64_t grid = std::min<int64_t>(want, (int64_t)sms * 16);
    eval_kernel<P, LAYOUT, UNI, GRAD, SORTED><<<(unsigned)grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

template <int P, int LAYOUT, bool UNI, bool GRAD>
static cudaError_t launch_eval_t(const EvalArgs& a, cudaStream_t st) {
    if ((is_bez(LAYOUT) || eval_lines<P, LAYOUT>() || (MFA_EVAL_CELLS_QUADS && LAYOUT == kQuads)) && a.rec && a.bin_cnt) {
        eval_cells_kernel<P, LAYOUT, UNI, GRAD><<<(unsigned)(a.nbins + 1), kCellThreads, 0, st>>>(a);
        return cudaGetLastError();
    }
    if (a.rec) return launch_eval_s<P, LAYOUT, UNI, GRAD, true>(a, st);
    return launch_eval_s<P, LAYOUT, UNI, GRAD, false>(a, st);
}

template <int P, int LAYOUT>
static cudaError_t dispatch_eval_l(const EvalArgs& a, bool uni, bool grad, cudaStream_t st) {
    if (uni)
        return grad ? launch_eval_t<P, LAYOUT, true, true>(a, st) : launch_eval_t<P, LAYOUT, true, false>(a, st);
    return grad ? launch_eval_t<P, LAYOUT, false, true>(a, st) : launch_eval_t<P, LAYOUT, false, false>(a, st);
}

template <int P>
static cudaError_t dispatch_eval(const EvalArgs& a, int layout, bool uni, bool grad, cudaStream_t st) {
    if constexpr (P <= 3) {
        if (layout == kBezier) return dispatch_eval_l<P, kBezier>(a, uni, grad, st);
        if constexpr (P == 3)
            if (layout == kBezierG) return dispatch_eval_l<P, kBezierG>(a, uni, grad, st);
        if (layout == kBricks) return dispatch_eval_l<P, kBricks>(a, uni, grad, st);
    }
    return dispatch_eval_l<P, kQuads>(a, uni, grad, st);
}

// ---------------------------------------------------------------------------
// Spatial binning of a large point batch (mfa_eval_batch with a workspace).
// Random points gather their (p+1)^3 neighbourhoods from random places: each
// point touches ~16 separate 128-byte lines of a grid far larger than L2, so
// the kernel is HBM-bound on over-fetched lines (C3: ~1.5 KB of DRAM reads per
// point).  Grouping the points by a coarse parameter-space bin (about 8^3
// knot spans per bin; bin = floor(u * NB) per axis) makes the points a CTA
// processes share neighbourhoods, which then come from L1/L2: a counting sort
// (per-CTA shared-memory histogram, one scan, an atomic-cursor scatter of
// (u, v, w, index) records), then the evaluation in bin order writing each
// result at its original index.  The result of a point does not depend on
// its position in the order, so outputs stay deterministic.
// ---------------------------------------------------------------------------
#ifndef MFA_CURSOR_STRIDE  // unsigned words between scatter cursors (8: one 32-byte sector each)
#define MFA_CURSOR_STRIDE 8
#endif
#ifndef MFA_BIN_ILP      // points per thread per iteration in the binning / gather kernels (1 -> 4: C3 eval +6 %)
#define MFA_BIN_ILP 4
#endif
constexpr int kBinILP = MFA_BIN_ILP;
#ifndef MFA_BIN_SPANS    // knot spans per bin edge
#define MFA_BIN_SPANS 8
#endif

struct BinGrid {
    int nb[3];
    int nbins;   // nb0 * nb1 * nb2; points outside [0,1]^3 (or NaN) go to bin nbins
};

__device__ __forceinline__ int point_bin(const BinGrid& g, float u, float v, float w) {
    if (!(u >= 0.f && u <= 1.f && v >= 0.f && v <= 1.f && w >= 0.f && w <= 1.f)) return g.nbins;
    const int bu = min((int)(u * (float)g.nb[0]), g.nb[0] - 1);
    const int bv = min((int)(v * (float)g.nb[1]), g.nb[1] - 1);
    const int bw = min((int)(w * (float)g.nb[2]), g.nb[2] - 1);
    return (bw * g.nb[1] + bv) * g.nb[0] + bu;
}

#ifndef MFA_BIN_SMEM       // bins counted in shared memory (dynamic, opt-in above 48 KB)
#define MFA_BIN_SMEM 53248 // 208 KB: C3's 32^3 bins fit
#endif
constexpr int kBinSmem = MFA_BIN_SMEM;
#ifndef MFA_BIN_FIT   // 1: coarsen the bins of large models until the histogram fits in shared memory
#define MFA_BIN_FIT 1
#endif

__global__ void __launch_bounds__(1024) bin_count_kernel(const float* __restrict__ u, const float* __restrict__ v,
                                                        const float* __restrict__ w, int64_t n, const BinGrid g,
                                                        int* __restrict__ bins, unsigned* __restrict__ counts) {
    extern __shared__ unsigned sh[];
    const bool local = g.nbins + 1 <= kBinSmem;
    if (local)
        for (int b = threadIdx.x; b <= g.nbins; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    // kBinILP points per thread per iteration, each slice coalesced across the
    // grid: their loads are independent, so kBinILP x more are in flight
    const int64_t S = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += kBinILP * S) {
        float q[kBinILP][3];
#pragma unroll
        for (int k = 0; k < kBinILP; ++k) {
            const int64_t i = i0 + k * S;
            if (i < n) {
                q[k][0] = __ldg(u + i);
                q[k][1] = __ldg(v + i);
                q[k][2] = __ldg(w + i);
            }
        }
#pragma unroll
        for (int k = 0; k < kBinILP; ++k) {
            const int64_t i = i0 + k * S;
            if (i < n) {
                const int b = point_bin(g, q[k][0], q[k][1], q[k][2]);
                bins[i] = b;
                if (local) atomicAdd(sh + b, 1u);
                else atomicAdd(counts + b, 1u);
            }
        }
    }
    __syncthreads();
    if (local)
        for (int b = threadIdx.x; b <= g.nbins; b += blockDim.x)
            if (sh[b]) atomicAdd(counts + b, sh[b]);
}

// exclusive scan of nbins+1 counts into cursors: one CTA of 1024 threads walks
// the counts in tiles of 4096 (a coalesced 16-byte load per thread, a block
// scan by warp shuffles, a running carry)
__global__ void __launch_bounds__(1024) bin_scan_kernel(const unsigned* __restrict__ counts, int nb,
                                                        unsigned* __restrict__ cursor) {
    __shared__ unsigned wsum[32];
    __shared__ unsigned carry_s;
    const int tid = threadIdx.x;
    if (tid == 0) carry_s = 0;
    __syncthreads();
    for (int t0 = 0; t0 < nb; t0 += 4096) {
        unsigned c[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int b = t0 + 4 * tid + e;
            c[e] = b < nb ? counts[b] : 0u;
        }
        const unsigned tsum = c[0] + c[1] + c[2] + c[3];
        unsigned x = tsum;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if ((tid & 31) >= o) x += y;
        }
        if ((tid & 31) == 31) wsum[tid >> 5] = x;
        __syncthreads();
        if (tid < 32) {
            unsigned w = wsum[tid];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
                if (tid >= o) w += y;
            }
            wsum[tid] = w;   // inclusive over warps
        }
        __syncthreads();
        const unsigned carry = carry_s;
        unsigned run = carry + x - tsum + ((tid >> 5) ? wsum[(tid >> 5) - 1] : 0u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int b = t0 + 4 * tid + e;
            if (b < nb) cursor[(size_t)b * MFA_CURSOR_STRIDE] = run;
            run += c[e];
        }
        __syncthreads();
        if (tid == 1023) carry_s = run;
        __syncthreads();
    }
}

// bins[i] is replaced by the point's sorted position (for the gather back)
__global__ void __launch_bounds__(256) bin_scatter_kernel(const float* __restrict__ u, const float* __restrict__ v,
                                                          const float* __restrict__ w, int64_t n,
                                                          int* __restrict__ bins, unsigned* __restrict__ cursor,
                                                          float4* __restrict__ rec) {
    // kBinILP independent (load bin -> cursor atomic -> record store) chains
    // per thread (no gain measured here: the kernel is bound by the L2 atomic
    // rate, ~49 G cursor atomics/s; an atomic-free matrix variant with
    // per-chunk ranks measured slower)
    const int64_t S = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += kBinILP * S) {
        int b[kBinILP];
        unsigned pos[kBinILP];
#pragma unroll
        for (int k = 0; k < kBinILP; ++k) b[k] = i0 + k * S < n ? bins[i0 + k * S] : 0;
#pragma unroll
        for (int k = 0; k < kBinILP; ++k)
            if (i0 + k * S < n) pos[k] = atomicAdd(cursor + (size_t)b[k] * MFA_CURSOR_STRIDE, 1u);
#pragma unroll
        for (int k = 0; k < kBinILP; ++k) {
            const int64_t i = i0 + k * S;
            if (i < n) {
                rec[pos[k]] = make_float4(__ldg(u + i), __ldg(v + i), __ldg(w + i), __int_as_float((int)i));
                bins[i] = (int)pos[k];
            }
        }
    }
}

// results back to the caller's SoA arrays: coalesced writes at i, one 16-byte
// gather from the sorted position
__global__ void __launch_bounds__(256) bin_gather_kernel(const float4* __restrict__ out4, const int* __restrict__ pos,
                                                         int64_t n, float* __restrict__ value, float* __restrict__ du,
                                                         float* __restrict__ dv, float* __restrict__ dw) {
    const int64_t S = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += kBinILP * S) {
        int p[kBinILP];
        float4 r[kBinILP];
#pragma unroll
        for (int k = 0; k < kBinILP; ++k) p[k] = i0 + k * S < n ? __ldg(pos + i0 + k * S) : 0;
#pragma unroll
        for (int k = 0; k < kBinILP; ++k)
            if (i0 + k * S < n) r[k] = __ldg(out4 + p[k]);   // kBinILP random 16-byte reads in flight
#pragma unroll
        for (int k = 0; k < kBinILP; ++k) {
            const int64_t i = i0 + k * S;
            if (i < n) {
                value[i] = r[k].x;
                if (du) {
                    du[i] = r[k].y;
                    dv[i] = r[k].z;
                    dw[i] = r[k].w;
                }
            }
        }
    }
}

static BinGrid make_bins(const Model* m) {
    BinGrid g;
    int64_t total = 1;
    for (int d = 0; d < 3; ++d) {
        const int64_t S = m->n[d] - m->p;
        g.nb[d] = (int)std::max<int64_t>(1, (S + MFA_BIN_SPANS - 1) / MFA_BIN_SPANS);
        total *= g.nb[d];
    }
    while (total > (1 << 22)) {   // keep the bin table small
        for (int d = 0; d < 3; ++d) g.nb[d] = std::max(1, g.nb[d] / 2);
        total = (int64_t)g.nb[0] * g.nb[1] * g.nb[2];
    }
#if MFA_BIN_FIT
    // coarsen the axis with the most bins until the histogram fits in shared memory
    while (total + 1 > kBinSmem) {
        int d = 0;
        for (int e = 1; e < 3; ++e)
            if (g.nb[e] > g.nb[d]) d = e;
        if (g.nb[d] == 1) break;
        g.nb[d] = (g.nb[d] + 1) / 2;
        total = (int64_t)g.nb[0] * g.nb[1] * g.nb[2];
    }
#endif
    g.nbins = (int)total;
    return g;
}

size_t bin_workspace_bytes(const Model* m, int64_t n) {
    const BinGrid g = make_bins(m);
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return up(sizeof(int) * (size_t)n) + up(sizeof(float4) * (size_t)n) + up(sizeof(unsigned) * (g.nbins + 1)) +
           up(sizeof(unsigned) * (g.nbins + 1) * MFA_CURSOR_STRIDE);
}

size_t eval_workspace_bytes(const Model* m, int64_t n) { return bin_workspace_bytes(m, n); }

BinnedPoints bin_points(const Model* m, int64_t n, const float* u, const float* v, const float* w, void* ws,
                        cudaStream_t st) {
    const BinGrid g = make_bins(m);
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    char* b = (char*)ws;
    int* bins = (int*)b;
    float4* rec = (float4*)(b + up(sizeof(int) * (size_t)n));
    unsigned* counts = (unsigned*)(b + up(sizeof(int) * (size_t)n) + up(sizeof(float4) * (size_t)n));
    unsigned* cursor = (unsigned*)((char*)counts + up(sizeof(unsigned) * (g.nbins + 1)));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
    cudaMemsetAsync(counts, 0, sizeof(unsigned) * (g.nbins + 1), st);
    const size_t smem = g.nbins + 1 <= kBinSmem ? sizeof(unsigned) * (g.nbins + 1) : 0;
    unsigned cgrid = grid;
    if (smem > 48 * 1024) {   // one CTA per SM with a large table: fewer, longer CTAs amortise the flush
        cudaFuncSetAttribute(bin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(unsigned) * kBinSmem));
        cgrid = (unsigned)std::min<int64_t>((n + 1023) / 1024, (int64_t)sms);
    }
    bin_count_kernel<<<cgrid, smem > 48 * 1024 ? 1024 : 256, smem, st>>>(u, v, w, n, g, bins, counts);
    bin_scan_kernel<<<1, 1024, 0, st>>>(counts, g.nbins + 1, cursor);
    bin_scatter_kernel<<<grid, 256, 0, st>>>(u, v, w, n, bins, cursor, rec);
    return BinnedPoints{rec, bins, counts, cursor, MFA_CURSOR_STRIDE, {g.nb[0], g.nb[1], g.nb[2]}, g.nbins};
}

mfa_status launch_eval(const Model* m, int64_t n, const float* u, const float* v, const float* w, float* value,
                       float* du, float* dv, float* dw, unsigned long long* n_err, cudaStream_t st, void* ws,
                       size_t ws_bytes) {
    EvalArgs a;
    a.rec = nullptr;
    a.out4 = nullptr;
    a.pos = nullptr;
    a.bin_cnt = nullptr;
    a.bin_end = nullptr;
    if (ws && bin_worthwhile(m, n) && ws_bytes >= eval_workspace_bytes(m, n)) {
        const BinnedPoints bp = bin_points(m, n, u, v, w, ws, st);
        a.rec = bp.rec;
        a.out4 = bp.rec;   // results overwrite the records (after they are read)
        a.pos = bp.pos;
        if (MFA_EVAL_CELLS) {
            a.bin_cnt = bp.counts;
            a.bin_end = bp.cursor;
            a.bin_stride = bp.stride;
            for (int d = 0; d < 3; ++d) a.nb[d] = bp.nb[d];
            a.nbins = bp.nbins;
        }
    }
    a.Q = m->Q;
    a.g.nbx = m->nb[0];
    a.g.nby = m->nb[1];
    a.g.q_f4 = m->q_f4;
    a.bg.q_f4 = m->q_f4;
    a.bg.S0 = (int)(m->n[0] - m->p);
    a.bg.S1 = (int)(m->n[1] - m->p);
    a.bg.S0g = bez_groups(a.bg.S0, kGLu);
    a.bg.S1g = bez_groups(a.bg.S1, kGLv);
    for (int d = 0; d < 3; ++d) a.ax[d] = make_axis_args(m->ax[d]);
    a.u = u;
    a.v = v;
    a.w = w;
    a.value = value;
    a.du = du;
    a.dv = dv;
    a.dw = dw;
    a.n_err = n_err;
    a.n = n;
    const bool uni = m->uniform[0] && m->uniform[1] && m->uniform[2];
    const bool grad = du != nullptr;
    cudaError_t e;
    switch (m->p) {
        case 1: e = dispatch_eval<1>(a, m->layout, uni, grad, st); break;
        case 2: e = dispatch_eval<2>(a, m->layout, uni, grad, st); break;
        case 3: e = dispatch_eval<3>(a, m->layout, uni, grad, st); break;
        case 4: e = dispatch_eval<4>(a, m->layout, uni, grad, st); break;
        default: e = dispatch_eval<5>(a, m->layout, uni, grad, st); break;
    }
    if (e == cudaSuccess && a.rec) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
        bin_gather_kernel<<<grid, 256, 0, st>>>(a.out4, a.pos, n, value, du, dv, dw);
        e = cudaGetLastError();
    }
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "eval launch");
}

}  // namespace mfa
