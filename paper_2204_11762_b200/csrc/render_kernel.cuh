// render_kernel: Algorithm 1 fused per ray (shared by render.cu and
// truth.cu, which instantiate it without / with the extensions: the analytic
// ground-truth field of NEXT-2 and several directional lights, NEXT-4).
//
//   work = warp units of 4x8 pixels (8 per 16x16 tile) handed out by a global
//          atomic counter to persistent warps (grid = SMs x resident CTAs), so
//          early-terminating rays never leave an SM idle and no warp waits on
//          its CTA's slowest warp; consecutive units are neighbouring tiles.
//   ray  = one thread.  a1-a2 ray setup in fp64; sample positions are kept in
//          64-bit fixed point (the "fixed-point ray cast model"):
//          uniform axes in span units * 2^40, non-uniform axes in parameter
//          units * 2^62, advanced by an exact integer add per sample.
//   loop = a3 position -> a4 span/t -> a5 basis -> a6/a7 gather+contract ->
//          a8 TF (shared-memory table) -> a9 Phong -> a10 composite; the warp
//          leaves the loop when no lane is live (__any_sync), i.e. early ray
//          termination per ray with a warp-vote exit.
//   out  = premultiplied RGBA (fp32 or fp16) to the image or to a packed tile.
#pragma once
#include <type_traits>
#include <cuda_fp16.h>
#include <math.h>

#include <algorithm>
#include <mutex>

#include "kernels.cuh"

// MFA_ORDER = 1: the next sample's contraction waits on the current sample's
// compositing, so ptxas places the shading between the block loads and their
// first use (hides part of the reload latency; C5 +1.8 %)
// MFA_FLAT_LOOP = 1: branch-free sample loop for the register-cached layouts
// (finished lanes re-query a frozen sample, which never reloads); C5 +2 %, C3 +7 %
#ifndef MFA_UNIT_SHAPE   // lanes of a warp unit: 0 = 8x4 pixels, 1 = 4x8 (C5 +0.8 %, C4 +3 %), 2 = 16x2, 3 = 2x16
#define MFA_UNIT_SHAPE 1
#endif
#ifndef MFA_QUAD_LANES   // 1: on the grouped Bezier layout, 8 x 4 units whose 4-lane groups are 2 x 2 pixel quads
#define MFA_QUAD_LANES 1
#endif
#ifndef MFA_CENTER_OUT   // 1: single-view launches issue supertile rows from the image centre outward
#define MFA_CENTER_OUT 0
#endif
#ifndef MFA_VIEW_GROUP   // full-frame work order: >1 interleaves groups of orbit-adjacent views
#define MFA_VIEW_GROUP 4 // C5: DRAM per launch 506 -> 343 GB, L2 hit 44 -> 56 %, +1.4 %
#endif
#ifndef MFA_VIEW_ORDER   // with MFA_VIEW_GROUP > 1: 1 = per supertile, 2 = per supertile row, 3 = per tile
#define MFA_VIEW_ORDER 1
#endif
#ifndef MFA_MULTI_DEFER   // multi-span steps fixed behind one warp-uniform vote (see flat_loop)
#define MFA_MULTI_DEFER 2   // 2: and the block fetched before the span records arrive (C5 58.9 -> 61.4 G)
#endif
#ifndef MFA_DIAG_MULTICOUNT
#define MFA_DIAG_MULTICOUNT 0
#endif
#ifndef MFA_DIAG_NOMULTI   // diagnostic only (wrong where a step crosses several spans): never run the multi-span loop
#define MFA_DIAG_NOMULTI 0
#endif
#ifndef MFA_TF_PAIR   // the TF lerp as paired FP32 instructions
#define MFA_TF_PAIR 1   // C5 +0.35 % with the deferred multi-span loop (neutral before it)
#endif
#ifndef MFA_PRED_ADV   // experiment: the sample advance as a predicated add instead of a select
#define MFA_PRED_ADV 0
#endif
#ifndef MFA_BULK_PF   // experiment: bulk async prefetch of the block of the sample after next into shared memory
#define MFA_BULK_PF 0
#endif
#ifndef MFA_PREFETCH_NEXT   // experiment: 1 / 2 = prefetch the predicted next block into L1 / L2
#define MFA_PREFETCH_NEXT 0
#endif
#ifndef MFA_EARLY_LOAD   // experiment: issue the next sample's block load right after this sample's contraction
#define MFA_EARLY_LOAD 0
#endif
#ifndef MFA_FLAT_LOOP
#define MFA_FLAT_LOOP 1
#endif
#ifndef MFA_ORDER
#define MFA_ORDER 1
#endif

namespace mfa {

// NEXT-2 ground truth: the analytic field (Eq. 1-2) a sample takes
// its value and/or gradient from (see field_eval below).
struct FieldArgs {
    int kind;                     // MFA_FIELD_GAUSSIAN_BEAM / MFA_FIELD_MARSCHNER_LOBB
    int vsrc, gsrc;               // 1: analytic, 0: MFA query
    double prm[6];
    double fx_scale[3];           // fixed-point sample coordinate -> parameter u
    float invL[3];                // parameter-space gradient -> physical (R-4)
};

// NEXT-4 ("multiple light sources can be added in the future"):
// directional lights, unit direction towards the light and intensity.
constexpr int kMaxLights = MFA_MAX_LIGHTS;
struct LightArgs {
    int n;                        // 0: the headlight (R-11)
    float dir[kMaxLights][3];
    float intensity[kMaxLights];
};

struct ViewFrame {
    double eye[3], f[3], A[3], B[3];
    int ortho;
};

struct RenderArgs {
    const float4* Q;
    BrickGrid g;
    BezGrid bg;
    AxisArgs ax[3];
    const float4* tf;
    int tf_n;
    float v_lo, s_scale;          // f = (v - v_lo) * s_scale = s * (n - 1)
    double bmin[3], L[3];
    double step;
    // host-derived setup scales (render.cu): world offset -> fixed point per
    // axis ((S or 1) * 2^frac / L), 1 / step, 2 / W, 2 / H
    double fxs[3], inv_step, inv_w2, inv_h2;
    float gsc[3];                 // gradient scale to physical units (uniform: S/L; non-uniform: 1/L)
    float o_max, ka, kd, ks, shin, eps2;
    int W, H, tiles_x, tiles_y;
    int st_x, st_y;               // supertiles (MFA_SUPERTILE^2 tiles) per view, full-frame order
    int n_views;
    const int* tiles;             // NULL: full frames
    int tile_scatter;             // tiles: 1 = write pixels at their image position, 0 = packed tiles
    int64_t n_tiles;
    int64_t n_units;              // warp units = 8 per tile
    int view_base;                // full frames: output view index of cams[0]
    unsigned int* queue;          // work counter (zeroed before the launch)
    void* out;
    int out_fp16;
    unsigned long long* samples;
    FieldArgs fld;                // used by the EXT instantiations only
    LightArgs lights;             // used by the EXT instantiations only
    struct {                      // curvature transfer function (EXT only; R-31)
        const float4* tab;        // [n][n] RGBA, [kappa_2][kappa_1]
        int n;                    // 0: off
        float scale, range;       // index = (kappa + range) * scale, scale = (n - 1) / (2 range)
    } curv;
    const unsigned* tbits;        // SHADE == 3: bit per macro block, 1 = the TF is transparent over its value range
    int mm0, mm1;                 // SHADE == 3: macro blocks along u, v
    int mm_n;                     // SHADE == 3: macro blocks in all (bounds checks)
    ViewFrame frames[kMaxViewsPerLaunch];   // per view, computed on the host (compute_frame)
};

__host__ __device__ inline void compute_frame(const mfa_camera& c, ViewFrame& fr) {
    double f[3] = {c.look_at[0] - c.eye[0], c.look_at[1] - c.eye[1], c.look_at[2] - c.eye[2]};
    double lf = sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
    for (int i = 0; i < 3; ++i) f[i] /= lf;
    double r[3] = {f[1] * c.up[2] - f[2] * c.up[1], f[2] * c.up[0] - f[0] * c.up[2], f[0] * c.up[1] - f[1] * c.up[0]};
    double lr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    for (int i = 0; i < 3; ++i) r[i] /= lr;
    double u[3] = {r[1] * f[2] - r[2] * f[1], r[2] * f[0] - r[0] * f[2], r[0] * f[1] - r[1] * f[0]};
    const double aspect = (double)c.width / (double)c.height;
    double sx, sy;
    if (c.fov_y_deg > 0.0) {
        const double th = tan(0.5 * c.fov_y_deg * 3.14159265358979323846 / 180.0);
        sx = aspect * th;
        sy = th;
        fr.ortho = 0;
    } else {
        sx = aspect * c.ortho_half_height;
        sy = c.ortho_half_height;
        fr.ortho = 1;
    }
    for (int i = 0; i < 3; ++i) {
        fr.eye[i] = c.eye[i];
        fr.f[i] = f[i];
        fr.A[i] = sx * r[i];
        fr.B[i] = sy * u[i];
    }
}

// Analytic field value and parameter-space gradient at parameter point u
// (fp64).  x = 2u - 1 on [-1,1]^3, d/du = 2 d/dx.
//   Gaussian beam (Eq. 1): F = V_min + (V_max - V_min) G(r/R),
//     G(l) = exp(-(l - mu)^2 / (2 sigma^2)), r = |x|
//   Marschner-Lobb (Eq. 2): F = (1 - sin(pi z/2) + alpha (1 + rho(r))) / (2 (1 + alpha)),
//     rho(r) = cos(2 pi f_M cos(pi r/2)), r = sqrt(x^2 + y^2)
__device__ __forceinline__ void field_eval(const FieldArgs& f, const double (&u)[3], double (&out)[4]) {
    const double x = 2.0 * u[0] - 1.0, y = 2.0 * u[1] - 1.0, z = 2.0 * u[2] - 1.0;
    if (f.kind == MFA_FIELD_GAUSSIAN_BEAM) {
        const double r = sqrt(x * x + y * y + z * z), l = r / f.prm[4], dl = l - f.prm[2];
        const double G = exp(-dl * dl / (2.0 * f.prm[3] * f.prm[3]));
        const double A = f.prm[1] - f.prm[0];
        out[0] = f.prm[0] + A * G;
        const double c = r > 0.0 ? 2.0 * A * G * (-dl / (f.prm[3] * f.prm[3])) / (f.prm[4] * r) : 0.0;
        out[1] = c * x;
        out[2] = c * y;
        out[3] = c * z;
    } else {
        const double fm = f.prm[0], al = f.prm[1], den = 2.0 * (1.0 + al);
        const double r = sqrt(x * x + y * y);
        double sr, cr, sz, cz;
        sincospi(0.5 * r, &sr, &cr);
        sincospi(0.5 * z, &sz, &cz);
        double sa, ca;
        sincospi(2.0 * fm * cr, &sa, &ca);
        out[0] = (1.0 - sz + al * (1.0 + ca)) / den;
        const double drho = sa * 2.0 * M_PI * fm * sr * (0.5 * M_PI);
        const double c = r > 0.0 ? 2.0 * al * drho / (r * den) : 0.0;
        out[1] = c * x;
        out[2] = c * y;
        out[3] = 2.0 * (-(0.5 * M_PI) * cz / den);
    }
}

#ifndef MFA_FAST_POW
#define MFA_FAST_POW 1
#endif

// x^n for the Phong specular term: 2^(n log2 x) with the ftz approximations
// (no denormal fix-up sequences; x = 0 -> 0 for n > 0; a specular term below
// 2^-126 is flushed to 0, far under the image tolerance)
// 1/sqrt(x) for x >= 1e-37 (a normal float): the ftz form has no denormal
// fix-up (3 instructions per sample) and gives the same result on this domain
__device__ __forceinline__ float rsqrt_normal(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float pow_spec(float x, float n) {
#if MFA_FAST_POW
    float l, r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(n * l));
    return r;
#else
    return exp2f(n * __log2f(x));
#endif
}

// Launch shape per instantiation (measured on B200):
//   p <= 3 (neighbourhood cache, ~160-170 registers): 128-thread CTAs, >= 3 per SM
//   p >= 4 (streamed slabs): 256-thread CTAs capped at 128 registers (2 per SM)
#ifndef MFA_RENDER_CACHE
#define MFA_RENDER_CACHE 1
#endif
#ifndef MFA_BEZ_CACHE
#define MFA_BEZ_CACHE 1
#endif
#ifndef MFA_LANE_STATS   // diagnostic build only
#define MFA_LANE_STATS 0
#endif
#ifndef MFA_SMEM_FRAMES  // 1: per-view frames in shared memory (computed once per CTA)
#define MFA_SMEM_FRAMES 0
#endif
#ifndef MFA_CARVE_FLOOR  // sized carveout: at least this percentage of shared memory
#define MFA_CARVE_FLOOR 8
#endif
#ifndef MFA_CARVEOUT     // -1: sized for MINB CTAs (default), else a fixed percentage
#define MFA_CARVEOUT -1
#endif
#ifndef MFA_CTA_TILES    // -1: per shape (p >= 4), 0: off, 1: on
#define MFA_CTA_TILES -1
#endif

template <int P, int LAYOUT>
struct RenderShape {
    static constexpr bool BEZ = is_bez(LAYOUT);
    static constexpr bool CACHE = BEZ ? (bool)MFA_BEZ_CACHE : (MFA_RENDER_CACHE && P <= 3);
#ifdef MFA_RENDER_THREADS
    static constexpr int THREADS = MFA_RENDER_THREADS;
#else
    static constexpr int THREADS = P <= 3 ? 128 : 256;
#endif
#ifdef MFA_RENDER_MINB
    static constexpr int MINB = MFA_RENDER_MINB;
#else
    // plain bricks: the 8-float row windows of a reload need registers (2 CTAs)
    static constexpr int MINB = LAYOUT == kBricks ? 2 : (P <= 3 ? (CACHE ? 3 : 4) : 2);
#endif
    // p >= 4: a CTA (8 warps) takes a whole 16x16 tile so its sub-tiles share L1
    static constexpr bool CTA_TILES = MFA_CTA_TILES < 0 ? (P >= 4 && THREADS == 256) : (bool)MFA_CTA_TILES;
};

// SHADE: 0 = ShadingOn false (value only, Alg. 1 l.8), 1 = the ★ path (value
// + gradient for every sample, R-20), 2 = NEXT-1's measured variant: the
// gradient contraction and Phong are skipped for a sample whose TF opacity is
// 0 (it composites with weight 0, so the image is bit-identical to SHADE = 1);
// 3 = the transparent-block skip: a sample whose macro block's value range
// (Bernstein convex hull) maps to TF opacity 0 is neither fetched nor queried
// (it too composites with weight 0: bit-identical to SHADE = 1)
#ifdef MFA_RENDER_MAXNREG   // experiment: an explicit register cap instead of the launch-bounds occupancy
#define MFA_RENDER_BOUNDS __maxnreg__(MFA_RENDER_MAXNREG)
#else
#define MFA_RENDER_BOUNDS __launch_bounds__(RenderShape<P, LAYOUT>::THREADS, RenderShape<P, LAYOUT>::MINB)
#endif
template <int P, int LAYOUT, bool UNI, int SHADE, bool EXT>
__global__ void MFA_RENDER_BOUNDS render_kernel(const __grid_constant__ RenderArgs args) {
    constexpr bool BEZ = is_bez(LAYOUT);
    constexpr int SEC = bez_sec(LAYOUT == kBezierG);
    constexpr bool CACHE = RenderShape<P, LAYOUT>::CACHE;
    extern __shared__ float4 s_tf[];
#if MFA_SMEM_FRAMES
    __shared__ ViewFrame s_frame[kMaxViewsPerLaunch];
#endif

#if MFA_SMEM_FRAMES
    for (int v = threadIdx.x; v < args.n_views; v += blockDim.x) s_frame[v] = args.frames[v];
#endif
    for (int i = threadIdx.x; i < args.tf_n; i += blockDim.x) s_tf[i] = __ldg(args.tf + i);
#if MFA_BULK_PF
    // experiment: the block of the sample after next is prefetched by a bulk
    // async copy (cp.async.bulk, completion on a per-thread mbarrier) into a
    // per-thread shared-memory slot a whole iteration before it is needed
    constexpr bool kPF = LAYOUT == kBezier && CACHE && !EXT && !UNI && P == 3;
    constexpr int kPFT = kPF ? RenderShape<P, LAYOUT>::THREADS : 1;
    __shared__ __align__(16) float s_pf[kPFT][kPF ? 68 : 4];   // 256 B + 16 B pad: conflict-free float4 reads
    __shared__ __align__(8) unsigned long long s_mbar[kPFT];
    if constexpr (kPF) {
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&s_mbar[threadIdx.x]);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int pf_key = -1;
    unsigned pf_phase = 0;
    bool pf_pending = false;
    auto pf_wait = [&]() {
        if constexpr (kPF) {
            const unsigned mb = (unsigned)__cvta_generic_to_shared(&s_mbar[threadIdx.x]);
            asm volatile(
                "{\n\t.reg .pred P1;\n\t"
                "LAB_WAIT:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                "@P1 bra DONE;\n\t"
                "bra LAB_WAIT;\n\t"
                "DONE:\n\t}" ::"r"(mb),
                "r"(pf_phase)
                : "memory");
            pf_phase ^= 1u;
            pf_pending = false;
        }
    };
#endif
    __syncthreads();

    const int lane = threadIdx.x & 31;
    constexpr int kST = MFA_SUPERTILE, kST2 = MFA_SUPERTILE * MFA_SUPERTILE;
    const int per_view = args.st_x * args.st_y * kST2;   // units are ordered by supertiles of tiles
    unsigned long long my_samples = 0;
#if MFA_DIAG_MULTICOUNT   // diagnostic: lane-samples / warp-iterations with a multi-span step (samples[1..3])
    unsigned long long dm_lane = 0, dm_warp = 0, dm_iters = 0;
#endif
#if MFA_LANE_STATS
    unsigned long long lane_slots = 0, lane_live = 0;
#endif

    constexpr int kWarps = RenderShape<P, LAYOUT>::THREADS / 32;
    __shared__ unsigned s_tile;
    unsigned tile_base = 0;
    int round_sub = 0;
    for (;;) {
        unsigned unit = 0;
        if constexpr (RenderShape<P, LAYOUT>::CTA_TILES) {
            // ---- the CTA takes a whole 16x16 tile; its warps share its 8
            // sub-units, so neighbouring rays reuse blocks in this SM's L1
            if (round_sub == 0) {
                __syncthreads();
                if (threadIdx.x == 0) s_tile = atomicAdd(args.queue, 1u);
                __syncthreads();
                tile_base = s_tile * 8u;
            }
            unit = tile_base + (unsigned)((threadIdx.x >> 5) + round_sub * kWarps);
            round_sub = (round_sub + 1) % (8 / kWarps);
            if (tile_base >= args.n_units) break;
        } else {
            // ---- next warp unit (32 pixels, MFA_UNIT_SHAPE) from the global queue ---------
            if (lane == 0) unit = atomicAdd(args.queue, 1u);
            unit = __shfl_sync(0xffffffffu, unit, 0);
            if (unit >= args.n_units) break;
        }
        const int64_t tile_id = unit >> 3;
        const int sub = unit & 7;
        int view, tx, ty;
        if (args.tiles) {
            view = __ldg(args.tiles + 3 * tile_id);
            tx = __ldg(args.tiles + 3 * tile_id + 1);
            ty = __ldg(args.tiles + 3 * tile_id + 2);
            // padding units (view = -1, multi-GPU equal-size buffers) and any
            // malformed entry (view or tile outside this launch) are skipped:
            // a bad list must never index frames[] or store outside the image
            if (view < 0 || view >= args.n_views || tx < 0 || ty < 0 || tx >= args.tiles_x || ty >= args.tiles_y)
                continue;
        } else {
            // supertile order: the ~200 tiles in flight form a compact image
            // region, so neighbouring rays reuse control blocks from L1/L2
            const unsigned tid32 = (unsigned)tile_id;   // < 2^29 (n_units < 2^32)
#if MFA_VIEW_GROUP > 1
            // cross-view order: groups of MFA_VIEW_GROUP consecutive (orbit-
            // adjacent) views; inside a group the same supertile (ORDER 1) or
            // supertile row (ORDER 2) of every view is issued back to back
            unsigned st, lt;
            {
                constexpr unsigned G = MFA_VIEW_GROUP;
                const unsigned grp = tid32 / ((unsigned)per_view * G);
                const unsigned r = tid32 - grp * (unsigned)per_view * G;
                const unsigned gv = min(G, (unsigned)args.n_views - grp * G);   // views in this group
#if MFA_VIEW_ORDER == 2
                const unsigned row = (unsigned)args.st_x * kST2;                 // tiles per supertile row
                const unsigned rr = r / (row * gv), rem = r - rr * row * gv;
                const unsigned vin = rem / row, q = rem - vin * row;
                st = rr * (unsigned)args.st_x + q / kST2;
                lt = q % kST2;
#elif MFA_VIEW_ORDER == 3   // per tile: tile (st, lt) of every view of the group back to back
                st = r / (kST2 * gv);
                const unsigned rem = r - st * kST2 * gv;
                lt = rem / gv;
                const unsigned vin = rem - lt * gv;
#else
                st = r / (kST2 * gv);
                const unsigned rem = r - st * kST2 * gv;
                const unsigned vin = rem / kST2;
                lt = rem - vin * kST2;
#endif
                view = (int)(grp * G + vin);
            }
#else
            view = (int)(tid32 / (unsigned)per_view);
            const unsigned t = tid32 - (unsigned)view * (unsigned)per_view;
            const unsigned st = t / kST2, lt = t % kST2;
#endif
            unsigned sty = st / (unsigned)args.st_x;
            unsigned stx = st - sty * (unsigned)args.st_x;
#if MFA_CENTER_OUT
            // single-view launches (short: C2 0.18 ms, C3 0.87 ms): supertile rows
            // from the image centre outward (mid, mid-1, mid+1, ...), so the
            // longest rays start first and the short border rays form the
            // launch's tail; a permutation of the work order only
            if (args.n_views == 1) {
                const unsigned mid = (unsigned)args.st_y >> 1, h = (sty + 1u) >> 1;
                sty = (sty & 1u) ? mid - h : mid + h;
#if MFA_CENTER_OUT == 2   // columns too: each row's corners last
                const unsigned midx = (unsigned)args.st_x >> 1, hx = (stx + 1u) >> 1;
                stx = (stx & 1u) ? midx - hx : midx + hx;
#endif
            }
#endif
            tx = (int)(stx * kST + lt % kST);
            ty = (int)(sty * kST + lt / kST);
            if (tx >= args.tiles_x || ty >= args.tiles_y) continue;
        }
#if MFA_SMEM_FRAMES
        const ViewFrame& fr = s_frame[view];
#else
        // the view's frame (kernel parameters, computed on the host by
        // compute_frame; uniform across the warp, no shared memory)
        const ViewFrame& fr = args.frames[view];
#endif
        // MFA_UNIT_SHAPE; on the grouped Bezier layout the unit is 8 x 4 pixels
        // with its aligned 4-lane groups as 2 x 2 pixel quads (the L1 data pipe
        // serves an LDG.256 in groups of 4 lanes, one wavefront per distinct
        // 128-byte line in a group): C5 61.45 -> 62.2 G samples/s (4 x 8 with
        // quads: 61.69), images bit-identical; the quad layout keeps 4 x 8 with
        // 4 x 1 rows (quads there: C3 -2.5 %)
        constexpr int kShape = (MFA_UNIT_SHAPE == 1 && MFA_QUAD_LANES && LAYOUT == kBezierG) ? 5 : MFA_UNIT_SHAPE;
        int lx, ly;
        if constexpr (kShape == 1) {          // 4 x 8 pixels per warp unit, 4-lane groups 4 x 1
            lx = (sub & 3) * 4 + (lane & 3);
            ly = (sub >> 2) * 8 + (lane >> 2);
        } else if constexpr (kShape == 4) {   // 4 x 8, 4-lane groups 2 x 2 (experiment)
            lx = (sub & 3) * 4 + ((lane >> 2) & 1) * 2 + (lane & 1);
            ly = (sub >> 2) * 8 + (lane >> 3) * 2 + ((lane >> 1) & 1);
        } else if constexpr (kShape == 5) {   // 8 x 4, 4-lane groups 2 x 2 (grouped Bezier default)
            lx = (sub & 1) * 8 + ((lane >> 2) & 3) * 2 + (lane & 1);
            ly = (sub >> 1) * 4 + (lane >> 4) * 2 + ((lane >> 1) & 1);
        } else if constexpr (kShape == 6) {   // 16 x 2, 4-lane groups 2 x 2 (experiment)
            lx = (lane >> 2) * 2 + (lane & 1);
            ly = sub * 2 + ((lane >> 1) & 1);
        } else if constexpr (kShape == 2) {   // 16 x 2
            lx = lane & 15;
            ly = sub * 2 + (lane >> 4);
        } else if constexpr (kShape == 3) {   // 2 x 16
            lx = sub * 2 + (lane & 1);
            ly = lane >> 1;
        } else {                              // 8 x 4
            lx = (sub & 1) * 8 + (lane & 7);
            ly = (sub >> 1) * 4 + (lane >> 3);
        }
        const int px = tx * MFA_TILE + lx, py = ty * MFA_TILE + ly;
        const bool valid = px < args.W && py < args.H;

        // ---- a1: ray through the pixel centre (fp64) -----------------------
        double o[3], d[3];
        {
            const double X = (px + 0.5) * args.inv_w2 - 1.0;
            const double Y = 1.0 - (py + 0.5) * args.inv_h2;
            if (fr.ortho) {
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    o[i] = fr.eye[i] + X * fr.A[i] + Y * fr.B[i];
                    d[i] = fr.f[i];
                }
            } else {
                double l2 = 0.0;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    o[i] = fr.eye[i];
                    d[i] = fr.f[i] + X * fr.A[i] + Y * fr.B[i];
                    l2 += d[i] * d[i];
                }
                const double il = 1.0 / sqrt(l2);
#pragma unroll
                for (int i = 0; i < 3; ++i) d[i] *= il;
            }
        }
        // ---- a2: slab clip; K samples at t_in + (k+1/2) step (R-7) ---------
        int K = 0;
        double t_in = 0.0;
        {
            double tn = -1e300, tf = 1e300;
            bool hit = valid;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const double bmax = args.bmin[i] + args.L[i];
                if (d[i] == 0.0) {
                    if (o[i] < args.bmin[i] || o[i] > bmax) hit = false;
                    continue;
                }
                const double id = 1.0 / d[i];
                const double t0 = (args.bmin[i] - o[i]) * id, t1 = (bmax - o[i]) * id;
                tn = fmax(tn, fmin(t0, t1));
                tf = fmin(tf, fmax(t0, t1));
            }
            t_in = fmax(tn, 0.0);
            if (hit && tf > t_in) {
                const double frc = (tf - t_in) * args.inv_step - 0.5;
                // (validate_render bounds the box diagonal / step below 2^30)
                K = frc > 0.0 ? (int)ceil(fmin(frc, 1073741824.0)) : 0;
            }
        }
        // ---- a3 setup: fixed-point sample coordinates per axis --------------
        long long F[3], DF[3];
        NUAxis nu[UNI ? 1 : 3];
        {
            const double t0 = t_in + 0.5 * args.step;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                // u = (x - b) / L in fixed point: one scale per axis from the host
                F[i] = llrint((o[i] + t0 * d[i] - args.bmin[i]) * args.fxs[i]);
                DF[i] = llrint(args.step * d[i] * args.fxs[i]);
                if (!UNI) {
                    if constexpr (!UNI) {
#if MFA_FLAT_LOOP   // every lane keeps a valid span state (lanes without samples query a fixed point)
                        if (K == 0) F[i] = DF[i] = 0;
                        nu_init(args.ax[i], F[i], nu[i]);
#else
                        if (K > 0) nu_init(args.ax[i], F[i], nu[i]);
#endif
                    }
                }
            }
        }
        const float dx = (float)d[0], dy = (float)d[1], dz = (float)d[2];

        float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
        int k = 0;
        bool live = K > 0;
        float nb[CACHE ? P + 1 : 1][P + 1][P + 1];   // cached neighbourhood (CACHE)
        std::conditional_t<BEZ, int, int64_t> nb_key = -1;   // Bezier: 32-bit block index
        constexpr bool kFlat = MFA_FLAT_LOOP && !EXT && CACHE;   // without the cache a frozen lane would reload

        // a6: make the neighbourhood of span triple s resident (CACHE layouts)
        auto fetch = [&](const int (&s)[3]) {
            if constexpr (BEZ && CACHE && LAYOUT == kBezierG) {
                // key = the block's offset in 32-byte units (< 2^31: mfa_model_create)
                const int e = bez_group_key<int>(args.bg.S0g, args.bg.S1g, s[0], s[1], s[2]);
                if (e != nb_key) {
                    load_bblock<P, SEC>(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(args.Q) + (int64_t)e * 8), nb);
                    nb_key = e;
                }
            } else if constexpr (BEZ && CACHE) {
                const int e = (s[2] * args.bg.S1 + s[1]) * args.bg.S0 + s[0];
#if MFA_DIAG_NORELOAD   // diagnostic only (wrong images): a lane keeps its first block, no reloads
                if (nb_key < 0) {
#else
                if (e != nb_key) {       // reload only when the span triple changed
#endif
#if MFA_DIAG_L1   // diagnostic only (wrong images): every reload reads one of 64 L1-resident blocks
                    load_bblock<P>(bez_block_at<P>(args.Q, args.bg, e & 63), nb);
#else
                    load_bblock<P>(bez_block_at<P>(args.Q, args.bg, e), nb);
#endif
                    nb_key = e;
                }
            } else if constexpr (CACHE && LAYOUT == kBricks) {
                const PlainRef e = plain_entry<P>(args.g, s[0], s[1], s[2]);
                if (e.base + e.o != nb_key) {
                    load_pblock<P>(args.Q, e, nb);
                    nb_key = e.base + e.o;
                }
            } else if constexpr (CACHE) {
                const int64_t e = brick_entry<P>(args.g, s[0], s[1], s[2]);
                if (e != nb_key) {
                    load_block<P>(args.Q + e, nb);
                    nb_key = e;
                }
            }
        };
        // SHADE == 3: is the sample's macro block transparent under this TF?
        auto transparent = [&](const int (&s)[3]) -> bool {
            if constexpr (SHADE == 3) {
                const int mi = ((s[2] >> kMacroLog) * args.mm1 + (s[1] >> kMacroLog)) * args.mm0 + (s[0] >> kMacroLog);
                MFA_DCHECK(mi >= 0 && mi < args.mm_n);
                return (__ldg(args.tbits + (mi >> 5)) >> (mi & 31)) & 1u;
            } else {
                return false;
            }
        };
        // a4: span + local coordinate per axis of the sample at F
        auto locate = [&](int (&s)[3], float (&t)[3], float (&gs)[3], auto multi_tag) {
            constexpr bool MULTI = decltype(multi_tag)::value;
#if MFA_NU_SPLIT
            if constexpr (!UNI) {
#pragma unroll
                for (int i = 0; i < 3; ++i) nu_cross(args.ax[i], F[i], nu[i]);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    t[i] = nu_finish<MULTI>(args.ax[i], F[i], nu[i]);
                    s[i] = nu[i].s;
                    gs[i] = nu_gscale(args.ax[i], nu[i]);
                }
                return;
            }
#endif
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                if constexpr (UNI) {
                    uni_span_fx(F[i], args.ax[i].nsp, s[i], t[i]);
                    gs[i] = args.gsc[i];
                } else {
#if MFA_NU_SPLIT
                    __builtin_unreachable();   // handled above
#else
                    t[i] = nu_span(args.ax[i], F[i], nu[i]);
                    s[i] = nu[i].s;
                    gs[i] = nu_gscale(args.ax[i], nu[i]);
#endif
                }
            }
        };
        // a8 lookup position: f = s (n - 1) clamped, i0 = round(f - 1/2) via the
        // 2^23 magic number (no F2I; any i0 in {floor(f), f - 1 at integers}
        // gives the same lerp), weight wt (shared by shade_composite and the
        // SHADE == 2 opacity test, so both see the same alpha)
        auto tf_pos = [&](float v, int& i0, float& wt) {
            float f = (v - args.v_lo) * args.s_scale;
            f = fminf(fmaxf(f, 0.f), (float)(args.tf_n - 1));
            const float fm = f + 8388607.5f;
            i0 = __float_as_int(fm) - 0x4b000000;
            i0 = min(max(i0, 0), args.tf_n - 2);
            wt = f - (float)i0;
        };
        auto tf_alpha = [&](float v) {
            int i0;
            float wt;
            tf_pos(v, i0, wt);
            const float a0 = s_tf[i0].w, a1 = s_tf[i0 + 1].w;
            return fmaf(wt, a1 - a0, a0);
        };
        // a5 + a7: value and t-space gradient of the sample (after fetch)
        auto query = [&](const int (&s)[3], const float (&t)[3], float& val, float& gu, float& gv, float& gw) {
            gu = gv = gw = 0.f;
            if constexpr (BEZ && !CACHE) {   // stream the block slab by slab
                const float4* q = bez_block<P, SEC>(args.Q, args.bg, s[0], s[1], s[2]);
                float r0[P + 1][P + 1];
                load_bslab<P, SEC>(q, r0);
                if (SHADE) {
                    float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
                    bernstein<P, false>(t[0], Bu);
                    bernstein<P, true>(t[1], Bv);
                    bernstein<P, false>(t[2], Bw);
                    contract_vg_bez<P, SEC>(q, r0, Bu, Bv, Bw, val, gu, gv, gw);
                } else {
                    float nbv[P + 1][P + 1][P + 1];
                    load_bblock<P, SEC>(q, nbv);
                    float Nu[P + 1], Nv[P + 1], Nw[P + 1];
                    bernstein_value<P>(t[0], Nu);
                    bernstein_value<P>(t[1], Nv);
                    bernstein_value<P>(t[2], Nw);
                    val = contract_v_cached<P>(nbv, Nu, Nv, Nw);
                }
            } else if constexpr (BEZ) {
                if (SHADE) {  // Bernstein basis, the same polynomials on every span
                    float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
                    bernstein<P, false>(t[0], Bu);
                    bernstein<P, true>(t[1], Bv);
                    bernstein<P, false>(t[2], Bw);
                    if constexpr (SHADE == 2) {   // value first; the gradient only where the TF is not transparent
                        val = contract_v_pairs<P>(nb, Bu, Bv, Bw);
                        if (tf_alpha(val) > 0.f) contract_vg_cached<P>(nb, Bu, Bv, Bw, val, gu, gv, gw);
                    } else {
                        contract_vg_cached<P>(nb, Bu, Bv, Bw, val, gu, gv, gw);
                    }
                } else {
                    float Nu[P + 1], Nv[P + 1], Nw[P + 1];
                    bernstein_value<P>(t[0], Nu);
                    bernstein_value<P>(t[1], Nv);
                    bernstein_value<P>(t[2], Nw);
                    val = contract_v_cached<P>(nb, Nu, Nv, Nw);
                }
            } else if constexpr (CACHE) {
                if (SHADE) {
                    float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
                    axis_basis<P, false>(args.ax[0], UNI, s[0], t[0], Bu);
                    axis_basis<P, true>(args.ax[1], UNI, s[1], t[1], Bv);
                    axis_basis<P, false>(args.ax[2], UNI, s[2], t[2], Bw);
                    if constexpr (SHADE == 2) {
                        val = contract_v_pairs<P>(nb, Bu, Bv, Bw);
                        if (tf_alpha(val) > 0.f) contract_vg_cached<P>(nb, Bu, Bv, Bw, val, gu, gv, gw);
                    } else {
                        contract_vg_cached<P>(nb, Bu, Bv, Bw, val, gu, gv, gw);
                    }
                } else {
                    float Nu[P + 1], Nv[P + 1], Nw[P + 1];
                    axis_basis_value<P>(args.ax[0], UNI, s[0], t[0], Nu);
                    axis_basis_value<P>(args.ax[1], UNI, s[1], t[1], Nv);
                    axis_basis_value<P>(args.ax[2], UNI, s[2], t[2], Nw);
                    val = contract_v_cached<P>(nb, Nu, Nv, Nw);
                }
            } else {
                const float4* q = args.Q + brick_entry<P>(args.g, s[0], s[1], s[2]);
                // issue slab 0 before the basis math; slabs stream through a double buffer
                float r0[P + 1][P + 1];
                load_slab<P>(q, r0);
                if (SHADE) {  // a5 + a7 with derivatives (Alg.1 l.6 and l.9)
                    float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
                    axis_basis<P, false>(args.ax[0], UNI, s[0], t[0], Bu);
                    axis_basis<P, true>(args.ax[1], UNI, s[1], t[1], Bv);
                    axis_basis<P, false>(args.ax[2], UNI, s[2], t[2], Bw);
                    contract_vg<P>(q, r0, Bu, Bv, Bw, val, gu, gv, gw);
                } else {      // value only (Alg.1 l.8 ShadingOn == false)
                    float Nu[P + 1], Nv[P + 1], Nw[P + 1];
                    axis_basis_value<P>(args.ax[0], UNI, s[0], t[0], Nu);
                    axis_basis_value<P>(args.ax[1], UNI, s[1], t[1], Nv);
                    axis_basis_value<P>(args.ax[2], UNI, s[2], t[2], Nw);
                    val = contract_v<P>(q, r0, Nu, Nv, Nw);
                }
            }
        };
        // a8-a10 for one queried sample, branch-free (so it can interleave
        // with the next sample's query)
        float order_dep = 0.f;   // MFA_ORDER: the value the next contraction waits on
        bool comp_on = true;     // MFA_FLAT_LOOP: this lane composites the sample it shades
        auto shade_composite = [&](float val, float gu, float gv, float gw, const float (&gs)[3], float k1,
                                   float k2) {
            // a8: transfer function (l.7)
            int i0;
            float wt;
            tf_pos(val, i0, wt);
            MFA_DCHECK(i0 >= 0 && i0 + 1 < args.tf_n);
            const float4 T0 = s_tf[i0], T1 = s_tf[i0 + 1];
#if MFA_TF_PAIR   // the same lerps as paired FP32 (FADD2 / FFMA2): bit-identical, half the instructions
            const float2 w2 = make_float2(wt, wt);
            const float2 rg = __ffma2_rn(w2, __fadd2_rn(make_float2(T1.x, T1.y), make_float2(-T0.x, -T0.y)),
                                         make_float2(T0.x, T0.y));
            const float2 ba = __ffma2_rn(w2, __fadd2_rn(make_float2(T1.z, T1.w), make_float2(-T0.z, -T0.w)),
                                         make_float2(T0.z, T0.w));
            float cr = rg.x, cg = rg.y, cb = ba.x;
            float a = ba.y;
#else
            float cr = fmaf(wt, T1.x - T0.x, T0.x);
            float cg = fmaf(wt, T1.y - T0.y, T0.y);
            float cb = fmaf(wt, T1.z - T0.z, T0.z);
            float a = fmaf(wt, T1.w - T0.w, T0.w);
#endif
            if constexpr (EXT) {   // curvature TF: bilinear in (kappa_1, kappa_2), modulates colour and opacity
                if (args.curv.n > 0) {
                    const float x = fminf(fmaxf((k1 + args.curv.range) * args.curv.scale, 0.f), (float)(args.curv.n - 1));
                    const float y = fminf(fmaxf((k2 + args.curv.range) * args.curv.scale, 0.f), (float)(args.curv.n - 1));
                    const int ix = min((int)x, args.curv.n - 2), iy = min((int)y, args.curv.n - 2);
                    const float fx = x - (float)ix, fy = y - (float)iy;
                    const float4* T = args.curv.tab + (int64_t)iy * args.curv.n + ix;
                    const float4 a00 = __ldg(T), a01 = __ldg(T + 1), a10 = __ldg(T + args.curv.n),
                                 a11 = __ldg(T + args.curv.n + 1);
                    auto bl = [&](float p00, float p01, float p10, float p11) {
                        return fmaf(fy, fmaf(fx, p11 - p10, p10) - fmaf(fx, p01 - p00, p00), fmaf(fx, p01 - p00, p00));
                    };
                    cr *= bl(a00.x, a01.x, a10.x, a11.x);
                    cg *= bl(a00.y, a01.y, a10.y, a11.y);
                    cb *= bl(a00.z, a01.z, a10.z, a11.z);
                    a *= bl(a00.w, a01.w, a10.w, a11.w);
                }
            }
            // a9: Phong with a headlight (l.10-11; R-11); zero gradient -> ambient
            bool lit_done = false;
            if constexpr (SHADE && EXT) {
                if (args.lights.n > 0) {  // several directional lights (R-30)
                    const float gx = gu * gs[0], gy = gv * gs[1], gz = gw * gs[2];
                    const float n2 = fmaf(gx, gx, fmaf(gy, gy, gz * gz));
                    const bool zero = n2 <= args.eps2;
                    const float inv = rsqrt_normal(fmaxf(n2, 1e-37f));
                    const float ndv = fmaf(gx, dx, fmaf(gy, dy, gz * dz)) * inv;   // N . V, V = -d
                    float dif = 0.f, spe = 0.f;
                    for (int l = 0; l < args.lights.n; ++l) {
                        const float* L = args.lights.dir[l];
                        const float ndl = -fmaf(gx, L[0], fmaf(gy, L[1], gz * L[2])) * inv;  // N . L
                        const float ldv = -fmaf(L[0], dx, fmaf(L[1], dy, L[2] * dz));         // L . V
                        const float rv = fmaxf(fmaf(2.f * ndl, ndv, -ldv), 0.f);              // R . V
                        float sp = args.shin == 0.f ? 1.f : pow_spec(rv, args.shin);
                        dif = fmaf(args.lights.intensity[l], fmaxf(ndl, 0.f), dif);
                        spe = fmaf(args.lights.intensity[l], ndl > 0.f ? sp : 0.f, spe);
                    }
                    const float lit = zero ? args.ka : fmaf(args.kd, dif, args.ka);
                    const float add = zero ? 0.f : args.ks * spe;
                    cr = __saturatef(fmaf(cr, lit, add));
                    cg = __saturatef(fmaf(cg, lit, add));
                    cb = __saturatef(fmaf(cb, lit, add));
                    lit_done = true;
                }
            }
            if (SHADE && !lit_done) {
                const float gx = gu * gs[0], gy = gv * gs[1], gz = gw * gs[2];
                const float n2 = fmaf(gx, gx, fmaf(gy, gy, gz * gz));
                const bool zero = n2 <= args.eps2;
                const float ndl = fmaf(gx, dx, fmaf(gy, dy, gz * dz)) * rsqrt_normal(fmaxf(n2, 1e-37f));
                const float dif = fmaxf(ndl, 0.f);
                const float rv = fmaxf(fmaf(2.f * ndl, ndl, -1.f), 0.f);
                float spe = pow_spec(rv, args.shin);                  // rv = 0 -> 0 (shin > 0)
                if (args.shin == 0.f) spe = 1.f;                       // 0^0 = 1, as pow()
                spe = ndl > 0.f ? spe : 0.f;
                const float lit = zero ? args.ka : fmaf(args.kd, dif, args.ka);
                const float add = zero ? 0.f : args.ks * spe;
                cr = __saturatef(fmaf(cr, lit, add));
                cg = __saturatef(fmaf(cg, lit, add));
                cb = __saturatef(fmaf(cb, lit, add));
            }
            // a10: front-to-back compositing (l.13)
            const float wgt = comp_on ? (1.f - A) * a : 0.f;   // MFA_FLAT_LOOP: finished lanes add nothing
            C0 = fmaf(wgt, cr, C0);
            C1 = fmaf(wgt, cg, C1);
            C2 = fmaf(wgt, cb, C2);
            A += wgt;
#if MFA_ORDER == 1
            order_dep = A;
#endif
        };

        // curvature TF (EXT): principal curvatures of the MFA's isosurface at the
        // sample from its gradient and Hessian (t-space, scaled by the MFA's gs)
        auto curv_query = [&](const int (&s)[3], const float (&t)[3], const float (&gsm)[3], float& k1, float& k2) {
            float Nu[P + 1], Du[P + 1], Eu[P + 1], Nv[P + 1], Dv[P + 1], Ev[P + 1], Nw[P + 1], Dw[P + 1], Ew[P + 1];
            constexpr int BL = BEZ ? kBezier : kQuads;
            basis3<P, BL, UNI>(args.ax[0], s[0], t[0], Nu, Du, Eu);
            basis3<P, BL, UNI>(args.ax[1], s[1], t[1], Nv, Dv, Ev);
            basis3<P, BL, UNI>(args.ax[2], s[2], t[2], Nw, Dw, Ew);
            float o[10];
#pragma unroll
            for (int q = 0; q < 10; ++q) o[q] = 0.f;
            if constexpr (CACHE) {
                fetch(s);
#pragma unroll
                for (int c = 0; c <= P; ++c) contract_vgh_slab<P>(nb[c], Nu, Du, Eu, Nv, Dv, Ev, Nw[c], Dw[c], Ew[c], o);
            } else {
#pragma unroll
                for (int c = 0; c <= P; ++c) {
                    float r[P + 1][P + 1];
                    if constexpr (BEZ)
                        load_bslab<P, SEC>(bslab_ptr<P, SEC>(bez_block<P, SEC>(args.Q, args.bg, s[0], s[1], s[2]), c), r);
                    else
                        load_slab<P>(args.Q + brick_entry<P>(args.g, s[0], s[1], s[2]) + c * Brick<P>::SLAB, r);
                    contract_vgh_slab<P>(r, Nu, Du, Eu, Nv, Dv, Ev, Nw[c], Dw[c], Ew[c], o);
                }
            }
            const float g[3] = {o[1] * gsm[0], o[2] * gsm[1], o[3] * gsm[2]};
            const float h[6] = {o[4] * gsm[0] * gsm[0], o[5] * gsm[1] * gsm[1], o[6] * gsm[2] * gsm[2],
                                o[7] * gsm[0] * gsm[1], o[8] * gsm[0] * gsm[2], o[9] * gsm[1] * gsm[2]};
            if (fmaf(g[0], g[0], fmaf(g[1], g[1], g[2] * g[2])) <= args.eps2) {   // no isosurface (R-31)
                k1 = k2 = 0.f;
            } else {
                curvatures(g, h, k1, k2);
            }
        };

        // NEXT-2 (EXT instantiations): the sample takes its value and/or its
        // gradient from the analytic field at the same parameter point
        auto sample_field = [&](const int (&s)[3], const float (&t)[3], float& v, float& g0, float& g1, float& g2,
                                float (&gsx)[3]) {
            if (!(args.fld.vsrc && args.fld.gsrc)) {
                fetch(s);
                query(s, t, v, g0, g1, g2);
            }
            double uu[3], fa[4];
#pragma unroll
            for (int i = 0; i < 3; ++i) uu[i] = fmin(fmax((double)F[i] * args.fld.fx_scale[i], 0.0), 1.0);
            field_eval(args.fld, uu, fa);
            if (args.fld.vsrc) v = (float)fa[0];
            if (args.fld.gsrc) {
                g0 = (float)fa[1];
                g1 = (float)fa[2];
                g2 = (float)fa[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) gsx[i] = args.fld.invL[i];
            }
        };

        // two-stage pipeline: iteration k queries sample k+1 while it shades
        // and composites sample k; the ERT test (l.14-15; R-13) follows.
        float val = 0.f, gu = 0.f, gv = 0.f, gw = 0.f, gs[3] = {0.f, 0.f, 0.f};
        bool tr_cur = false;   // SHADE == 3: the sample being shaded lies in a transparent macro block
        float ck1 = 0.f, ck2 = 0.f;   // curvatures of the sample being shaded (EXT curvature TF)
        if (live) {
            int s[3];
            float t[3];
            locate(s, t, gs, std::true_type{});
            if constexpr (EXT) {
                if (args.curv.n > 0) curv_query(s, t, gs, ck1, ck2);
                sample_field(s, t, val, gu, gv, gw, gs);
            } else {
                tr_cur = transparent(s);
                if (!tr_cur) {
                    fetch(s);
                    query(s, t, val, gu, gv, gw);
                }
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) F[i] += (!kFlat || K > 1) ? DF[i] : 0;
        }
#if MFA_FLAT_LOOP
        // branch-free body: every lane runs it; a finished lane's sample
        // position is frozen (no reloads) and its compositing weight is 0.
        // Iteration k composites sample k and queries sample min(k+1, K-1).
        auto flat_loop = [&](auto multi_tag) {
            // MFA_MULTI_DEFER == 2: the block load issued from the single-step span
            // triple before the span records arrive (refetched in the rare fixup)
            constexpr bool kFetchEarly = MFA_MULTI_DEFER >= 2 && !UNI;
            // MFA_MULTI_DEFER == 3: and the previous sample shaded before the vote
            constexpr bool kShadeEarly = MFA_MULTI_DEFER == 3 && SHADE != 3 && !UNI;
#if MFA_EARLY_LOAD
            constexpr bool kEarly = BEZ && SHADE != 3;
            constexpr bool kEarlyNU = kEarly && !UNI;
            static_assert(!kEarlyNU || (MFA_NU_SHIFTCMP && MFA_NU_UCMP), "the early load predicts the UCMP rule");
            int dn[3] = {0, 0, 0};   // kEarlyNU: span offsets of the next sample, computed one iteration ahead
            if constexpr (kEarlyNU) {
#pragma unroll
                for (int i = 0; i < 3; ++i) dn[i] = nu_offset(args.ax[i], F[i], nu[i]);
            }
#endif
            while (__any_sync(0xffffffffu, live)) {
                int s[3];
                float t[3], gs1[3];
#if MFA_DIAG_MULTICOUNT
                int s_before[3];
                if constexpr (!UNI) {
#pragma unroll
                    for (int i = 0; i < 3; ++i) s_before[i] = nu[i].s;
                }
#endif
#if MFA_MULTI_DEFER
                if constexpr (!UNI && decltype(multi_tag)::value) {
                    // the straight-line single-crossing tracker, and the rare step that
                    // crossed more than one span (0.2 % of C5's lane-samples, 1.8 % of its
                    // warp-iterations) fixed behind one warp-uniform vote instead of a
                    // divergent search branch per axis in the common path
#pragma unroll
                    for (int i = 0; i < 3; ++i) nu_cross(args.ax[i], F[i], nu[i]);
                    if constexpr (kFetchEarly) {   // the block of the single-step span triple, before the records arrive
#pragma unroll
                        for (int i = 0; i < 3; ++i) s[i] = nu[i].s;
                        if (!transparent(s)) fetch(s);   // (SHADE == 3: transparent blocks are not fetched)
                    }
                    if constexpr (kShadeEarly) {   // the previous sample's shading overlaps the record loads
                        comp_on = live && !tr_cur;
                        shade_composite(val, gu, gv, gw, gs, 0.f, 0.f);
                    }
                    int d[3];
                    bool mh = false;
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        d[i] = nu_offset(args.ax[i], F[i], nu[i]);
                        mh |= (unsigned)d[i] >= (unsigned)nu[i].wsh;
                    }
                    if (__any_sync(0xffffffffu, mh)) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            if ((unsigned)d[i] >= (unsigned)nu[i].wsh) {
                                nu_search(args.ax[i], F[i], nu[i]);
                                d[i] = nu_offset(args.ax[i], F[i], nu[i]);
                            }
                        }
                        if constexpr (kFetchEarly) {   // lanes whose span triple moved refetch
                            int s2[3];
#pragma unroll
                            for (int i = 0; i < 3; ++i) s2[i] = nu[i].s;
                            if (!transparent(s2)) fetch(s2);
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        t[i] = nu_t(args.ax[i], d[i], nu[i]);
                        s[i] = nu[i].s;
                        gs1[i] = nu_gscale(args.ax[i], nu[i]);
                    }
                } else
#endif
#if MFA_EARLY_LOAD
                if constexpr (kEarlyNU) {
                    constexpr bool MULTI = decltype(multi_tag)::value;
#pragma unroll
                    for (int i = 0; i < 3; ++i) nu_cross_d(args.ax[i], dn[i], nu[i]);
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        t[i] = nu_finish<MULTI>(args.ax[i], F[i], nu[i]);
                        s[i] = nu[i].s;
                        gs1[i] = nu_gscale(args.ax[i], nu[i]);
                    }
                } else
#endif
                locate(s, t, gs1, multi_tag);
                const bool tr_next = transparent(s);
#if MFA_DIAG_MULTICOUNT
                if constexpr (!UNI) {
                    bool mh = false;
#pragma unroll
                    for (int i = 0; i < 3; ++i) mh |= abs(s[i] - s_before[i]) > 1;
                    mh = mh && live;
                    dm_lane += mh ? 1 : 0;
                    if (__any_sync(0xffffffffu, mh) && lane == 0) ++dm_warp;
                    if (lane == 0) ++dm_iters;
                }
#endif
#if MFA_BULK_PF
                if constexpr (kPF) {
                    const int e = (s[2] * args.bg.S1 + s[1]) * args.bg.S0 + s[0];
                    if (!tr_next && e != nb_key) {
                        if (pf_pending && pf_key == e) {   // prefetched one iteration ago
                            pf_wait();
                            const float4* sl = reinterpret_cast<const float4*>(&s_pf[threadIdx.x][0]);
#pragma unroll
                            for (int q = 0; q < 16; ++q) {
                                const float4 x = sl[q];
                                nb[q >> 2][q & 3][0] = x.x;
                                nb[q >> 2][q & 3][1] = x.y;
                                nb[q >> 2][q & 3][2] = x.z;
                                nb[q >> 2][q & 3][3] = x.w;
                            }
                        } else {
                            load_bblock<P>(bez_block_at<P>(args.Q, args.bg, e), nb);
                        }
                        nb_key = e;
                    }
                    if (live) {   // predict the block of the sample after next (one crossing per axis)
                        int s2[3];
#pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            const int d2 = nu_offset(args.ax[i], F[i] + DF[i], nu[i]);
                            s2[i] = s[i] + (d2 >= nu[i].wsh ? 1 : 0) - (d2 < 0 && s[i] > 0 ? 1 : 0);
                        }
                        const int e2 = (s2[2] * args.bg.S1 + s2[1]) * args.bg.S0 + s2[0];
                        if (e2 != nb_key && !(pf_pending && pf_key == e2)) {
                            if (pf_pending) pf_wait();   // the slot is reused
                            const unsigned mb = (unsigned)__cvta_generic_to_shared(&s_mbar[threadIdx.x]);
                            const unsigned dst = (unsigned)__cvta_generic_to_shared(&s_pf[threadIdx.x][0]);
                            const float* src = reinterpret_cast<const float*>(bez_block_at<P>(args.Q, args.bg, e2));
                            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(256)
                                         : "memory");
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                                "l"(src), "r"(256), "r"(mb)
                                : "memory");
                            pf_key = e2;
                            pf_pending = true;
                        }
                    }
                } else
#endif
                if (!kFetchEarly || UNI || !decltype(multi_tag)::value) {
                    if (!tr_next) fetch(s);
                }
#if MFA_PREFETCH_NEXT
                if constexpr (LAYOUT == kBezier && !UNI) {   // linear blocks only
                    // predict the span triple of the sample after this one from the
                    // current span bounds (one crossing per axis at most) and pull
                    // its block towards the SM a whole iteration before its load
                    int s2[3];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
#if MFA_NU_SHIFTCMP
                        const int d2 = nu_offset(args.ax[i], F[i] + DF[i], nu[i]);
                        s2[i] = s[i] + (d2 >= nu[i].wsh ? 1 : 0) - (d2 < 0 && s[i] > 0 ? 1 : 0);
#else
                        const long long F2 = F[i] + DF[i];
                        s2[i] = s[i] + (F2 >= nu[i].hi ? 1 : 0) - (F2 < nu[i].lo && s[i] > 0 ? 1 : 0);
#endif
                    }
                    const int e2 = (s2[2] * args.bg.S1 + s2[1]) * args.bg.S0 + s2[0];
                    if (e2 != nb_key && live) {
                        const char* q = reinterpret_cast<const char*>(bez_block_at<P>(args.Q, args.bg, e2));
#if MFA_PREFETCH_NEXT == 2
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(q + 128));
#else
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(q + 128));
#endif
                    }
                }
#endif
                if (!kShadeEarly || UNI || !decltype(multi_tag)::value) {
                    comp_on = live && !tr_cur;   // a transparent sample composites with weight 0
                    shade_composite(val, gu, gv, gw, gs, 0.f, 0.f);
                }
#if MFA_ORDER
                t[0] = fmaf(order_dep, 0.f, t[0]);   // exact: t[0] + 0 (A is finite)
#endif
                if (!tr_next) query(s, t, val, gu, gv, gw);
                tr_cur = tr_next;
                const bool adv = live && k + 2 < K;
#pragma unroll
                for (int i = 0; i < 3; ++i) gs[i] = gs1[i];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
#if MFA_PRED_ADV
                    if (adv) F[i] += DF[i];   // predicated 64-bit add
#else
                    F[i] += adv ? DF[i] : 0;
#endif
                }
                k += live ? 1 : 0;
                live = live && !(A > args.o_max) && k < K;
#if MFA_EARLY_LOAD
                // the block of the NEXT iteration's sample, issued as soon as this
                // iteration's contraction has read the cached one: its span triple
                // follows from the span state and the advanced position by the
                // same single-crossing rule nu_cross applies (exact unless a step
                // crosses several spans, which the next fetch() then corrects), so
                // the load latency overlaps the next locate and shading too.
                if constexpr (kEarly) {
                    int s2[3];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        if constexpr (UNI) {
                            float t2;
                            uni_span_fx(F[i], args.ax[i].nsp, s2[i], t2);
                        } else {
                            dn[i] = nu_offset(args.ax[i], F[i], nu[i]);   // reused by the next nu_cross_d
                            s2[i] = (unsigned)dn[i] >= (unsigned)nu[i].wsh ? max(nu[i].s + ((dn[i] >> 31) | 1), 0)
                                                                           : nu[i].s;
                        }
                    }
                    if (live) fetch(s2);
                }
#endif
            }
        };
        if constexpr (kFlat) {
            if (!MFA_DIAG_NOMULTI && !UNI && (args.ax[0].multi | args.ax[1].multi | args.ax[2].multi))   // launch-uniform
                flat_loop(std::true_type{});
            else
                flat_loop(std::false_type{});
        }
#endif
        while (!kFlat && __any_sync(0xffffffffu, live)) {
#if MFA_LANE_STATS   // diagnostic: warp-iterations x 32 and live lanes (samples[1], samples[2])
            if (lane == 0) {
                lane_slots += 32;
                lane_live += __popc(__ballot_sync(0xffffffffu, live));
            } else {
                __ballot_sync(0xffffffffu, live);
            }
#endif
            if (live) {
                if (k + 1 < K) {
                    int s[3];
                    float t[3], gs1[3];
                    locate(s, t, gs1, std::true_type{});
                    float val1 = 0.f, gu1 = 0.f, gv1 = 0.f, gw1 = 0.f;
                    if constexpr (EXT) {
                        float nk1 = 0.f, nk2 = 0.f;
                        if (args.curv.n > 0) curv_query(s, t, gs1, nk1, nk2);
                        shade_composite(val, gu, gv, gw, gs, ck1, ck2);
                        sample_field(s, t, val1, gu1, gv1, gw1, gs1);
                        ck1 = nk1;
                        ck2 = nk2;
                    } else {
                        fetch(s);
                        shade_composite(val, gu, gv, gw, gs, 0.f, 0.f);
#if MFA_ORDER
                        t[0] = fmaf(order_dep, 0.f, t[0]);   // exact: t[0] + 0 (A is finite)
#endif
                        query(s, t, val1, gu1, gv1, gw1);
                    }
                    val = val1;
                    gu = gu1;
                    gv = gv1;
                    gw = gw1;
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        gs[i] = gs1[i];
                        F[i] += DF[i];
                    }
                } else {
                    shade_composite(val, gu, gv, gw, gs, ck1, ck2);
                }
                ++k;
                live = !(A > args.o_max) && k < K;
            }
        }
        // ---- a11: pixel write ---------------------------------------------
        if (valid) {
            int64_t idx;
            if (args.tiles && !args.tile_scatter)
                idx = tile_id * (MFA_TILE * MFA_TILE) + ly * MFA_TILE + lx;
            else   // full frame, or a tile list stored straight to its image position
                   // (possibly a peer GPU's image: the multi-GPU direct-store path)
                idx = ((int64_t)(args.view_base + view) * args.H + py) * args.W + px;
            if (args.out_fp16) {
                __half2* o2 = reinterpret_cast<__half2*>(args.out) + 2 * idx;
                o2[0] = __floats2half2_rn(C0, C1);
                o2[1] = __floats2half2_rn(C2, A);
            } else {
                reinterpret_cast<float4*>(args.out)[idx] = make_float4(C0, C1, C2, A);
            }
        }
        my_samples += (unsigned)k;
    }
#if MFA_BULK_PF
    if (pf_pending) pf_wait();   // no bulk copy may still be writing this CTA's shared memory at exit
#endif
    if (args.samples) {   // 64-bit warp sum (a warp may composite more than 2^32 samples)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) my_samples += __shfl_xor_sync(0xffffffffu, my_samples, o);
        if (lane == 0 && my_samples) atomicAdd(args.samples, my_samples);
#if MFA_DIAG_MULTICOUNT
        for (int o = 16; o > 0; o >>= 1) dm_lane += __shfl_xor_sync(0xffffffffu, dm_lane, o);
        if (lane == 0) {
            atomicAdd(args.samples + 1, dm_lane);
            atomicAdd(args.samples + 2, dm_warp);
            atomicAdd(args.samples + 3, dm_iters);
        }
#endif
#if MFA_LANE_STATS
        if (lane == 0) {
            atomicAdd(args.samples + 1, lane_slots);
            atomicAdd(args.samples + 2, lane_live);
        }
#endif
    }
}

template <int P, int LAYOUT, bool UNI, int SHADE, bool EXT>
static cudaError_t launch_render_t(const RenderArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(float4) * a.tf_n;
    auto kern = render_kernel<P, LAYOUT, UNI, SHADE, EXT>;
    constexpr int kThreads = RenderShape<P, LAYOUT>::THREADS;
    // launch shape per (device, TF size): the carveout and the occupancy query
    // cost several driver calls, which dominated a tiny frame's launch (C1:
    // 64 x 64 pixels); cached here, computed on first use
    struct Shape {
        int sms = 0, occ = 0;
        size_t smem = (size_t)-1;
    };
    static Shape cache[64];
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    Shape sh;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 64) sh = cache[dev];
    }
    if (sh.smem != smem) {
        sh.smem = smem;
        sh.sms = 148;
        cudaDeviceGetAttribute(&sh.sms, cudaDevAttrMultiProcessorCount, dev);
        // shared-memory carveout: enough for MINB resident CTAs but at least
        // MFA_CARVE_FLOOR (8 %), the rest of the unified 256 KB is L1 (the block
        // caches live there).  The driver's default (more shared memory) measured
        // C5 -15%, C4 -37%; a 25 % floor: C5 -1 %, C4 -1.4 %
        int pct = MFA_CARVEOUT;
        if (pct < 0) {
            cudaFuncAttributes fa;
            int max_sm = 233472;
            cudaDeviceGetAttribute(&max_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
            if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && max_sm > 0) {
                const size_t need = (fa.sharedSizeBytes + smem + 1024) * RenderShape<P, LAYOUT>::MINB;
                pct = (int)std::min<size_t>(100, std::max<size_t>(MFA_CARVE_FLOOR, (100 * need + max_sm - 1) / max_sm + 2));
            }
        }
        if (pct >= 0) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
        sh.occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sh.occ, kern, kThreads, smem);
        if (sh.occ < 1) sh.occ = 1;
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 64) cache[dev] = sh;
    }
    int64_t grid = (int64_t)sh.sms * sh.occ;
    const int64_t need = (a.n_units + kThreads / 32 - 1) / (kThreads / 32);
    if (grid > need) grid = need > 0 ? need : 1;
    kern<<<(unsigned)grid, kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

template <int P, int LAYOUT, bool EXT>
static cudaError_t dispatch_render_l(const RenderArgs& a, bool uni, int shade, cudaStream_t st) {
    constexpr bool kSkip = !EXT && RenderShape<P, LAYOUT>::CACHE;   // SHADE = 2 is built for the hot path only
    constexpr bool kSkipBlk = kSkip && is_bez(LAYOUT);               // SHADE = 3 needs the macro-block bounds
    if (shade == 2 && !kSkip) shade = 1;
    if (shade == 3 && !(kSkipBlk && a.tbits)) shade = 1;
    if (uni) {
        if (shade == 0) return launch_render_t<P, LAYOUT, true, 0, EXT>(a, st);
        if constexpr (kSkip)
            if (shade == 2) return launch_render_t<P, LAYOUT, true, 2, EXT>(a, st);
        if constexpr (kSkipBlk)
            if (shade == 3) return launch_render_t<P, LAYOUT, true, 3, EXT>(a, st);
        return launch_render_t<P, LAYOUT, true, 1, EXT>(a, st);
    }
    if (shade == 0) return launch_render_t<P, LAYOUT, false, 0, EXT>(a, st);
    if constexpr (kSkip)
        if (shade == 2) return launch_render_t<P, LAYOUT, false, 2, EXT>(a, st);
    if constexpr (kSkipBlk)
        if (shade == 3) return launch_render_t<P, LAYOUT, false, 3, EXT>(a, st);
    return launch_render_t<P, LAYOUT, false, 1, EXT>(a, st);
}

template <int P, bool EXT>
static cudaError_t dispatch_render(const RenderArgs& a, int layout, bool uni, int shade, cudaStream_t st) {
    if constexpr (P <= 3) {
        if (layout == kBezier) return dispatch_render_l<P, kBezier, EXT>(a, uni, shade, st);
        if constexpr (P == 3)
            if (layout == kBezierG) return dispatch_render_l<P, kBezierG, EXT>(a, uni, shade, st);
        if (layout == kBricks) return dispatch_render_l<P, kBricks, EXT>(a, uni, shade, st);
    }
    return dispatch_render_l<P, kQuads, EXT>(a, uni, shade, st);
}

// defined in render.cu (the hot path) and truth.cu (analytic field, several lights)
cudaError_t dispatch_render_main(const RenderArgs& a, int p, int layout, bool uni, int shade, cudaStream_t st);
cudaError_t dispatch_render_ext(const RenderArgs& a, int p, int layout, bool uni, int shade, cudaStream_t st);

}  // namespace mfa
