// Microbenchmark: L1 data-pipe wavefronts of 256-bit / 128-bit global loads
// under different lane-address patterns (which lanes share a 128-byte line or
// a 32-byte sector, how many lanes are active).  Run under ncu:
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,
//       l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum ./ldg_wavefronts
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const float* p, float (&r)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld128(const float* p, float (&r)[4]) {
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "l"(p));
}

// pattern: byte offset of lane l = (l / share) * stride + (l % share) * inner; lanes >= active idle
template <int W>
__global__ void k(const float* __restrict__ base, float* out, int active, int share, int stride, int inner, int iters) {
    const int l = threadIdx.x & 31;
    float acc = 0.f;
    if (l < active) {
        const char* p = reinterpret_cast<const char*>(base) + (size_t)(l / share) * stride + (size_t)(l % share) * inner;
        for (int i = 0; i < iters; ++i) {
            const float* q = reinterpret_cast<const float*>(p + (size_t)(i & 7) * 4096);
            if (W == 256) {
                float r[8];
                ld256(q, r);
                acc += ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            } else {
                float r[4];
                ld128(q, r);
                acc += (r[0] + r[1]) + (r[2] + r[3]);
            }
        }
    }
    if (acc == 12345.f) out[threadIdx.x] = acc;
}

int main() {
    float* d;
    cudaMalloc(&d, 64 << 20);
    cudaMemset(d, 0, 64 << 20);
    float* o;
    cudaMalloc(&o, 4096);
    struct P { int w, active, share, stride, inner; const char* name; };
    P ps[] = {
        {256, 32, 1, 128, 0, "256: 32 lanes, distinct lines"},
        {256, 32, 32, 0, 0, "256: 32 lanes, one sector"},
        {256, 32, 4, 128, 32, "256: 32 lanes, 4 lanes per line (distinct sectors)"},
        {256, 32, 2, 128, 32, "256: 32 lanes, 2 lanes per line"},
        {256, 10, 1, 128, 0, "256: 10 lanes, distinct lines"},
        {256, 10, 2, 128, 32, "256: 10 lanes, 2 per line"},
        {256, 10, 2, 128, 0, "256: 10 lanes, 2 per sector"},
        {256, 1, 1, 128, 0, "256: 1 lane"},
        {128, 32, 1, 128, 0, "128: 32 lanes, distinct lines"},
        {128, 32, 8, 128, 16, "128: 32 lanes, 8 lanes per line"},
        {128, 10, 1, 128, 0, "128: 10 lanes, distinct lines"},
    };
    for (auto& p : ps) {
        printf("pattern %s\n", p.name);
        fflush(stdout);
        if (p.w == 256) k<256><<<1, 32>>>(d, o, p.active, p.share, p.stride, p.inner, 1000);
        else k<128><<<1, 32>>>(d, o, p.active, p.share, p.stride, p.inner, 1000);
        cudaDeviceSynchronize();
    }
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
