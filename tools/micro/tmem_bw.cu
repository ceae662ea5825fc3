// TMEM read-throughput probe: one CTA per SM, W warps, each warp loops over
// tcgen05.ld.32x32b.x32 (4 KB per warp instruction) of its lane quadrant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

template <int DEPTH>
__global__ void probe(int iters, uint32_t* out) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = base + (((warp & 3) * 32u) << 16);
    uint32_t acc = 0;
    const uint32_t col0 = (warp >> 2) * 64;
    for (int i = 0; i < iters; ++i) {
        uint32_t r[DEPTH][32];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) ld32(t + ((col0 + (i * DEPTH + d) * 32) & 511), r[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int d = 0; d < DEPTH; ++d)
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += r[d][j];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, sizeof(uint32_t) * sms * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4000;
    for (int warps : {4, 8, 12, 16}) {
        for (int depth : {1, 2}) {
            auto k = depth == 1 ? probe<1> : probe<2>;
            k<<<sms, warps * 32>>>(10, out);
            cudaEventRecord(a);
            k<<<sms, warps * 32>>>(iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = double(sms) * warps * iters * depth * 4096.0;
            int clk = 0;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            printf("warps %2d depth %d: %.3f ms  %.1f TB/s  %.1f B/clk/SM (at %d MHz)  err=%s\n", warps, depth, ms,
                   bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
