// probe.cu -- measured FP32 FFMA peak of this GPU (the roofline denominator
// for the fp32-bound screen kernels; MEASURED_PEAKS.json carries HBM and bf16
// tensor peaks only).  Register-operand FFMAs, 16 independent chains per
// thread, 8 CTAs of 256 threads per SM, timed with CUDA events.
#include "kernels.cuh"

namespace {

__global__ void __launch_bounds__(256) ffma_probe_kernel(const float* in, float* out, int iters) {
    float a[16];
    const float x = in[threadIdx.x & 31], y = in[32 + (threadIdx.x & 31)];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = in[64 + j] + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], x, y);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j];
    if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

}  // namespace

extern "C" int pqg_fp32_probe(pqg_ctx* ctx, double* tflops) {
    try {
        pqg::Scope sc(ctx);
        float* buf = pqg::scratch<float>(ctx, 128);
        PQG_CUDA(cudaMemsetAsync(buf, 0, 128 * sizeof(float), ctx->stream));
        const int iters = 1 << 14;
        const unsigned blocks = ctx->num_sms * 8;
        cudaEvent_t a, b;
        PQG_CUDA(cudaEventCreate(&a));
        PQG_CUDA(cudaEventCreate(&b));
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            PQG_CUDA(cudaEventRecord(a, ctx->stream));
            pqg::launch(ctx, "fp32_probe", ffma_probe_kernel, dim3(blocks), dim3(256), 0,
                        (const float*)buf, buf + 100, iters);
            PQG_CUDA(cudaEventRecord(b, ctx->stream));
            PQG_CUDA(cudaEventSynchronize(b));
            float ms = 0.f;
            PQG_CUDA(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        const double flops = 2.0 * 16.0 * iters * double(blocks) * 256.0;
        *tflops = flops / (best * 1e-3) / 1e12;
        return PQG_OK;
    } catch (const pqg::Error& e) {
        return e.code;
    }
}
