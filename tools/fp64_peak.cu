// fp64_peak.cu -- measure the B200's FP64 SIMT (DFMA) and FP64 tensor (DMMA,
// mma.sync m8n8k4) throughput, which MEASURED_PEAKS.json does not record.
// Prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fma_rn(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double d[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { d[i][0] = 0; d[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void ffma_kernel(float *out, int iters, float a, float b)
{
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fmaf_rn(x[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[0] = s;
}

__global__ void tf32_kernel(float *out, int iters)
{
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
    float d[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
    if (s == 12345.678f) out[0] = s;
}

__global__ void bf16_kernel(float *out, int iters)
{
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
    float d[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
    if (s == 12345.678f) out[0] = s;
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *dout;
    cudaMalloc(&dout, 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    float ms;
    double best_dfma = 0, best_dmma = 0, best_ffma = 0, best_tf32 = 0, best_bf16 = 0;
    for (int rep = 0; rep < 5; ++rep) {
        int blocks = nsm * 4, threads = 512;
        cudaEventRecord(a);
        dfma_kernel<<<blocks, threads>>>(dout, iters, 0.999999, 1e-7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 8 * iters * (double)blocks * threads;
        if (fl / (ms * 1e-3) > best_dfma) best_dfma = fl / (ms * 1e-3);

        cudaEventRecord(a);
        dmma_kernel<<<blocks, threads>>>(dout, iters / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl = 2.0 * 256 * 8 * (iters / 4) * (double)blocks * (threads / 32);
        if (fl / (ms * 1e-3) > best_dmma) best_dmma = fl / (ms * 1e-3);

        cudaEventRecord(a);
        ffma_kernel<<<blocks, threads>>>((float *)dout, iters, 0.999999f, 1e-7f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl = 2.0 * 8 * iters * (double)blocks * threads;
        if (fl / (ms * 1e-3) > best_ffma) best_ffma = fl / (ms * 1e-3);

        cudaEventRecord(a);
        tf32_kernel<<<blocks, threads>>>((float *)dout, iters / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl = 2.0 * 16 * 8 * 8 * 8 * (iters / 4) * (double)blocks * (threads / 32);
        if (fl / (ms * 1e-3) > best_tf32) best_tf32 = fl / (ms * 1e-3);

        cudaEventRecord(a);
        bf16_kernel<<<blocks, threads>>>((float *)dout, iters / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl = 2.0 * 16 * 8 * 16 * 8 * (iters / 4) * (double)blocks * (threads / 32);
        if (fl / (ms * 1e-3) > best_bf16) best_bf16 = fl / (ms * 1e-3);
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"ffma_tflops\": %.3f, "
           "\"mma_sync_tf32_tflops\": %.3f, \"mma_sync_bf16_tflops\": %.3f, \"err\": \"%s\"}\n",
           nsm, best_dfma * 1e-12, best_dmma * 1e-12, best_ffma * 1e-12, best_tf32 * 1e-12, best_bf16 * 1e-12,
           cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
