// k4_ceiling.cu -- compute ceiling of K4's fp64 T-tile item (Y = U_a^T X,
// W = Y U_c, both 64^3 on DMMA m8n8k4 from shared memory) with no global
// traffic: 3 CTAs x 256 threads per SM, each CTA repeating the item on its
// own shared-memory operands.  Variants:
//   0: as k_block_apply_f64x3 (k-chunked products, a barrier per 16-k chunk)
//   1: unchunked products (one barrier between the two GEMMs)
// Prints TF/s per variant; compare with the DMMA peak (tools/fp64_peak.cu).
// Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2211_03339_b200/csrc tools/k4_ceiling.cu -o tools/k4_ceiling
#include <cstdio>
#include "mpj_device.cuh"
#include "mpj_block.cuh"
using namespace mpj;
using namespace mpj::blk;

template <int VAR>
__global__ void __launch_bounds__(NT, 3) k4c(double *out, int items)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int LD = Lay<double>::LD;
    double *xb = (double *)smem_raw, *ub = xb + TW * LD;
    for (int e = threadIdx.x; e < TW * LD; e += NT) {
        xb[e] = 1e-3 * ((e * 7 + blockIdx.x) % 13);
        ub[e] = 1e-3 * ((e * 5 + blockIdx.x) % 11);
    }
    __syncthreads();
    double s = 0.0;
    for (int it = 0; it < items; ++it) {
        Acc<double> acc;
        if (VAR == 0) {
            tile_mm_chunked<true>(ub, xb, acc, [&](int) { __syncthreads(); });
            __syncthreads();
            acc.each([&](int i, int j, double v) { xb[i + j * LD] = v * 1e-3; });
            tile_mm_chunked<false>(xb, ub, acc, [&](int) { __syncthreads(); });
        } else {
            acc.zero();
            tile_mm_acc<true>(ub, xb, acc);
            __syncthreads();
            acc.each([&](int i, int j, double v) { xb[i + j * LD] = v * 1e-3; });
            __syncthreads();
            acc.zero();
            tile_mm_acc<false>(xb, ub, acc);
        }
        __syncthreads();
        acc.each([&](int, int, double v) { s += v; });
    }
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int VAR>
static void run(int items, int nbuf = 2)
{
    const int smem = nbuf * TW * Lay<double>::LD * 8;
    cudaFuncSetAttribute(k4c<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4c<VAR>, NT, smem);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm * per_sm;
    double *out;
    cudaMalloc(&out, 4096 * 8);
    k4c<VAR><<<grid, NT, smem>>>(out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k4c<VAR><<<grid, NT, smem>>>(out, items);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double flop = (double)grid * items * 2 * 2.0 * TW * TW * TW;
    printf("variant %d: %d CTAs/SM, grid %d, %.3f ms, %.2f TF/s (%s)\n", VAR, per_sm, grid, ms, flop / ms * 1e-9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main()
{
    run<0>(2000);
    run<1>(2000);
    run<0>(2000);
    run<1>(2000);
    run<0>(2000, 3);   // 2 CTAs / SM
    run<1>(2000, 3);
    run<0>(2000, 5);   // 1 CTA / SM
    run<1>(2000, 5);
    return 0;
}
