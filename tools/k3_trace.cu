// k3_trace.cu -- per-round timeline of K3's inner rounds (inner_rounds_wide)
// on one CTA: clock64 when the parameter warp finishes rot_params (event 0),
// when the last update warp finishes its work (event 1, max over warps) and
// after the round's barrier (event 2).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -I paper_2211_03339_b200/csrc tools/k3_trace.cu -o tools/k3_trace
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
__device__ unsigned long long g_tr[3][64];
__device__ __forceinline__ void k3_trace(int ev, int s)
{
    if (blockIdx.x != 0) return;
    const unsigned long long t = clock64();
    if (ev == 0) { if ((threadIdx.x & 31) == 0) g_tr[0][s] = t; }
    else if (ev == 1) { if ((threadIdx.x & 31) == 0) atomicMax(&g_tr[1][s], t); }
    else if (threadIdx.x == 0) g_tr[2][s] = t;
}
#define MPJ_K3_TRACE(event, round) k3_trace(event, round)
#include "mpj_device.cuh"
#include "mpj_block.cuh"
using namespace mpj;
using namespace mpj::blk;

template <typename R>
__global__ void __launch_bounds__(NTW) k3(const R *Din, R *Uout, R nu)
{
    constexpr int LD = LayK<R>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *D0 = (R *)smem_raw, *D1 = D0 + TW * LD, *U = D1 + TW * LD;
    __shared__ unsigned nrot;
    __shared__ WideParams<R> P[2];
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        D0[li + lj * LD] = Din[li + lj * TW];
        U[li + lj * LD] = (li == lj) ? R(1) : R(0);
    }
    __syncthreads();
    if (threadIdx.x == 0) g_tr[2][63] = clock64();
    const R *D = inner_rounds_wide<R>(D0, D1, U, make_int2(0, 1), false, nullptr, nu, 0, P, &nrot);
    for (int e = threadIdx.x; e < TW * TW; e += NTW) Uout[e] = U[(e & 63) + (e >> 6) * LD] + D[(e & 63) + (e >> 6) * LD];
}

// shared-memory cross rounds vs the library rounds (U in registers): bit-identical
template <typename R>
__global__ void __launch_bounds__(NTW) k3ab(const R *Din, R *out, R nu, int2 bp, int reg)
{
    constexpr int LD = LayK<R>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *D0 = (R *)smem_raw, *D1 = D0 + TW * LD, *U = D1 + TW * LD;
    __shared__ unsigned nrot;
    __shared__ WideParams<R> P[2];
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        D0[li + lj * LD] = Din[li + lj * TW];
        U[li + lj * LD] = (li == lj) ? R(1) : R(0);
    }
    __syncthreads();
    unsigned cnt = 0;
    const R *D;
    if (reg) D = inner_rounds_wide<R>(D0, D1, U, bp, false, nullptr, nu, 0, P, &nrot);
    else { D = smem_rounds_wide<R, false>(D0, D1, U, bp, false, BW, nullptr, nu, 0, P, cnt); __syncthreads(); }
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        out[e] = D[(e & 63) + (e >> 6) * LD];
        out[4096 + e] = U[(e & 63) + (e >> 6) * LD];
    }
}

template <typename R>
bool ab(const char *name)
{
    std::vector<R> h(64 * 64);
    srand(7);
    for (int j = 0; j < 64; ++j)
        for (int i = 0; i <= j; ++i) h[i + 64 * j] = h[j + 64 * i] = (i == j ? 1 + 0.01 * i : 0) + (R)rand() / RAND_MAX * 0.3;
    R *d, *o;
    cudaMalloc(&d, sizeof(R) * 4096);
    cudaMalloc(&o, sizeof(R) * 8192);
    cudaMemcpy(d, h.data(), sizeof(R) * 4096, cudaMemcpyHostToDevice);
    const int sm = 3 * TW * LayK<R>::LD * sizeof(R);
    cudaFuncSetAttribute(k3ab<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    bool ok = true;
    for (int f = 0; f < 2; ++f) {
        const int2 bp = f ? make_int2(5, 2) : make_int2(2, 5);
        std::vector<R> a(8192), b(8192);
        k3ab<R><<<1, NTW, sm>>>(d, o, R(1e-14), bp, 0);
        cudaMemcpy(a.data(), o, sizeof(R) * 8192, cudaMemcpyDeviceToHost);
        k3ab<R><<<1, NTW, sm>>>(d, o, R(1e-14), bp, 1);
        cudaMemcpy(b.data(), o, sizeof(R) * 8192, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 8192; ++i) bad += memcmp(&a[i], &b[i], sizeof(R)) != 0;
        printf("%s flip=%d: %d of 8192 words differ (%s)\n", name, f, bad, cudaGetErrorString(cudaGetLastError()));
        ok = ok && bad == 0;
    }
    return ok;
}

template <typename R>
void run(const char *name, int ctas)
{
    std::vector<R> h(64 * 64);
    srand(1);
    for (int j = 0; j < 64; ++j)
        for (int i = 0; i <= j; ++i) h[i + 64 * j] = h[j + 64 * i] = (i == j ? 2 + i : 0) + (R)rand() / RAND_MAX * 0.1;
    R *d, *u;
    cudaMalloc(&d, sizeof(R) * 4096 * ctas);
    cudaMalloc(&u, sizeof(R) * 4096 * ctas);
    for (int c = 0; c < ctas; ++c) cudaMemcpy(d + 4096 * c, h.data(), sizeof(R) * 4096, cudaMemcpyHostToDevice);
    const int sm = 3 * TW * LayK<R>::LD * sizeof(R);
    cudaFuncSetAttribute(k3<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int it = 0; it < 3; ++it) {
        unsigned long long z[3][64] = {};
        cudaMemcpyToSymbol(g_tr, z, sizeof(z));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k3<R><<<ctas, NTW, sm>>>(d, u, R(20) * (sizeof(R) == 8 ? R(1.1102230246251565e-16) : R(5.96e-8)));
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, a, b);
        cudaMemcpyFromSymbol(z, g_tr, sizeof(z));
        if (it < 2) continue;
        printf("%s ctas=%d kernel %.2f us (%s)\n", name, ctas, ms * 1e3, cudaGetErrorString(e));
        unsigned long long t0 = z[2][63], prev = t0;
        double sp = 0, sa = 0, sb = 0;
        for (int s = 0; s < 32; ++s) {
            const double p = (double)(z[0][s] - prev), a1 = (double)(z[1][s] - prev), b1 = (double)(z[2][s] - prev);
            if (s < 4 || s == 31) printf("  round %2d: params done +%6.0f  updates done +%6.0f  barrier +%6.0f cycles\n", s, p, a1, b1);
            if (s < 31) sp += p;
            sa += a1; sb += b1;
            prev = z[2][s];
        }
        printf("  mean per round: params %.0f  updates %.0f  round %.0f cycles\n", sp / 31, sa / 32, sb / 32);
    }
}

int main()
{
    const bool ok = ab<double>("fp64") & ab<float>("fp32");
    printf("bit-identical: %s\n", ok ? "yes" : "NO");
    run<double>("fp64", 1);
    run<double>("fp64", 148);
    run<float>("fp32", 1);
    run<float>("fp32", 148);
    return 0;
}
