// rot_latency.cu -- latency (cycles) of one dependent Lemma 3.1 parameter
// computation (mpj::rot_params) and of its pieces, one warp, clock64().
#include <cstdio>
#include "../paper_2211_03339_b200/csrc/mpj_device.cuh"

template <typename R>
__global__ void k(R *out, long long *cyc, int iters)
{
    R app = 1.0 + threadIdx.x * 1e-3, aqq = 2.0, apq = 0.3;
    long long t0 = clock64();
    R acc = 0;
    for (int i = 0; i < iters; ++i) {
        R t, s, u;
        mpj::rot_params<R>(app, aqq, apq, R(1e-15), 0, t, s, u);
        apq = apq + u * R(1e-30);   // dependence on the result
        acc += s;
    }
    long long t1 = clock64();
    R x = aqq;
    for (int i = 0; i < iters; ++i) x = mpj::divR(R(1), x + R(1));
    long long t2 = clock64();
    R y = aqq;
    for (int i = 0; i < iters; ++i) y = mpj::sqrtR(y + R(1));
    long long t3 = clock64();
    R z = aqq;
    for (int i = 0; i < iters; ++i) z = mpj::fmaR(z, R(0.999), R(0.001));
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1) / iters; cyc[2] = (t3 - t2) / iters; cyc[3] = (t4 - t3) / iters;
    }
    out[threadIdx.x] = acc + x + y + z;
}

int main()
{
    double *o; long long *c, h[4];
    cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
    k<double><<<1, 32>>>(o, c, 1000); cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("{\"f64_rot_params_cycles\": %lld, \"f64_div\": %lld, \"f64_sqrt\": %lld, \"f64_fma\": %lld, ", h[0], h[1], h[2], h[3]);
    k<float><<<1, 32>>>((float *)o, c, 1000); cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("\"f32_rot_params_cycles\": %lld, \"f32_div\": %lld, \"f32_sqrt\": %lld, \"f32_fma\": %lld}\n", h[0], h[1], h[2], h[3]);
    return 0;
}
