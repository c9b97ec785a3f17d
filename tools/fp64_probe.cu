// Throughput of the epilogue's FP64-pipe instructions on this GPU (per SM per
// clock): DMUL, DADD, F2F.F32.F64 (double -> float RN), I2F.F64.S32, with FMUL
// as the FP32 reference. 8 independent chains per thread, grid = 4 x SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_probe.cu -o tools/fp64_probe.bin
#include <cuda_runtime.h>
#include <cstdio>

constexpr int kIters = 4096;

__global__ void k_dmul(double* out, double s) {
    double v[8];
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __dmul_rn(v[i], s);
    double r = 0;
    for (int i = 0; i < 8; ++i) r += v[i];
    if (r == 1.2345) out[0] = r;
}
__global__ void k_dadd(double* out, double s) {
    double v[8];
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __dadd_rn(v[i], s);
    double r = 0;
    for (int i = 0; i < 8; ++i) r += v[i];
    if (r == 1.2345) out[0] = r;
}
__global__ void k_f2f(double* out, double s) {
    double v[8];
    float acc[8];
    for (int i = 0; i < 8; ++i) { v[i] = (threadIdx.x + i) * s; acc[i] = 0.f; }
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) { v[i] = __dmul_rn(v[i], s); acc[i] += __double2float_rn(v[i]); }  // DMUL + F2F + FADD
    float r = 0;
    for (int i = 0; i < 8; ++i) r += acc[i];
    if (r == 1.2345f) out[0] = r;
}
__global__ void k_i2f(double* out, double s) {
    int v[8];
    double acc[8];
    for (int i = 0; i < 8; ++i) { v[i] = threadIdx.x * 7 + i; acc[i] = 0; }
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc[i] = __dadd_rn(acc[i], __int2double_rn(v[i] + it)); }  // I2F + DADD
    double r = 0;
    for (int i = 0; i < 8; ++i) r += acc[i];
    if (r == 1.2345) out[0] = r;
}
__global__ void k_fmul(double* out, double s) {
    float v[8];
    const float sf = float(s);
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fmul_rn(v[i], sf);
    float r = 0;
    for (int i = 0; i < 8; ++i) r += v[i];
    if (r == 1.2345f) out[0] = r;
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, void (*k)(double*, double)) {
        const int blocks = 4 * sms, threads = 256;
        k<<<blocks, threads>>>(out, 1.0000001);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(out, 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = double(blocks) * threads * kIters * 8;
        const double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
        printf("%-28s %8.3f ms  %7.1f ops/clk/SM (at %.0f MHz nominal)\n", name, ms, per_sm_clk, clk / 1e3);
    };
    run("DMUL", k_dmul);
    run("DADD", k_dadd);
    run("DMUL+F2F.F32.F64+FADD", k_f2f);
    run("I2F.F64+DADD", k_i2f);
    run("FMUL", k_fmul);
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
}
