#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include "lqg_gemm.cuh"
using namespace lqg;
__global__ void k(const double* in, uint32_t* bad, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  double y = in[i];
  float a = f64_to_f32_rn(y), b = __double2float_rn(y);
  if (__float_as_uint(a) != __float_as_uint(b)) atomicAdd(bad, 1u);
  __nv_bfloat16 c = f32_to_bf16_rn(b), d = __float2bfloat16_rn(b);
  if (b == b && __bfloat16_as_ushort(c) != __bfloat16_as_ushort(d)) atomicAdd(bad + 1, 1u);  // NaN unreachable in the kernel
  int32_t ai = (int32_t)(((unsigned)i * 2654435761u));
  if (i32_to_f64_exact(ai) != (double)ai) atomicAdd(bad + 2, 1u);
}
int main() {
  const int n = 1 << 24;
  double* h = (double*)malloc(n * 8);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    uint64_t bits = s;
    int mode = i % 4;
    if (mode == 0) { double v; memcpy(&v, &bits, 8); h[i] = v; }                 // any bit pattern
    else if (mode == 1) h[i] = (double)(int32_t)bits * 1e-7 * (double)((bits >> 40) & 0xFFF);  // epilogue-like
    else if (mode == 2) { uint64_t b2 = (bits & 0x800FFFFFFFFFFFFFull) | ((uint64_t)(0x380 + (bits >> 52) % 0x100) << 52); double v; memcpy(&v,&b2,8); h[i]=v; } // near float range edges
    else { uint64_t b2 = (bits & 0xFFFFFFFFE0000000ull) | 0x10000000ull; double v; memcpy(&v,&b2,8); h[i] = v; } // exact ties
  }
  double* d; uint32_t* bad; cudaMalloc(&d, n * 8); cudaMalloc(&bad, 12); cudaMemset(bad, 0, 12);
  cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(d, bad, n);
  uint32_t hb[3]; cudaMemcpy(hb, bad, 12, cudaMemcpyDeviceToHost);
  printf("f32 mismatches %u  bf16 mismatches %u  i32->f64 mismatches %u  (err %s)\n", hb[0], hb[1], hb[2], cudaGetErrorString(cudaGetLastError()));
  return hb[0] || hb[1] || hb[2];
}
