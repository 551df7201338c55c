// Probe: (1) the register layout of ldmatrix.m16n16.x1.trans.b8 on sm_100a,
// (2) the issue cost of e4m3x2 -> f16x2 conversion (F2FP.F16.E4M3.UNPACK_B)
// against a plain FMUL stream, per SM.  Prints one line per item.
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>

__global__ void layout_kernel(uint32_t* out) {
  __shared__ __align__(128) uint8_t s[256];
  for (int i = threadIdx.x; i < 256; i += 32) s[i] = i;  // s[r*16+c] = (r<<4)|c
  __syncwarp();
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(s) + (threadIdx.x & 15) * 16;
  uint32_t r0, r1;
  asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(a));
  out[threadIdx.x * 2] = r0;
  out[threadIdx.x * 2 + 1] = r1;
}

template <int MODE>
__global__ void tput_kernel(uint32_t* out, int iters, long long* cyc) {
  uint32_t x[8];
  for (int i = 0; i < 8; ++i) x[i] = 0x38383838u + threadIdx.x + i;
  uint32_t acc = 0;
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = 1.0f + threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(x[i]) : "h"((unsigned short)x[i]));
      } else {
        f[i] = f[i] * 1.0001f;
      }
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < 8; ++i) acc ^= x[i];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  for (int i = 0; i < 8; ++i) acc ^= __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint32_t* d;
  long long* c;
  cudaMalloc(&d, 1 << 24);
  cudaMalloc(&c, 1 << 16);
  layout_kernel<<<1, 32>>>(d);
  uint32_t h[64];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("ldmatrix.m16n16.x1.trans.b8: thread -> bytes (row<<4|col) of r0 | r1\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%02d:", t);
    for (int j = 0; j < 2; ++j)
      for (int b = 0; b < 4; ++b) printf(" %02x", (h[2 * t + j] >> (8 * b)) & 0xff);
    printf("%s", t % 2 ? "\n" : "   ");
  }
  const int iters = 4096, threads = 512, blocks = 148;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) tput_kernel<0><<<blocks, threads>>>(d, iters, c);
      else tput_kernel<1><<<blocks, threads>>>(d, iters, c);
    }
    cudaDeviceSynchronize();
    long long cy;
    cudaMemcpy(&cy, c, sizeof(cy), cudaMemcpyDeviceToHost);
    const double ops = double(iters) * 8 * threads;  // per SM (one CTA per SM)
    printf("%s: %.1f thread-ops/clk/SM (%lld cycles)\n", mode == 0 ? "cvt e4m3x2->f16x2" : "FMUL", ops / cy, cy);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
