// Throughput probe: cycles per tcgen05.mma for the shapes the attention kernels issue.
//   1-CTA  SS  M=128 N=64/128/256  (v4 S = Q K^T uses N=64)
//   1-CTA  TS  M=128 N=128         (v4 O += P V)
//   2-CTA  SS  M=256 N=128/256     (v5 S)
//   2-CTA  TS  M=256 N=128         (v5 O += P V)
// Optionally 4 extra warps stream tcgen05.ld from a disjoint TMEM region meanwhile
// (what the softmax warpgroups do), to see whether TMEM reads slow the MMA pipe.
// Operands are whatever is in shared memory: only timing matters here.
#include <cstdio>
#include <cstdlib>
#include "sm100.cuh"

using namespace rcp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int kIters = 2048;

__device__ __forceinline__ void mma1_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma1_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// kind: 0 = SS, 1 = TS.  CTA2: cta_group::2 (launched as clusters of 2).
template <bool CTA2>
__device__ void body(int kind, int n, int ld_traffic, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  __shared__ volatile int stop;
  const uint32_t w = warp_id();
  const uint32_t rank = CTA2 ? cluster_rank() : 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (w == 0) {
    if (CTA2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_slot)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_slot)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CTA2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_slot;
  if (w == 0 && rank == 0) {
    if (elect_one()) {
      const int m = CTA2 ? 256 : 128;
      const uint32_t idesc = make_idesc_bf16_f32(m, n, 0, kind == 1 ? 1 : 0);
      const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 65536);
      const long long t0 = clock64();
      for (int i = 0; i < kIters; ++i) {
        const int kk = i & 7;
        const uint64_t b = kind == 0 ? make_sw128_desc(b0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024)
                                     : make_sw128_desc(b0 + kk * 2048, 16384, 1024);
        if (kind == 0) {
          const uint64_t a = make_sw128_desc(a0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          if (CTA2) mma2_ss(tbase, a, b, idesc, kk > 0); else mma1_ss(tbase, a, b, idesc, kk > 0);
        } else {
          if (CTA2) mma2_ts(tbase + 256, tbase + kk * 8, b, idesc, kk > 0);
          else mma1_ts(tbase + 256, tbase + kk * 8, b, idesc, kk > 0);
        }
      }
      if (CTA2)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     :: "r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(smem_u32(&bar)) : "memory");
      mbar_wait(&bar, 0);
      const long long t1 = clock64();
      out[blockIdx.x] = (unsigned long long)(t1 - t0);
      stop = 1;
    }
    __syncwarp();
  } else if (w == 0) {
    mbar_wait(&bar, 0);
    stop = 1;
  } else if (w >= 4 && ld_traffic) {
    // stream TMEM reads from columns [384, 512) (never written by the MMAs)
    const uint32_t lane_addr = tbase + (((w & 3) * 32) << 16) + 384;
    float acc = 0.f;
    while (!stop) {
      for (int c = 0; c < 128; c += 32) {
        uint32_t r[32];
        tmem_ld32(lane_addr + c, r);
        tmem_ld_wait();
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
      }
    }
    if (acc == 12345.f) out[1023] = 1;
  }
  tc_fence_before();
  if (CTA2) cluster_sync(); else __syncthreads();
  if (w == 0) {
    if (CTA2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tbase), "n"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "n"(512));
  }
}

__global__ void __launch_bounds__(256, 1) k1(int kind, int n, int ld, unsigned long long* out) { body<false>(kind, n, ld, out); }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) k2(int kind, int n, int ld, unsigned long long* out) {
  body<true>(kind, n, ld, out);
}

int main() {
  unsigned long long* d; CK(cudaMalloc(&d, 1024 * 8));
  const int smem = 196608 + 1024;
  CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  struct Case { int cta2, kind, n; const char* name; } cases[] = {
      {0, 0, 64, "1CTA SS M128 N64 "}, {0, 0, 128, "1CTA SS M128 N128"}, {0, 0, 256, "1CTA SS M128 N256"},
      {0, 1, 128, "1CTA TS M128 N128"}, {0, 1, 256, "1CTA TS M128 N256"},
      {1, 0, 128, "2CTA SS M256 N128"}, {1, 0, 256, "2CTA SS M256 N256"}, {1, 1, 128, "2CTA TS M256 N128"},
      {1, 1, 256, "2CTA TS M256 N256"}};
  for (int grid : {2, 148}) {
    for (int ld = 0; ld < 2; ++ld) {
      for (auto& c : cases) {
        for (int rep = 0; rep < 2; ++rep) {
          if (c.cta2) k2<<<grid, 256, smem>>>(c.kind, c.n, ld, d); else k1<<<grid, 256, smem>>>(c.kind, c.n, ld, d);
          CK(cudaGetLastError());
          CK(cudaDeviceSynchronize());
        }
        unsigned long long h; CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
        const double per = (double)h / kIters;
        // ideal: M x N x 16 MACs at 4096 MAC/clk/SM (8192 dense bf16 flop/clk/SM); 2-CTA spans 2 SMs
        const int m = c.cta2 ? 256 : 128;
        const double ideal = (double)m * c.n * 16 / (4096.0 * (c.cta2 ? 2 : 1));
        printf("grid %3d ld_traffic %d  %s : %7.1f clk/mma (ideal %5.1f) -> %5.1f%%\n", grid, ld, c.name, per, ideal,
               100.0 * ideal / per);
      }
    }
  }
  return 0;
}
