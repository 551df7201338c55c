// Hardware probe for the 2-CTA (cta_group::2) encodings of the planned v5 kernel:
//   cluster of 2 CTAs, CTA r holds Q rows [128r, 128r+128) (K-major SW128),
//   K keys [64r, 64r+64) (K-major SW128), V dims [64r, 64r+64) of all 128 keys
//   (MN-major SW128).  Leader issues S = Q K^T (M=256, N=128) and, after both
//   CTAs write P = bf16(0.05 S) into their TMEM, O = P V (TS, M=256, N=128).
//   TMA completions of both CTAs land on the leader's barrier; commits multicast.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cudaTypedefs.h>
#include "sm100.cuh"

using namespace rcp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

struct Maps { CUtensorMap q, k, v; };

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma2sm(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;  // leader CTA's barrier
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%3, %4}], [%2];" :: "r"(smem_u32(dst)), "l"((uint64_t)m), "r"(b), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(b) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe2(const __grid_constant__ Maps maps, float* s_out, __nv_bfloat16* p_out, float* o_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = smem;              // 32 KB: 128 rows x 128 dims
  uint8_t* Ks = smem + 32768;      // 16 KB: 64 keys x 128 dims
  uint8_t* Vs = smem + 49152;      // 16 KB: 128 keys x 64 dims
  __shared__ uint64_t bar_load, bar_s, bar_p, bar_o;
  __shared__ uint32_t tmem_slot;
  const uint32_t rank = cluster_rank();
  const uint32_t w = warp_id(), l = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_s, 1);
    mbar_init(&bar_p, 2 * 4);  // 4 warps per CTA, both CTAs
    mbar_init(&bar_o, 1);
    fence_mbar_init();
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_slot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_slot;
  if (threadIdx.x == 0) {
    if (rank == 0) mbar_arrive_expect_tx(&bar_load, 2 * (32768 + 16384 + 16384));
    for (int h = 0; h < 2; ++h) {
      tma2sm(Qs + h * 16384, &maps.q, &bar_load, h * 64, rank * 128);
      tma2sm(Ks + h * 8192, &maps.k, &bar_load, h * 64, rank * 64);
    }
    tma2sm(Vs, &maps.v, &bar_load, rank * 64, 0);
  }
  if (rank == 0 && threadIdx.x == 0) {
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t idesc = make_idesc_bf16_f32(256, 128, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = make_sw128_desc(smem_u32(Qs) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
      const uint64_t b = make_sw128_desc(smem_u32(Ks) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
      mma2_ss(tbase, a, b, idesc, kk > 0);
    }
    commit2_mc(&bar_s);
  }
  __syncwarp();
  mbar_wait(&bar_s, 0);
  tc_fence_after();
  const uint32_t row = rank * 128 + w * 32 + l;
  const uint32_t lane_addr = tbase + ((w * 32) << 16);
  float s[128];
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(lane_addr + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(r[i]);
  }
  for (int c = 0; c < 128; ++c) s_out[row * 128 + c] = s[c];
  uint32_t p[64];
  for (int i = 0; i < 64; ++i) p[i] = pack_bf16x2(0.05f * s[2 * i], 0.05f * s[2 * i + 1]);
  for (int i = 0; i < 64; ++i) {
    __nv_bfloat162 v2 = *reinterpret_cast<__nv_bfloat162*>(&p[i]);
    p_out[row * 128 + 2 * i] = v2.x;
    p_out[row * 128 + 2 * i + 1] = v2.y;
  }
  tmem_st32(lane_addr + 0, p);
  tmem_st32(lane_addr + 32, p + 32);
  tmem_st_wait();
  tc_fence_before();
  __syncwarp();
  if (l == 0) arrive_leader(&bar_p);
  if (rank == 0 && threadIdx.x == 0) {
    mbar_wait(&bar_p, 0);
    tc_fence_after();
    const uint32_t idesc = make_idesc_bf16_f32(256, 128, 0, 1);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t b = make_sw128_desc(smem_u32(Vs) + kk * 2048, 16384, 1024);
      mma2_ts(tbase + 128, tbase + kk * 8, b, idesc, kk > 0);
    }
    commit2_mc(&bar_o);
  }
  __syncwarp();
  mbar_wait(&bar_o, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(lane_addr + 128 + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) o_out[row * 128 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  cluster_sync();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tbase), "n"(512));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}
static CUtensorMap mk(void* p, int rows, int box_rows) {
  CUtensorMap m; cuuint64_t dims[2] = {128, (cuuint64_t)rows}; cuuint64_t st[1] = {256};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}; cuuint32_t es[2] = {1, 1};
  if (enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc\n"); exit(1); }
  return m;
}
static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  const int MQ = 256, NK = 128, D = 128;
  std::vector<__nv_bfloat16> hq(MQ * D), hk(NK * D), hv(NK * D);
  std::vector<float> fq(MQ * D), fk(NK * D), fv(NK * D);
  srand(3);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  for (int i = 0; i < MQ * D; ++i) { fq[i] = bf(rnd()); hq[i] = __float2bfloat16(fq[i]); }
  for (int i = 0; i < NK * D; ++i) { fk[i] = bf(rnd()); hk[i] = __float2bfloat16(fk[i]); fv[i] = bf(rnd()); hv[i] = __float2bfloat16(fv[i]); }
  void *dq, *dk, *dv; float *ds, *dout; __nv_bfloat16* dp;
  CK(cudaMalloc(&dq, MQ * D * 2)); CK(cudaMalloc(&dk, NK * D * 2)); CK(cudaMalloc(&dv, NK * D * 2));
  CK(cudaMalloc(&ds, MQ * 128 * 4)); CK(cudaMalloc(&dout, MQ * 128 * 4)); CK(cudaMalloc(&dp, MQ * 128 * 2));
  CK(cudaMemcpy(dq, hq.data(), MQ * D * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, hk.data(), NK * D * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), NK * D * 2, cudaMemcpyHostToDevice));
  Maps maps{mk(dq, MQ, 128), mk(dk, NK, 64), mk(dv, NK, 128)};
  const int smem = 65536 + 1024;
  CK(cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe2<<<2, 128, smem>>>(maps, ds, dp, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> hs(MQ * 128), ho(MQ * 128); std::vector<__nv_bfloat16> hp(MQ * 128);
  CK(cudaMemcpy(hs.data(), ds, MQ * 128 * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ho.data(), dout, MQ * 128 * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hp.data(), dp, MQ * 128 * 2, cudaMemcpyDeviceToHost));
  double es = 0, eo = 0;
  for (int m = 0; m < MQ; ++m)
    for (int n = 0; n < 128; ++n) {
      double r = 0; for (int k = 0; k < D; ++k) r += (double)fq[m * D + k] * fk[n * D + k];
      es = fmax(es, fabs(r - hs[m * 128 + n]));
      double o = 0; for (int k = 0; k < NK; ++k) o += (double)__bfloat162float(hp[m * 128 + k]) * fv[k * D + n];
      eo = fmax(eo, fabs(o - ho[m * 128 + n]));
    }
  printf("2CTA S (M=256 SS, B split by N)  max_abs_err=%.3e %s\n", es, es < 1e-2 ? "OK" : "FAIL");
  printf("2CTA O (M=256 TS, V split by N)  max_abs_err=%.3e %s\n", eo, eo < 1e-2 ? "OK" : "FAIL");
  return 0;
}
