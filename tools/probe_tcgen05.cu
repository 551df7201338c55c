// Hardware probe for the encodings the attention kernel relies on:
//   S  = Q K^T      SS MMA, both operands K-major SWIZZLE_128B via TMA
//   O1 = P V        TS MMA, P (bf16) written to TMEM by tcgen05.st, V MN-major SW128
//   O2 = P V        SS MMA, P written to smem in the K-major SW128 layout by threads
//   O3 = P V        TS MMA with V^T given K-major
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2411_01783_b200/csrc
//        probe_tcgen05.cu -o probe_tcgen05
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cudaTypedefs.h>
#include "sm100.cuh"

using namespace rcp;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

struct Maps {
  CUtensorMap q, k, v, vt;
};

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const __grid_constant__ Maps maps, float* s_out, __nv_bfloat16* p_out,
                 float* o1, float* o2, float* o3) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = smem;
  uint8_t* Ks = smem + 32768;
  uint8_t* Vs = smem + 65536;
  uint8_t* Vts = smem + 98304;
  uint8_t* Ps = smem + 131072;
  __shared__ uint64_t bar_load, bar_s, bar_o;
  __shared__ uint32_t tmem_slot;

  const uint32_t w = warp_id(), l = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_s, 1);
    mbar_init(&bar_o, 1);
    fence_mbar_init();
  }
  if (w == 0) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_slot;

  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    mbar_arrive_expect_tx(&bar_load, 4 * 32768);
    for (int h = 0; h < 2; ++h) {
      tma_load_2d(Qs + h * 16384, &maps.q, &bar_load, h * 64, 0, pol);
      tma_load_2d(Ks + h * 16384, &maps.k, &bar_load, h * 64, 0, pol);
      tma_load_2d(Vs + h * 16384, &maps.v, &bar_load, h * 64, 0, pol);
      tma_load_2d(Vts + h * 16384, &maps.vt, &bar_load, h * 64, 0, pol);
    }
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t idesc = make_idesc_bf16_f32(128, 128, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      mma_ss(tbase, make_sw128_desc(smem_u32(Qs) + off, 16, 1024),
             make_sw128_desc(smem_u32(Ks) + off, 16, 1024), idesc, kk > 0);
    }
    mma_commit(&bar_s);
  }
  __syncwarp();
  mbar_wait(&bar_s, 0);
  tc_fence_after();

  const uint32_t row = w * 32 + l;
  const uint32_t lane_addr = tbase + ((w * 32) << 16);
  float s[128];
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(lane_addr + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(r[i]);
  }
  for (int c = 0; c < 128; ++c) s_out[row * 128 + c] = s[c];
  // P = bf16(0.05 * S)
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
  // P into smem, K-major SW128: element (m,k) -> atom k/64, 16B chunk ((k%64)/8) ^ (m%8)
  for (int k8 = 0; k8 < 16; ++k8) {
    const int atom = k8 >> 3, chunk = k8 & 7;
    const int swz = chunk ^ (row & 7);
    uint4 val = make_uint4(p[k8 * 4 + 0], p[k8 * 4 + 1], p[k8 * 4 + 2], p[k8 * 4 + 3]);
    *reinterpret_cast<uint4*>(Ps + atom * 16384 + row * 128 + swz * 16) = val;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t id_mn = make_idesc_bf16_f32(128, 128, 0, 1);
    const uint32_t id_k = make_idesc_bf16_f32(128, 128, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t bv = make_sw128_desc(smem_u32(Vs) + kk * 2048, 16384, 1024);
      mma_ts(tbase + 128, tbase + kk * 8, bv, id_mn, kk > 0);
    }
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      const uint64_t bv = make_sw128_desc(smem_u32(Vs) + kk * 2048, 16384, 1024);
      mma_ss(tbase + 256, make_sw128_desc(smem_u32(Ps) + off, 16, 1024), bv, id_mn, kk > 0);
    }
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      mma_ts(tbase + 384, tbase + kk * 8, make_sw128_desc(smem_u32(Vts) + off, 16, 1024), id_k,
             kk > 0);
    }
    mma_commit(&bar_o);
  }
  __syncwarp();
  mbar_wait(&bar_o, 0);
  tc_fence_after();
  float* outs[3] = {o1, o2, o3};
  for (int which = 0; which < 3; ++which) {
    for (int c = 0; c < 128; c += 32) {
      uint32_t r[32];
      tmem_ld32(lane_addr + 128 * (which + 1) + c, r);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) outs[which][row * 128 + c + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tbase);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap make_map(void* ptr) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, 128};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  const int n = 128 * 128;
  std::vector<__nv_bfloat16> hq(n), hk(n), hv(n), hvt(n);
  std::vector<float> fq(n), fk(n), fv(n);
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  for (int i = 0; i < n; ++i) {
    fq[i] = bf(rnd()); fk[i] = bf(rnd()); fv[i] = bf(rnd());
    hq[i] = __float2bfloat16(fq[i]); hk[i] = __float2bfloat16(fk[i]); hv[i] = __float2bfloat16(fv[i]);
  }
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 128; ++c) hvt[c * 128 + r] = hv[r * 128 + c];
  void *dq, *dk, *dv, *dvt;
  float *ds, *o1, *o2, *o3;
  __nv_bfloat16* dp;
  CK(cudaMalloc(&dq, n * 2)); CK(cudaMalloc(&dk, n * 2)); CK(cudaMalloc(&dv, n * 2)); CK(cudaMalloc(&dvt, n * 2));
  CK(cudaMalloc(&ds, n * 4)); CK(cudaMalloc(&o1, n * 4)); CK(cudaMalloc(&o2, n * 4)); CK(cudaMalloc(&o3, n * 4));
  CK(cudaMalloc(&dp, n * 2));
  CK(cudaMemcpy(dq, hq.data(), n * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, hk.data(), n * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), n * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dvt, hvt.data(), n * 2, cudaMemcpyHostToDevice));
  Maps maps{make_map(dq), make_map(dk), make_map(dv), make_map(dvt)};
  const int smem = 5 * 32768 + 1024;
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_kernel<<<1, 128, smem>>>(maps, ds, dp, o1, o2, o3);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> hs(n), h1(n), h2(n), h3(n);
  std::vector<__nv_bfloat16> hp(n);
  CK(cudaMemcpy(hs.data(), ds, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hp.data(), dp, n * 2, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h1.data(), o1, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), o2, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h3.data(), o3, n * 4, cudaMemcpyDeviceToHost));
  double es = 0, e1 = 0, e2 = 0, e3 = 0, ms = 0, mo = 0;
  for (int m = 0; m < 128; ++m)
    for (int c = 0; c < 128; ++c) {
      double ref = 0;
      for (int k = 0; k < 128; ++k) ref += (double)fq[m * 128 + k] * fk[c * 128 + k];
      es = fmax(es, fabs(ref - hs[m * 128 + c]));
      ms = fmax(ms, fabs(ref));
      double ro = 0;
      for (int k = 0; k < 128; ++k) ro += (double)__bfloat162float(hp[m * 128 + k]) * fv[k * 128 + c];
      mo = fmax(mo, fabs(ro));
      e1 = fmax(e1, fabs(ro - h1[m * 128 + c]));
      e2 = fmax(e2, fabs(ro - h2[m * 128 + c]));
      e3 = fmax(e3, fabs(ro - h3[m * 128 + c]));
    }
  printf("S  (SS K/K)        max_abs_err=%.3e (max |S|=%.3f)  %s\n", es, ms, es < 1e-2 ? "OK" : "FAIL");
  printf("O1 (TS P, V MN)    max_abs_err=%.3e (max |O|=%.3f)  %s\n", e1, mo, e1 < 1e-2 ? "OK" : "FAIL");
  printf("O2 (SS P smem, MN) max_abs_err=%.3e  %s\n", e2, e2 < 1e-2 ? "OK" : "FAIL");
  printf("O3 (TS P, V^T K)   max_abs_err=%.3e  %s\n", e3, e3 < 1e-2 ? "OK" : "FAIL");
  printf("sample S[0][0..3]=%f %f %f %f\n", hs[0], hs[1], hs[2], hs[3]);
  printf("sample O1[0][0..3]=%f %f %f %f\n", h1[0], h1[1], h1[2], h1[3]);
  return 0;
}
