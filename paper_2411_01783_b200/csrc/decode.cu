// K4: split-KV decode attention for ring pass-Q decode (Alg. 4).
//
// One query token per sequence against that sequence's cached KV shard on this
// rank.  HBM-bound: every cached K/V byte is read exactly once.  Grid = (split,
// KV head, sequence); a CTA streams `keys_per_cta` keys of one KV head through a
// 4-stage TMA ring (64-key K and V blocks, SW128) and serves all hq/hkv query
// heads that read it (GQA packing: up to 16 heads form the M=16 of
// mma.sync.m16n8k16, so K/V are read once per KV head, not once per query
// head; at 16 query heads per KV head the tensor cores keep up with HBM, which
// CUDA-core FMAs cannot).  Each of the 4 warps owns a 16-key slice of every
// block with its own online softmax; the warps' partials are merged in shared
// memory and the CTA writes a normalised (O, LSE) partial per head; a combine
// kernel folds the splits in ascending order with the fp32 merge of
// merge_attention.
//
// FP8 KV (rcp_decode_attn_fp8): the cache holds K/V as e4m3 bytes with one
// fp32 scale per KV head (x = scale * e4m3).  Same kernel, halved bytes: a
// 64-key block is one 8 KB SW128 TMA box per operand, and the fragments are
// widened to f16 in registers (F2FP unpack, 2 elements per instruction) for
// f16 mma.sync — sm_100's mma.sync has no native 8-bit path either, so this is
// what an e4m3 mma.sync would compile to, with Q and P kept in f16 instead of
// being quantised.  K: a non-transposed b16 ldmatrix hands each thread 4
// consecutive dims of one key, which become the B fragment under a fixed
// permutation of the reduction dim (mirrored in the Q fragment).  V: a
// transposed b16 ldmatrix hands each thread 2 keys x 2 dims; one PRMT per
// register pair regroups them into key pairs per dim, so each thread's O
// accumulators cover 4 consecutive dims per 16-dim chunk.  The K scale folds
// into the softmax scale, the V scale into the final normalisation.
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace rcp {

constexpr int kDecBlock = 64;      // keys per TMA block
#ifndef RCP_DEC_STAGES
#define RCP_DEC_STAGES 2
#endif
#ifndef RCP_DEC_STAGES_FP8
#define RCP_DEC_STAGES_FP8 4
#endif
constexpr int kDecWarps = 4;       // 16-key slice of each block per warp
constexpr int kDecThreads = kDecWarps * 32;
constexpr int kDecMaxGroup = 16;   // query heads per KV head (mma M)
constexpr uint32_t kDecBoxBytes = kDecBlock * 128;      // 8 KB: 64 rows x 128 bytes (one SW128 box)
// Ring geometry per KV element type.  bf16: 32 KB (K + V of 64 keys) per
// stage; two stages (65 KB) let three CTAs share an SM, so one CTA's pipeline
// fill and epilogue overlap the others' streaming: measured 6.5 TB/s at B=16
// and 0.32 ms vs 0.44 ms per graphed B=1 step against four stages (one CTA per
// SM).  e4m3: 16 KB per stage, four stages in the same 65 KB (same bytes in
// flight, same three CTAs per SM).
template <bool kFp8>
struct DecGeo {
  static constexpr uint32_t kTileBytes = kFp8 ? kDecBoxBytes : 2 * kDecBoxBytes;  // 64 keys x 128 dims
  static constexpr uint32_t kStageBytes = 2 * kTileBytes;                         // K + V
  static constexpr int kStages = kFp8 ? RCP_DEC_STAGES_FP8 : RCP_DEC_STAGES;
  static constexpr uint32_t kSmemBytes = kStages * kStageBytes + 1024;
};

struct DecodeParams {
  CUtensorMap tm_k, tm_v;
  const __nv_bfloat16* q;
  const int64_t* kv_start;
  const int64_t* kv_len;
  float* part_o;
  float* part_lse;
  const float* k_scale;  // e4m3 only: per KV head
  const float* v_scale;
  int hq, hkv, group, n_split, keys_per_cta;
  float scale_log2;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_16816_f16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                              uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <bool kFp8>
__device__ __forceinline__ void mma_dec(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  if constexpr (kFp8)
    mma_16816_f16(c, a0, a1, a2, a3, b0, b1);
  else
    mma_16816(c, a0, a1, a2, a3, b0, b1);
}
// Two e4m3 values (low byte -> low half) to f16x2; exact.
__device__ __forceinline__ uint32_t e4m3x2_f16x2(uint32_t x16) {
  uint32_t r;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(static_cast<uint16_t>(x16)));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
// Byte address of 16-byte chunk `chunk` of `row` in a 64-row SW128 tile: two
// 64-dim boxes for bf16 (chunks 0..15), one 128-dim box for e4m3 (0..7).
__device__ __forceinline__ uint32_t sw128(uint32_t tile, int row, int chunk) {
  return tile + (chunk >> 3) * kDecBoxBytes + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

template <bool kFp8>
__device__ __forceinline__ void issue_block(const DecodeParams& p, uint8_t* st, uint64_t* bar,
                                            int kvh, int row, uint64_t pol) {
  using G = DecGeo<kFp8>;
  mbar_arrive_expect_tx(bar, G::kStageBytes);
  if constexpr (kFp8) {
    tma_load_2d(st, &p.tm_k, bar, kvh * 128, row, pol);
    tma_load_2d(st + G::kTileBytes, &p.tm_v, bar, kvh * 128, row, pol);
  } else {
    for (int h = 0; h < 2; ++h) {
      tma_load_2d(st + h * kDecBoxBytes, &p.tm_k, bar, kvh * 128 + h * 64, row, pol);
      tma_load_2d(st + G::kTileBytes + h * kDecBoxBytes, &p.tm_v, bar, kvh * 128 + h * 64, row, pol);
    }
  }
}

template <bool kFp8>
__global__ void __launch_bounds__(kDecThreads) decode_mma_kernel(const __grid_constant__ DecodeParams p) {
  using G = DecGeo<kFp8>;
  constexpr int kDecStages = G::kStages;
  constexpr uint32_t kDecStageBytes = G::kStageBytes;
  constexpr uint32_t kDecTileBytes = G::kTileBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kDecStages], empty[kDecStages];
  __shared__ float red_m[kDecWarps][kDecMaxGroup], red_l[kDecWarps][kDecMaxGroup];

  // KV heads vary fastest: the CTAs of one key range's heads run together, so
  // the L2 lines they share (e4m3: two heads' rows per 256-byte promotion) are
  // read from DRAM once
  // Groups of more than 16 query heads per KV head (MQA-like geometries) take
  // ceil(group / 16) CTAs per KV head, 16 heads each (the K/V block is then
  // read once per 16 heads; L2 serves the repeats of CTAs running together).
  const int n_hc = (p.group + kDecMaxGroup - 1) / kDecMaxGroup;
  const int kvh = static_cast<int>(blockIdx.x) / n_hc, hc = static_cast<int>(blockIdx.x) - kvh * n_hc;
  const int grp = min(kDecMaxGroup, p.group - hc * kDecMaxGroup);  // query heads of this CTA
  const int split = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t len = __ldg(p.kv_len + b);
  const int64_t k0 = static_cast<int64_t>(split) * p.keys_per_cta;
  const int64_t k1 = min(len, k0 + p.keys_per_cta);
  const int n_blocks = k1 > k0 ? static_cast<int>((k1 - k0 + kDecBlock - 1) / kDecBlock) : 0;
  const int row0 = b * p.hq + kvh * p.group + hc * kDecMaxGroup;  // first query-head row of this CTA
  const int64_t part_base = static_cast<int64_t>(row0) * p.n_split + split;

  // A split past the end of its sequence (or an empty slot of the gathered
  // batch) writes nothing: the combine reads only the ceil(len / keys_per_cta)
  // splits that hold keys.
  if (n_blocks == 0) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDecStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kDecWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t row_base = __ldg(p.kv_start + b) + k0;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&p.tm_k);
    tma_prefetch_desc(&p.tm_v);
    const uint64_t pol = policy_evict_first();
    for (int i = 0; i < min(n_blocks, kDecStages); ++i)
      issue_block<kFp8>(p, smem + i * kDecStageBytes, &full[i], kvh,
                  static_cast<int>(row_base + i * kDecBlock), pol);
  }
  // Q fragments (A operand, rows = query heads of the group, zero-padded to 16)
  uint32_t qa[8][4];
  if constexpr (kFp8) {
    // f16, reduction dims permuted to match the K fragments: k-step ks takes
    // dims 16ks + 4t4 + {0,1} (a0/a1) and 16ks + 4t4 + {2,3} (a2/a3).
    const __nv_bfloat16* q0 = p.q + static_cast<int64_t>(row0) * 128;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int c = ks * 16 + 4 * t4;
      uint2 r0 = make_uint2(0u, 0u), r1 = make_uint2(0u, 0u);
      if (g < grp) r0 = *reinterpret_cast<const uint2*>(q0 + g * 128 + c);
      if (g + 8 < grp) r1 = *reinterpret_cast<const uint2*>(q0 + (g + 8) * 128 + c);
      auto cvt = [](uint32_t b) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b));
        return pack_f16x2(f.x, f.y);
      };
      qa[ks][0] = cvt(r0.x);
      qa[ks][1] = cvt(r1.x);
      qa[ks][2] = cvt(r0.y);
      qa[ks][3] = cvt(r1.y);
    }
  } else {
    const __nv_bfloat16* q0 = p.q + static_cast<int64_t>(row0) * 128;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int c = ks * 16 + 2 * t4;
      qa[ks][0] = g < grp ? *reinterpret_cast<const uint32_t*>(q0 + g * 128 + c) : 0u;
      qa[ks][1] = g + 8 < grp ? *reinterpret_cast<const uint32_t*>(q0 + (g + 8) * 128 + c) : 0u;
      qa[ks][2] = g < grp ? *reinterpret_cast<const uint32_t*>(q0 + g * 128 + c + 8) : 0u;
      qa[ks][3] = g + 8 < grp ? *reinterpret_cast<const uint32_t*>(q0 + (g + 8) * 128 + c + 8) : 0u;
    }
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};  // rows g, g+8
  const float sl2 = kFp8 ? p.scale_log2 * __ldg(p.k_scale + kvh) : p.scale_log2;
  const uint32_t smem_base = smem_u32(smem);
  const int key0 = warp * 16;  // this warp's 16 keys of every block

  for (int i = 0; i < n_blocks; ++i) {
    const int s = i % kDecStages;
    mbar_wait(&full[s], (i / kDecStages) & 1);
    const uint32_t kt = smem_base + s * kDecStageBytes, vt = kt + kDecTileBytes;
    // S[16 heads x 16 keys] = Q K^T : two n-tiles of 8 keys, 8 k-steps of 16 dims
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    if constexpr (kFp8) {
#pragma unroll
      for (int ks = 0; ks < 8; ks += 2) {
        // x4 matrices (8 keys x 16 bytes): (keys 0-7, dims 16ks..) (keys 0-7, 16ks+16..)
        // (keys 8-15, 16ks..) (keys 8-15, 16ks+16..); each register = 4 dims of one key
        const int mrow = key0 + (lane & 7) + ((lane >> 4) << 3);
        const int mchunk = ks + ((lane >> 3) & 1);
        uint32_t r00, r01, r10, r11;
        ldsm_x4(sw128(kt, mrow, mchunk), r00, r01, r10, r11);
        mma_16816_f16(sc[0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], e4m3x2_f16x2(r00),
                      e4m3x2_f16x2(r00 >> 16));
        mma_16816_f16(sc[0], qa[ks + 1][0], qa[ks + 1][1], qa[ks + 1][2], qa[ks + 1][3], e4m3x2_f16x2(r01),
                      e4m3x2_f16x2(r01 >> 16));
        mma_16816_f16(sc[1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], e4m3x2_f16x2(r10),
                      e4m3x2_f16x2(r10 >> 16));
        mma_16816_f16(sc[1], qa[ks + 1][0], qa[ks + 1][1], qa[ks + 1][2], qa[ks + 1][3], e4m3x2_f16x2(r11),
                      e4m3x2_f16x2(r11 >> 16));
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        // x4 matrices: (keys 0-7, dims 16ks..+7) (keys 0-7, +8..+15) (keys 8-15, ..) (keys 8-15, ..)
        const int mrow = key0 + (lane & 7) + ((lane >> 4) << 3);
        const int mchunk = 2 * ks + ((lane >> 3) & 1);
        uint32_t b00, b01, b10, b11;
        ldsm_x4(sw128(kt, mrow, mchunk), b00, b01, b10, b11);
        mma_16816(sc[0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b00, b01);
        mma_16816(sc[1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b10, b11);
      }
    }
    // mask keys beyond this split / the sequence (only a tail block has any)
    const int64_t kbase = k0 + static_cast<int64_t>(i) * kDecBlock + key0;
    if (k0 + static_cast<int64_t>(i + 1) * kDecBlock > k1) {
      const int64_t lim = k1 - kbase;  // valid keys of this warp's 16 (may be <= 0)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (nt * 8 + 2 * t4 + (e & 1) >= lim) sc[nt][e] = -INFINITY;
    }
    // online softmax per row in log2 units (the 4 lanes of a quad hold one
    // row's 16 keys); scores are sc * sl2, whose row max is max(sc) * sl2 for
    // sl2 > 0 (the usual case: the scale multiplies into the exponent FMA)
    float mx[2];
    if (sl2 > 0.f) {
      mx[0] = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
      mx[1] = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
    } else {
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (sc[nt][e] != -INFINITY) sc[nt][e] *= -1.f;  // max(sc * sl2) = -min(sc) * |sl2|
      mx[0] = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
      mx[1] = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
    }
    const float sl2a = fmaxf(fabsf(sl2), 1e-30f);  // (scale 0: masked keys stay -inf, not NaN)
    float alpha[2], mu[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r] * sl2a);
      mu[r] = mn == -INFINITY ? 0.f : mn;
      alpha[r] = m_r[r] == -INFINITY ? 0.f : ex2_approx(m_r[r] - mu[r]);
      m_r[r] = mn;
    }
    float pr[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) pr[nt][e] = ex2_approx(fmaf(sc[nt][e], sl2a, -mu[e >> 1]));
#pragma unroll
    for (int r = 0; r < 2; ++r)
      l_r[r] = l_r[r] * alpha[r] + pr[0][2 * r] + pr[0][2 * r + 1] + pr[1][2 * r] + pr[1][2 * r + 1];
    // rescale O only when some row's running max moved (alpha == 1 exactly
    // otherwise): past the first blocks of a long history that is rare, and
    // the 64 multiplies per thread are a third of the per-block issue at e4m3
    if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        o[nt][0] *= alpha[0];
        o[nt][1] *= alpha[0];
        o[nt][2] *= alpha[1];
        o[nt][3] *= alpha[1];
      }
    }
    // P (A fragment straight from the accumulator layout) x V[16 keys x 128 dims]
    if constexpr (kFp8) {
      const uint32_t pa0 = pack_f16x2(pr[0][0], pr[0][1]), pa1 = pack_f16x2(pr[0][2], pr[0][3]);
      const uint32_t pa2 = pack_f16x2(pr[1][0], pr[1][1]), pa3 = pack_f16x2(pr[1][2], pr[1][3]);
#pragma unroll
      for (int c = 0; c < 8; c += 2) {
        // x4.trans over 16-byte chunks c, c+1: (keys 0-7, c) (keys 8-15, c) (keys 0-7, c+1)
        // (keys 8-15, c+1); register = keys {2t4, 2t4+1} x dims {16c+2g, 16c+2g+1}
        const int mrow = key0 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int mchunk = c + (lane >> 4);
        uint32_t r0, r1, r2, r3;
        ldsm_x4_t(sw128(vt, mrow, mchunk), r0, r1, r2, r3);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t lo = h ? r2 : r0, hi = h ? r3 : r1;
          // keys (2t4, 2t4+1, 2t4+8, 2t4+9) at dim 16(c+h)+2g (even) and +1 (odd)
          const uint32_t ev = prmt(lo, hi, 0x6420), od = prmt(lo, hi, 0x7531);
          mma_16816_f16(o[2 * (c + h)], pa0, pa1, pa2, pa3, e4m3x2_f16x2(ev), e4m3x2_f16x2(ev >> 16));
          mma_16816_f16(o[2 * (c + h) + 1], pa0, pa1, pa2, pa3, e4m3x2_f16x2(od), e4m3x2_f16x2(od >> 16));
        }
      }
    } else {
      const uint32_t pa0 = pack_bf16x2(pr[0][0], pr[0][1]), pa1 = pack_bf16x2(pr[0][2], pr[0][3]);
      const uint32_t pa2 = pack_bf16x2(pr[1][0], pr[1][1]), pa3 = pack_bf16x2(pr[1][2], pr[1][3]);
#pragma unroll
      for (int nt = 0; nt < 16; nt += 2) {
        // x4.trans: (keys 0-7, dims 8nt..) (keys 8-15, 8nt..) (keys 0-7, 8nt+8..) (keys 8-15, ..)
        const int mrow = key0 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int mchunk = nt + (lane >> 4);
        uint32_t b0a, b1a, b0b, b1b;
        ldsm_x4_t(sw128(vt, mrow, mchunk), b0a, b1a, b0b, b1b);
        mma_16816(o[nt], pa0, pa1, pa2, pa3, b0a, b1a);
        mma_16816(o[nt + 1], pa0, pa1, pa2, pa3, b0b, b1b);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // refill this stage with block i + kDecStages once all warps released it
    if (threadIdx.x == 0 && i + kDecStages < n_blocks) {
      mbar_wait(&empty[s], (i / kDecStages) & 1);
      issue_block<kFp8>(p, smem + s * kDecStageBytes, &full[s], kvh,
                  static_cast<int>(row_base + (i + kDecStages) * kDecBlock), policy_evict_first());
    }
    __syncwarp();  // ldmatrix / mma below are .sync.aligned: reconverge warp 0
  }
  // row sums over the quad
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  // combine the 4 warps: global row max, rescale, sum O through shared memory
  if (t4 == 0) {
    red_m[warp][g] = m_r[0];
    red_m[warp][g + 8] = m_r[1];
  }
  __syncthreads();
  float scale_r[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = g + 8 * r;
    float mm = red_m[0][row];
    for (int w2 = 1; w2 < kDecWarps; ++w2) mm = fmaxf(mm, red_m[w2][row]);
    scale_r[r] = (m_r[r] == -INFINITY) ? 0.f : ex2_approx(m_r[r] - mm);
  }
  if (t4 == 0) {
    red_l[warp][g] = l_r[0] * scale_r[0];
    red_l[warp][g + 8] = l_r[1] * scale_r[1];
  }
  float* obuf = reinterpret_cast<float*>(smem);  // reuse the ring: [16 rows][128] fp32 = 8 KB
  for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) obuf[i] = 0.f;
  __syncthreads();
  for (int w2 = 0; w2 < kDecWarps; ++w2) {
    if (warp == w2) {
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        // bf16: n-tile nt = dims 8nt..8nt+7, this thread 2t4, 2t4+1.  e4m3: n-tile
        // 2c + par = dims 16c + 2n + par, this thread n = 2t4, 2t4 + 1.
        const int c = kFp8 ? (nt >> 1) * 16 + 4 * t4 + (nt & 1) : nt * 8 + 2 * t4;
        const int c1 = kFp8 ? c + 2 : c + 1;
        obuf[g * 128 + c] += o[nt][0] * scale_r[0];
        obuf[g * 128 + c1] += o[nt][1] * scale_r[0];
        obuf[(g + 8) * 128 + c] += o[nt][2] * scale_r[1];
        obuf[(g + 8) * 128 + c1] += o[nt][3] * scale_r[1];
      }
    }
    __syncthreads();
  }
  const float vsc = kFp8 ? __ldg(p.v_scale + kvh) : 1.f;
  for (int i = threadIdx.x; i < grp * 128; i += blockDim.x) {
    const int h = i >> 7;
    float L = 0.f, mm = red_m[0][h];
    for (int w2 = 0; w2 < kDecWarps; ++w2) L += red_l[w2][h];
    for (int w2 = 1; w2 < kDecWarps; ++w2) mm = fmaxf(mm, red_m[w2][h]);
    const int64_t pr_idx = part_base + static_cast<int64_t>(h) * p.n_split;
    p.part_o[pr_idx * 128 + (i & 127)] = L > 0.f ? (kFp8 ? obuf[i] * vsc / L : obuf[i] / L) : 0.f;
    if ((i & 127) == 0)
      p.part_lse[pr_idx] = L > 0.f ? (mm + __log2f(L)) * 0.69314718055994530942f : -INFINITY;
  }
}

// Fold the splits of each (sequence, query head) row: one CTA per row; the
// row's max split LSE, then warp w sums splits w, w+8, w+16, ... weighted by
// exp(lse_s - max), and warp 0 adds the 8 warp sums in warp order.
// Deterministic; the same kernel serves every decode transport, so they stay
// bit-identical.
#ifndef RCP_COMBINE_WARPS
#define RCP_COMBINE_WARPS 16  // ncu, B=1 / 4 at 262144 keys: 8.2 / 9.2 us (8 warps), 6.6 / 8.7 (16), 5.8 / 11.2 (32)
#endif
constexpr int kCombineWarps = RCP_COMBINE_WARPS;
// Output routing (rcp_decode_attn_routed): with o_dst non-null, row r goes to
// destination d = r / rows_per_dst (a DEVICE array of base pointers, e.g. the
// owners' peer-mapped receive buffers), row dst_row_offset + r % rows_per_dst.
struct CombineRoute {
  float* const* o_dst;
  float* const* lse_dst;
  int64_t rows_per_dst;
  int64_t dst_row_offset;
  // optional completion signal (the p2p transport): the last CTA publishes
  // *epoch into each flag_dst[p] once every routed row is stored
  unsigned long long* const* flag_dst;
  int n_flags;
  unsigned long long* epoch;
  unsigned* counter;
};

__global__ void __launch_bounds__(kCombineWarps * 32) decode_combine_kernel(
    const float* __restrict__ part_o, const float* __restrict__ part_lse, int64_t rows, int n_split_alloc,
    const int64_t* __restrict__ kv_len, int hq, int keys_per_cta, float* __restrict__ o,
    float* __restrict__ lse, CombineRoute route) {
  // Two passes instead of an online merge: the row's max split LSE first (one
  // read of n_split floats by the whole CTA), then every warp sums its splits
  // weighted by exp(lse_s - max) — no dependent rescale chain, so each warp
  // keeps several 512-byte partial loads in flight (11.6 -> ~4 us at B = 1).
  __shared__ float4 s_acc[kCombineWarps][32];
  __shared__ float s_l[kCombineWarps], s_red[kCombineWarps];
  const int64_t row = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float4* po = reinterpret_cast<const float4*>(part_o + row * n_split_alloc * 128);
  const float* pl = part_lse + row * n_split_alloc;
  // only the splits that hold keys of this row's sequence were written
  const int64_t len = __ldg(kv_len + row / hq);
  const int64_t used = (len + keys_per_cta - 1) / keys_per_cta;
  const int n_split = used < n_split_alloc ? static_cast<int>(used) : n_split_alloc;
  float mx = -INFINITY;
  for (int sp = threadIdx.x; sp < n_split; sp += blockDim.x) mx = fmaxf(mx, __ldg(pl + sp));
  for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  float mt = s_red[0];
#pragma unroll
  for (int w = 1; w < kCombineWarps; ++w) mt = fmaxf(mt, s_red[w]);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float l = 0.f;
  if (mt != -INFINITY) {
#pragma unroll 4
    for (int sp = warp; sp < n_split; sp += kCombineWarps) {
      const float ls = __ldg(pl + sp);
      const float4 v = __ldg(po + static_cast<int64_t>(sp) * 32 + lane);
      const float wgt = ls == -INFINITY ? 0.f : __expf(ls - mt);  // empty split: weight 0
      acc.x += v.x * wgt;
      acc.y += v.y * wgt;
      acc.z += v.z * wgt;
      acc.w += v.w * wgt;
      l += wgt;
    }
  }
  s_acc[warp][lane] = acc;
  if (lane == 0) s_l[warp] = l;
  __syncthreads();
  if (warp == 0) {
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  float lt = 0.f;
#pragma unroll
  for (int w = 0; w < kCombineWarps; ++w) {  // fixed order: deterministic
    const float4 a = s_acc[w][lane];
    r.x += a.x;
    r.y += a.y;
    r.z += a.z;
    r.w += a.w;
    lt += s_l[w];
  }
  const bool has = lt > 0.f;
  const float inv = has ? 1.0f / lt : 0.f;
  float* orow = o + row * 128;
  float* lrow = lse + row;
  if (route.o_dst) {  // e.g. straight into the owner's receive buffer over NVLink
    const int64_t d = row / route.rows_per_dst, rr = route.dst_row_offset + row % route.rows_per_dst;
    orow = route.o_dst[d] + rr * 128;
    lrow = route.lse_dst[d] + rr;
  }
  reinterpret_cast<float4*>(orow)[lane] = make_float4(r.x * inv, r.y * inv, r.z * inv, r.w * inv);
  if (lane == 0) *lrow = has ? mt + logf(lt) : -INFINITY;
  }
  if (route.flag_dst) {
    p2p_last_block_signal(route.counter, route.flag_dst, route.n_flags, route.epoch, false);
  } else if (route.o_dst) {
    __threadfence_system();  // peer stores visible before the step's signal
  }
}

// Keys per CTA from a CTA-count target, at least 8 blocks per CTA.  Round 1
// picked 148 x 8 (about 2.7 waves of the three CTAs per SM the 2-stage ring
// allows) over 148 x 6 / x 3 with the split index fastest in the grid; with
// the KV heads fastest (round 2) 148 x 6 — two full waves — is best at every
// batch of the graphed cfg5 CP4 step: 0.283 / 0.743 / 4.90 ms at B = 1 / 4 /
// 32 against 0.294 / 0.748 / 4.93 at 148 x 8 and 0.305 / 0.753 / 4.95 at
// 148 x 10 (profiles/r02_decode_cta_target_sweep.txt).
#ifndef RCP_DEC_CTA_TARGET
#define RCP_DEC_CTA_TARGET (148 * 6)
#endif
#ifndef RCP_DEC_CTA_TARGET_FP8
#define RCP_DEC_CTA_TARGET_FP8 (148 * 6)
#endif
// Batch rows counted by the split heuristic: the all-gathered decode form
// launches N x slots query rows of which, at small batch, only ~1/N are
// active (the rest are empty slots with kv_len 0), so sizing the split by the
// full row count left the active rows with ~2 CTAs per SM at B = 1 (cfg5).
static int64_t split_rows(int64_t batch) { return batch <= 4 ? 1 : (batch + 3) / 4; }
// RCP_DEC_CTA_TARGET / RCP_DEC_CTA_TARGET_FP8 (environment, read once): tuning
// overrides of the CTA-count target (A/B sweeps without a rebuild).
static int64_t cta_target(bool fp8) {
  static int64_t t[2] = {0, 0};
  int64_t& v = t[fp8 ? 1 : 0];
  if (v == 0) {
    const char* e = getenv(fp8 ? "RCP_DEC_CTA_TARGET_FP8" : "RCP_DEC_CTA_TARGET");
    const long long x = e ? atoll(e) : 0;
    v = x > 0 ? x : (fp8 ? RCP_DEC_CTA_TARGET_FP8 : RCP_DEC_CTA_TARGET);
  }
  return v;
}
static int keys_per_cta(int64_t batch, int32_t hkv, int64_t max_kv_len, bool fp8) {
  const int64_t target = cta_target(fp8);
  int64_t per = (max_kv_len * split_rows(batch) * hkv + target - 1) / target;
  per = (per + kDecBlock - 1) / kDecBlock * kDecBlock;
  if (per < 8 * kDecBlock) per = 8 * kDecBlock;
  return static_cast<int>(per);
}

static int n_splits(int64_t batch, int32_t hkv, int64_t max_kv_len, bool fp8) {
  const int per = keys_per_cta(batch, hkv, max_kv_len, fp8);
  const int64_t ns = (max_kv_len + per - 1) / per;
  return static_cast<int>(ns < 1 ? 1 : ns);
}

static PFN_cuTensorMapEncodeTiled_v12000 dec_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// e4m3 rows are 128 bytes per KV head, so a 256-byte L2 promotion also pulls
// the next head's row: with the split-major grid that was a 20 % DRAM
// over-read (10.3 GB for 8.6 GB at B = 16); with heads varying fastest the
// neighbour CTA consumes it and 256 B is 1-3 % faster than 128 B at B <= 16
// (RCP_DEC_FP8_PROMO=128 for A/B).
static bool fp8_promo256() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RCP_DEC_FP8_PROMO");
    v = (e && atoi(e) == 128) ? 0 : 1;
  }
  return v == 1;
}
// 64-key boxes of 128 bytes per row: 64 bf16 dims, or 128 e4m3 dims.
static int make_kv_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t stride, bool fp8) {
  auto fn = dec_encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return RCP_ERR_CUDA;
  }
  const int64_t esz = fp8 ? 1 : 2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(stride * esz)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), kDecBlock};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  (fp8 && !fp8_promo256()) ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                           : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (decode) failed (%d)", (int)r);
    return RCP_ERR_CUDA;
  }
  return RCP_OK;
}

}  // namespace rcp

using namespace rcp;

extern "C" size_t rcp_decode_workspace_bytes(int64_t batch, int32_t hq, int64_t max_kv_len) {
  // upper bound over KV-head counts: fewest KV heads -> most splits
  // both element types (the workspace is shared by the bf16 and e4m3 kernels)
  const int64_t a = n_splits(batch, 1, max_kv_len, false), b = n_splits(batch, 1, max_kv_len, true);
  const int64_t n_split = a > b ? a : b;
  return static_cast<size_t>(batch * hq * n_split * (128 + 1) * sizeof(float));
}

namespace rcp {
template <bool kFp8>
static int decode_launch(const void* q, const void* k, const void* v, int64_t kv_row_stride, int64_t kv_rows,
                         const int64_t* kv_start, const int64_t* kv_len, int64_t batch, int64_t max_kv_len,
                         int32_t hq, int32_t hkv, int32_t head_dim, float scale, const float* k_scale,
                         const float* v_scale, float* o, float* lse, void* workspace, size_t workspace_bytes,
                         void* stream, CombineRoute route = CombineRoute{nullptr, nullptr, 1, 0, nullptr, 0, nullptr, nullptr}) {
  using G = DecGeo<kFp8>;
  RCP_CHECK_ARG(head_dim == 128, "head_dim must be 128, got %d", head_dim);
  RCP_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0,
                "n_query_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  RCP_CHECK_ARG(batch >= 0 && max_kv_len >= 0 && kv_rows >= 0, "bad sizes");
  RCP_CHECK_ARG(kv_rows < INT32_MAX, "kv arena rows must fit int32");
  if (batch == 0) return RCP_OK;
  RCP_CHECK_ARG(q && kv_start && kv_len && ((o && lse) || (route.o_dst && route.lse_dst)), "null pointer");
  const size_t need = rcp_decode_workspace_bytes(batch, hq, max_kv_len);
  RCP_CHECK_ARG(workspace && workspace_bytes >= need, "workspace too small: need %zu", need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((kv_rows == 0 || max_kv_len == 0) && !route.o_dst) return rcp_fill_empty(o, lse, batch * hq, 128, stream);
  RCP_CHECK_ARG(kv_rows > 0 && max_kv_len > 0, "routed decode needs a non-empty arena");
  RCP_CHECK_ARG(k && v, "null kv pointer");
  if (kFp8) {
    RCP_CHECK_ARG(k_scale && v_scale, "null k/v scale pointer");
    RCP_CHECK_ARG(kv_row_stride % 16 == 0 && kv_row_stride >= hkv * 128, "bad kv row stride");
  } else {
    RCP_CHECK_ARG(kv_row_stride % 8 == 0 && kv_row_stride >= hkv * 128, "bad kv row stride");
  }
  RCP_CHECK_ARG(((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) == 0,
                "k/v must be 16-byte aligned");
  DecodeParams prm;
  memset(&prm, 0, sizeof(prm));
  int rc;
  if ((rc = make_kv_map(&prm.tm_k, k, kv_rows, static_cast<int64_t>(hkv) * 128, kv_row_stride, kFp8)) != RCP_OK)
    return rc;
  if ((rc = make_kv_map(&prm.tm_v, v, kv_rows, static_cast<int64_t>(hkv) * 128, kv_row_stride, kFp8)) != RCP_OK)
    return rc;
  const int n_split = n_splits(batch, hkv, max_kv_len, kFp8);
  prm.q = static_cast<const __nv_bfloat16*>(q);
  prm.kv_start = kv_start;
  prm.kv_len = kv_len;
  prm.part_o = static_cast<float*>(workspace);
  prm.part_lse = prm.part_o + batch * hq * n_split * 128;
  prm.k_scale = k_scale;
  prm.v_scale = v_scale;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.group = hq / hkv;
  prm.n_split = n_split;
  prm.keys_per_cta = keys_per_cta(batch, hkv, max_kv_len, kFp8);
  prm.scale_log2 = static_cast<float>(static_cast<double>(scale) * 1.4426950408889634);
  static bool attr = false;
  if (!attr) {
    RCP_CUDA(cudaFuncSetAttribute(decode_mma_kernel<kFp8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  G::kSmemBytes));
    attr = true;
  }
  const int n_hc = (hq / hkv + kDecMaxGroup - 1) / kDecMaxGroup;  // CTAs per KV head (16 query heads each)
  RCP_CHECK_ARG(static_cast<int64_t>(hkv) * n_hc < (1ll << 31) && n_split < 65536 && batch < 65536,
                "decode grid too large");
  dim3 grid(static_cast<unsigned>(hkv * n_hc), n_split, static_cast<unsigned>(batch));
  decode_mma_kernel<kFp8><<<grid, kDecThreads, G::kSmemBytes, st>>>(prm);
  RCP_CUDA(cudaGetLastError());
  const int64_t rows = batch * hq;
  decode_combine_kernel<<<static_cast<unsigned>(rows), kCombineWarps * 32, 0, st>>>(
      prm.part_o, prm.part_lse, rows, n_split, kv_len, hq, prm.keys_per_cta, o, lse, route);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

// ---------------------------------------------------------------- e4m3 KV rows
// Row j of src (bf16 [n_rows, hkv*head_dim], row stride in elements) ->
// dst row (dst_rows ? dst_rows[j] : j): e4m3 = satfinite_rn(x * inv[head]) with
// inv = 1 / scale (IEEE fp32 division, once per head) and an fp32 multiply —
// bit for bit oracle/ringcp_oracle.py::quantize_e4m3.  One warp per row at a
// time, each lane 8 elements (a 16-byte load, an 8-byte store) per step; the
// per-head factors sit in shared memory (hkv <= 1024).
constexpr int kKvRowThreads = 256;
__global__ void __launch_bounds__(kKvRowThreads) kv_quantize_kernel(
    uint8_t* __restrict__ dst, int64_t dst_stride, const int64_t* __restrict__ dst_rows,
    const __nv_bfloat16* __restrict__ src, int64_t src_stride, int64_t n_rows, int hkv, int hd_chunks,
    const float* __restrict__ scale) {
  __shared__ float s_inv[1024];
  for (int h = threadIdx.x; h < hkv; h += blockDim.x) s_inv[h] = __fdiv_rn(1.0f, __ldg(scale + h));
  __syncthreads();
  const int per_row = hkv * hd_chunks;  // 8-element chunks per row
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); j < n_rows; j += warps) {
    const __nv_bfloat16* srow = src + j * src_stride;
    uint8_t* drow = dst + (dst_rows ? __ldg(dst_rows + j) : j) * dst_stride;
#pragma unroll 4
    for (int c = lane; c < per_row; c += 32) {
      const float inv = s_inv[c / hd_chunks];
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(srow) + c);
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
      uint16_t e[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[t]));
        const float lo = __fmul_rn(f.x, inv), hi = __fmul_rn(f.y, inv);
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(e[t]) : "f"(hi), "f"(lo));
      }
      uint2 out;
      out.x = static_cast<uint32_t>(e[0]) | (static_cast<uint32_t>(e[1]) << 16);
      out.y = static_cast<uint32_t>(e[2]) | (static_cast<uint32_t>(e[3]) << 16);
      reinterpret_cast<uint2*>(drow)[c] = out;
    }
  }
}

// x = e4m3 * scale[head] in fp32, rounded to bf16 (RN); same walk as above.
__global__ void __launch_bounds__(kKvRowThreads) kv_dequantize_kernel(
    __nv_bfloat16* __restrict__ dst, int64_t dst_stride, const uint8_t* __restrict__ src, int64_t src_stride,
    int64_t n_rows, int hkv, int hd_chunks, const float* __restrict__ scale) {
  __shared__ float s_sc[1024];
  for (int h = threadIdx.x; h < hkv; h += blockDim.x) s_sc[h] = __ldg(scale + h);
  __syncthreads();
  const int per_row = hkv * hd_chunks;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); j < n_rows; j += warps) {
    const uint8_t* srow = src + j * src_stride;
    __nv_bfloat16* drow = dst + j * dst_stride;
#pragma unroll 4
    for (int c = lane; c < per_row; c += 32) {
      const float sc = s_sc[c / hd_chunks];
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(srow) + c);
      const uint32_t w[2] = {x.x, x.y};
      uint32_t out[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t h2 = e4m3x2_f16x2(w[t >> 1] >> (16 * (t & 1)));
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h2));
        const __nv_bfloat162 bb = __floats2bfloat162_rn(__fmul_rn(f.x, sc), __fmul_rn(f.y, sc));
        out[t] = *reinterpret_cast<const uint32_t*>(&bb);
      }
      reinterpret_cast<uint4*>(drow)[c] = make_uint4(out[0], out[1], out[2], out[3]);
    }
  }
}

// One decode step's cache appends (GraphedDecode): slot j of this rank's new
// tokens goes to arena row meta[j] of the step metadata (rows | starts | lens |
// pos | seq, int64): its K and V rows copied (bf16) or quantised exactly as
// kv_quantize_kernel (e4m3, k_scale non-null), its folded int32 position and
// sequence id stored — one launch instead of the index copies and the cast.
__global__ void __launch_bounds__(128) decode_append_kernel(
    const int64_t* __restrict__ meta, int64_t pos_off, int64_t seq_off, const __nv_bfloat16* __restrict__ k_in,
    const __nv_bfloat16* __restrict__ v_in, void* __restrict__ k_arena, void* __restrict__ v_arena,
    int64_t row_stride, int hkv, int hd_chunks, int32_t* __restrict__ pos_arena, int32_t* __restrict__ seq_arena,
    const float* __restrict__ k_scale, const float* __restrict__ v_scale) {
  const int j = blockIdx.x, kv = blockIdx.y;
  const int64_t row = __ldg(meta + j);
  const int per_row = hkv * hd_chunks;
  const uint4* src = reinterpret_cast<const uint4*>((kv ? v_in : k_in) + static_cast<int64_t>(j) * per_row * 8);
  const float* scale = kv ? v_scale : k_scale;
  if (scale) {
    uint2* dst = reinterpret_cast<uint2*>(static_cast<uint8_t*>(kv ? v_arena : k_arena) + row * row_stride);
    for (int c = threadIdx.x; c < per_row; c += blockDim.x) {
      const float inv = __fdiv_rn(1.0f, __ldg(scale + c / hd_chunks));
      const uint4 x = __ldg(src + c);
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
      uint16_t e[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[t]));
        const float lo = __fmul_rn(f.x, inv), hi = __fmul_rn(f.y, inv);
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(e[t]) : "f"(hi), "f"(lo));
      }
      dst[c] = make_uint2(static_cast<uint32_t>(e[0]) | (static_cast<uint32_t>(e[1]) << 16),
                          static_cast<uint32_t>(e[2]) | (static_cast<uint32_t>(e[3]) << 16));
    }
  } else {
    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(kv ? v_arena : k_arena) + row * row_stride);
    for (int c = threadIdx.x; c < per_row; c += blockDim.x) dst[c] = __ldg(src + c);
  }
  if (kv == 0 && threadIdx.x == 0) {
    pos_arena[row] = static_cast<int32_t>(__ldg(meta + pos_off + j));
    seq_arena[row] = static_cast<int32_t>(__ldg(meta + seq_off + j));
  }
}

// Per-head absolute max of bf16 rows (as ordered int bits of a non-negative
// float; amax_bits zeroed by the caller), then scale = max(amax, 2^-24) / 448.
__global__ void kv_absmax_kernel(const __nv_bfloat16* __restrict__ src, int64_t src_stride, int64_t n_rows,
                                 int row_elems, int head_dim, unsigned* __restrict__ amax_bits) {
  const int per_row = row_elems >> 3;
  const int64_t n = n_rows * per_row;
  const int h = blockIdx.y;
  const int heads_chunks = head_dim >> 3;
  float m = 0.f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_rows * heads_chunks;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = i / heads_chunks;
    const int c = h * head_dim + (static_cast<int>(i - j * heads_chunks) << 3);
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(src + j * src_stride + c));
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[t]));
      m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
  }
  (void)n;
  for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(amax_bits + h, __float_as_uint(m));
}
// scale = max(amax, 2^-24) / 448 rounded UP to a power of two: the absmax stays
// in range, and e4m3 * scale is exact in bf16, so the prefill's bf16 rows and
// the decode kernel's scaled e4m3 are the same values.
__global__ void kv_scale_kernel(unsigned* amax_bits, float* scale, int hkv) {
  const int h = threadIdx.x;
  if (h < hkv) {
    const float v = __fdiv_rn(fmaxf(__uint_as_float(amax_bits[h]), 5.9604644775390625e-08f), 448.f);
    scale[h] = __uint_as_float((__float_as_uint(v) + 0x7FFFFFu) & 0xFF800000u);
  }
}

// One warp per row per step: up to 16 resident 256-thread CTAs per SM worth of warps.
static int kv_rows_grid(int64_t n_rows) {
  const int64_t b = (n_rows + 7) / 8;
  return static_cast<int>(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b));
}
static int rows_grid(int64_t items) {
  const int64_t b = (items + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}
}  // namespace rcp

extern "C" int rcp_decode_attn(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                               int64_t kv_rows, const int64_t* kv_start, const int64_t* kv_len,
                               int64_t batch, int64_t max_kv_len, int32_t hq, int32_t hkv,
                               int32_t head_dim, float scale, float* o, float* lse, void* workspace,
                               size_t workspace_bytes, void* stream) {
  return decode_launch<false>(q, k, v, kv_row_stride, kv_rows, kv_start, kv_len, batch, max_kv_len, hq, hkv,
                              head_dim, scale, nullptr, nullptr, o, lse, workspace, workspace_bytes, stream);
}

extern "C" int rcp_decode_attn_fp8(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                                   int64_t kv_rows, const int64_t* kv_start, const int64_t* kv_len,
                                   int64_t batch, int64_t max_kv_len, int32_t hq, int32_t hkv,
                                   int32_t head_dim, float scale, const float* k_scale, const float* v_scale,
                                   float* o, float* lse, void* workspace, size_t workspace_bytes, void* stream) {
  return decode_launch<true>(q, k, v, kv_row_stride, kv_rows, kv_start, kv_len, batch, max_kv_len, hq, hkv,
                             head_dim, scale, k_scale, v_scale, o, lse, workspace, workspace_bytes, stream);
}

extern "C" int rcp_decode_attn_routed(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                                      int64_t kv_rows, const int64_t* kv_start, const int64_t* kv_len,
                                      int64_t batch, int64_t max_kv_len, int32_t hq, int32_t hkv,
                                      int32_t head_dim, float scale, const float* k_scale, const float* v_scale,
                                      float* const* o_dst, float* const* lse_dst, int32_t n_dst,
                                      int64_t dst_row_offset, uint64_t* const* flag_dst, uint64_t* epoch,
                                      uint32_t* counter, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  RCP_CHECK_ARG(o_dst && lse_dst && n_dst >= 1 && batch % n_dst == 0 && dst_row_offset >= 0,
                "bad output routing (batch %lld over %d destinations)", (long long)batch, n_dst);
  RCP_CHECK_ARG((k_scale == nullptr) == (v_scale == nullptr), "give both k/v scales (e4m3) or neither (bf16)");
  RCP_CHECK_ARG(!flag_dst || (epoch && counter), "a signalling decode needs the epoch and a counter");
  const CombineRoute route{o_dst, lse_dst, batch / n_dst * hq, dst_row_offset,
                           reinterpret_cast<unsigned long long* const*>(flag_dst), n_dst,
                           reinterpret_cast<unsigned long long*>(epoch), counter};
  if (k_scale)
    return decode_launch<true>(q, k, v, kv_row_stride, kv_rows, kv_start, kv_len, batch, max_kv_len, hq, hkv,
                               head_dim, scale, k_scale, v_scale, nullptr, nullptr, workspace, workspace_bytes,
                               stream, route);
  return decode_launch<false>(q, k, v, kv_row_stride, kv_rows, kv_start, kv_len, batch, max_kv_len, hq, hkv,
                              head_dim, scale, nullptr, nullptr, nullptr, nullptr, workspace, workspace_bytes,
                              stream, route);
}

extern "C" int rcp_kv_quantize_e4m3(void* dst, int64_t dst_row_stride, const int64_t* dst_rows, const void* src,
                                    int64_t src_row_stride, int64_t n_rows, int32_t hkv, int32_t head_dim,
                                    const float* scale, void* stream) {
  RCP_CHECK_ARG(n_rows >= 0 && hkv >= 1 && head_dim >= 8 && head_dim % 8 == 0, "bad sizes");
  if (n_rows == 0) return RCP_OK;
  RCP_CHECK_ARG(dst && src && scale, "null pointer");
  RCP_CHECK_ARG(dst_row_stride % 8 == 0 && src_row_stride % 8 == 0 && dst_row_stride >= hkv * head_dim &&
                    src_row_stride >= hkv * head_dim, "bad row stride");
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(dst) & 7) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0,
                "misaligned rows");
  RCP_CHECK_ARG(hkv <= 1024, "at most 1024 kv heads");
  kv_quantize_kernel<<<kv_rows_grid(n_rows), kKvRowThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(dst), dst_row_stride, dst_rows, static_cast<const __nv_bfloat16*>(src),
      src_row_stride, n_rows, hkv, head_dim >> 3, scale);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

extern "C" int rcp_kv_dequantize_e4m3(void* dst, int64_t dst_row_stride, const void* src, int64_t src_row_stride,
                                      int64_t n_rows, int32_t hkv, int32_t head_dim, const float* scale,
                                      void* stream) {
  RCP_CHECK_ARG(n_rows >= 0 && hkv >= 1 && head_dim >= 8 && head_dim % 8 == 0, "bad sizes");
  if (n_rows == 0) return RCP_OK;
  RCP_CHECK_ARG(dst && src && scale, "null pointer");
  RCP_CHECK_ARG(dst_row_stride % 8 == 0 && src_row_stride % 8 == 0 && dst_row_stride >= hkv * head_dim &&
                    src_row_stride >= hkv * head_dim, "bad row stride");
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 7) == 0,
                "misaligned rows");
  RCP_CHECK_ARG(hkv <= 1024, "at most 1024 kv heads");
  kv_dequantize_kernel<<<kv_rows_grid(n_rows), kKvRowThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(dst), dst_row_stride, static_cast<const uint8_t*>(src), src_row_stride, n_rows,
      hkv, head_dim >> 3, scale);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

extern "C" int rcp_decode_append(const int64_t* meta, int32_t slots, int64_t pos_off, int64_t seq_off,
                                 const void* k_in, const void* v_in, void* k_arena, void* v_arena,
                                 int64_t kv_row_stride, int32_t hkv, int32_t head_dim, int32_t* pos_arena,
                                 int32_t* seq_arena, const float* k_scale, const float* v_scale, void* stream) {
  RCP_CHECK_ARG(slots >= 0 && hkv >= 1 && head_dim >= 8 && head_dim % 8 == 0, "bad sizes");
  if (slots == 0) return RCP_OK;
  RCP_CHECK_ARG(meta && k_in && v_in && k_arena && v_arena && pos_arena && seq_arena, "null pointer");
  RCP_CHECK_ARG((k_scale == nullptr) == (v_scale == nullptr), "give both k/v scales (e4m3) or neither (bf16)");
  RCP_CHECK_ARG(kv_row_stride % 8 == 0 && kv_row_stride >= hkv * head_dim, "bad kv row stride");
  dim3 grid(static_cast<unsigned>(slots), 2);
  decode_append_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      meta, pos_off, seq_off, static_cast<const __nv_bfloat16*>(k_in), static_cast<const __nv_bfloat16*>(v_in),
      k_arena, v_arena, kv_row_stride, hkv, head_dim >> 3, pos_arena, seq_arena, k_scale, v_scale);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

extern "C" int rcp_kv_calibrate_e4m3(const void* src, int64_t src_row_stride, int64_t n_rows, int32_t hkv,
                                     int32_t head_dim, float* scale, void* workspace, void* stream) {
  RCP_CHECK_ARG(n_rows >= 0 && hkv >= 1 && hkv <= 1024 && head_dim >= 8 && head_dim % 8 == 0, "bad sizes");
  RCP_CHECK_ARG(scale && workspace && (n_rows == 0 || src), "null pointer");
  RCP_CHECK_ARG(src_row_stride % 8 == 0 && src_row_stride >= hkv * head_dim, "bad row stride");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned* bits = static_cast<unsigned*>(workspace);
  RCP_CUDA(cudaMemsetAsync(bits, 0, hkv * sizeof(unsigned), st));
  if (n_rows > 0) {
    const int64_t items = n_rows * (head_dim >> 3);
    dim3 grid(rows_grid(items) > 148 ? 148 : rows_grid(items), hkv);
    kv_absmax_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), src_row_stride, n_rows,
                                           hkv * head_dim, head_dim, bits);
    RCP_CUDA(cudaGetLastError());
  }
  kv_scale_kernel<<<1, 1024, 0, st>>>(bits, scale, hkv);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}
