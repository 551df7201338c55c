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
#include <climits>
#include <cstring>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace rcp {

constexpr int kDecBlock = 64;      // keys per TMA block
#ifndef RCP_DEC_STAGES
#define RCP_DEC_STAGES 2
#endif
// 32 KB (K + V of 64 keys) per stage.  Two stages (65 KB) let three CTAs
// share an SM, so one CTA's pipeline fill and epilogue overlap the others'
// streaming: measured 6.5 TB/s at B=16 and 0.32 ms vs 0.44 ms per graphed
// B=1 step against four stages (one CTA per SM).
constexpr int kDecStages = RCP_DEC_STAGES;
constexpr int kDecWarps = 4;       // 16-key slice of each block per warp
constexpr int kDecThreads = kDecWarps * 32;
constexpr int kDecMaxGroup = 16;   // query heads per KV head (mma M)
constexpr uint32_t kDecBoxBytes = kDecBlock * 64 * 2;   // 8 KB: 64 keys x 64 dims
constexpr uint32_t kDecTileBytes = 2 * kDecBoxBytes;    // 16 KB: 64 keys x 128 dims
constexpr uint32_t kDecStageBytes = 2 * kDecTileBytes;  // K + V
constexpr uint32_t kDecSmemBytes = kDecStages * kDecStageBytes + 1024;

struct DecodeParams {
  CUtensorMap tm_k, tm_v;
  const __nv_bfloat16* q;
  const int64_t* kv_start;
  const int64_t* kv_len;
  float* part_o;
  float* part_lse;
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
// Byte address of 16-byte chunk `chunk` (0..15 over 128 dims) of `row` in a
// 64-row SW128 tile made of two 64-dim boxes (TMA SWIZZLE_128B layout).
__device__ __forceinline__ uint32_t sw128(uint32_t tile, int row, int chunk) {
  return tile + (chunk >> 3) * kDecBoxBytes + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

__device__ __forceinline__ void issue_block(const DecodeParams& p, uint8_t* st, uint64_t* bar,
                                            int kvh, int row, uint64_t pol) {
  mbar_arrive_expect_tx(bar, kDecStageBytes);
  for (int h = 0; h < 2; ++h) {
    tma_load_2d(st + h * kDecBoxBytes, &p.tm_k, bar, kvh * 128 + h * 64, row, pol);
    tma_load_2d(st + kDecTileBytes + h * kDecBoxBytes, &p.tm_v, bar, kvh * 128 + h * 64, row, pol);
  }
}

__global__ void __launch_bounds__(kDecThreads) decode_mma_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kDecStages], empty[kDecStages];
  __shared__ float red_m[kDecWarps][kDecMaxGroup], red_l[kDecWarps][kDecMaxGroup];

  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t len = __ldg(p.kv_len + b);
  const int64_t k0 = static_cast<int64_t>(split) * p.keys_per_cta;
  const int64_t k1 = min(len, k0 + p.keys_per_cta);
  const int n_blocks = k1 > k0 ? static_cast<int>((k1 - k0 + kDecBlock - 1) / kDecBlock) : 0;
  const int row0 = b * p.hq + kvh * p.group;  // first query-head row of this GQA group
  const int64_t part_base = static_cast<int64_t>(row0) * p.n_split + split;

  if (n_blocks == 0) {  // empty split: (0, -inf)
    for (int i = threadIdx.x; i < p.group * 128; i += blockDim.x) {
      const int h = i >> 7;
      p.part_o[(part_base + static_cast<int64_t>(h) * p.n_split) * 128 + (i & 127)] = 0.f;
      if ((i & 127) == 0) p.part_lse[part_base + static_cast<int64_t>(h) * p.n_split] = -INFINITY;
    }
    return;
  }
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
      issue_block(p, smem + i * kDecStageBytes, &full[i], kvh,
                  static_cast<int>(row_base + i * kDecBlock), pol);
  }
  // Q fragments (A operand, rows = query heads of the group, zero-padded to 16)
  uint32_t qa[8][4];
  {
    const __nv_bfloat16* q0 = p.q + static_cast<int64_t>(row0) * 128;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int c = ks * 16 + 2 * t4;
      qa[ks][0] = g < p.group ? *reinterpret_cast<const uint32_t*>(q0 + g * 128 + c) : 0u;
      qa[ks][1] = g + 8 < p.group ? *reinterpret_cast<const uint32_t*>(q0 + (g + 8) * 128 + c) : 0u;
      qa[ks][2] = g < p.group ? *reinterpret_cast<const uint32_t*>(q0 + g * 128 + c + 8) : 0u;
      qa[ks][3] = g + 8 < p.group ? *reinterpret_cast<const uint32_t*>(q0 + (g + 8) * 128 + c + 8) : 0u;
    }
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};  // rows g, g+8
  const float sl2 = p.scale_log2;
  const uint32_t smem_base = smem_u32(smem);
  const int key0 = warp * 16;  // this warp's 16 keys of every block

  for (int i = 0; i < n_blocks; ++i) {
    const int s = i % kDecStages;
    mbar_wait(&full[s], (i / kDecStages) & 1);
    const uint32_t kt = smem_base + s * kDecStageBytes, vt = kt + kDecTileBytes;
    // S[16 heads x 16 keys] = Q K^T : two n-tiles of 8 keys, 8 k-steps of 16 dims
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
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
    // scale to log2 units; mask keys beyond this split / the sequence (tail block)
    const int64_t kbase = k0 + static_cast<int64_t>(i) * kDecBlock + key0;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t kk = kbase + nt * 8 + 2 * t4 + (e & 1);
        sc[nt][e] = kk < k1 ? sc[nt][e] * sl2 : -INFINITY;
      }
    // online softmax per row (the 4 lanes of a quad hold one row's 16 keys)
    float mx[2];
    mx[0] = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
    mx[1] = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
    float alpha[2], mu[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r]);
      mu[r] = mn == -INFINITY ? 0.f : mn;
      alpha[r] = m_r[r] == -INFINITY ? 0.f : ex2_approx(m_r[r] - mu[r]);
      m_r[r] = mn;
    }
    float pr[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) pr[nt][e] = ex2_approx(sc[nt][e] - mu[e >> 1]);
#pragma unroll
    for (int r = 0; r < 2; ++r)
      l_r[r] = l_r[r] * alpha[r] + pr[0][2 * r] + pr[0][2 * r + 1] + pr[1][2 * r] + pr[1][2 * r + 1];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      o[nt][0] *= alpha[0];
      o[nt][1] *= alpha[0];
      o[nt][2] *= alpha[1];
      o[nt][3] *= alpha[1];
    }
    // P (bf16 A fragment straight from the accumulator layout) x V[16 keys x 128 dims]
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // refill this stage with block i + kDecStages once all warps released it
    if (threadIdx.x == 0 && i + kDecStages < n_blocks) {
      mbar_wait(&empty[s], (i / kDecStages) & 1);
      issue_block(p, smem + s * kDecStageBytes, &full[s], kvh,
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
        const int c = nt * 8 + 2 * t4;
        obuf[g * 128 + c] += o[nt][0] * scale_r[0];
        obuf[g * 128 + c + 1] += o[nt][1] * scale_r[0];
        obuf[(g + 8) * 128 + c] += o[nt][2] * scale_r[1];
        obuf[(g + 8) * 128 + c + 1] += o[nt][3] * scale_r[1];
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < p.group * 128; i += blockDim.x) {
    const int h = i >> 7;
    float L = 0.f, mm = red_m[0][h];
    for (int w2 = 0; w2 < kDecWarps; ++w2) L += red_l[w2][h];
    for (int w2 = 1; w2 < kDecWarps; ++w2) mm = fmaxf(mm, red_m[w2][h]);
    const int64_t pr_idx = part_base + static_cast<int64_t>(h) * p.n_split;
    p.part_o[pr_idx * 128 + (i & 127)] = L > 0.f ? obuf[i] / L : 0.f;
    if ((i & 127) == 0)
      p.part_lse[pr_idx] = L > 0.f ? (mm + __log2f(L)) * 0.69314718055994530942f : -INFINITY;
  }
}

// Fold the splits of each (sequence, query head) row: one CTA per row, warp w
// online-merges splits w, w+8, w+16, ... (independent loads, so a warp keeps
// several 512-byte partials in flight instead of one dependent chain), then
// warp 0 folds the 8 warp partials in warp order.  Deterministic; the same
// kernel serves every decode transport, so they stay bit-identical.
constexpr int kCombineWarps = 8;
__global__ void __launch_bounds__(kCombineWarps * 32) decode_combine_kernel(
    const float* __restrict__ part_o, const float* __restrict__ part_lse, int64_t rows, int n_split,
    float* __restrict__ o, float* __restrict__ lse) {
  __shared__ float4 s_acc[kCombineWarps][32];
  __shared__ float s_m[kCombineWarps], s_l[kCombineWarps];
  const int64_t row = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float4* po = reinterpret_cast<const float4*>(part_o + row * n_split * 128);
  const float* pl = part_lse + row * n_split;
  float m = -INFINITY, l = 0.f;  // running max / sum of exp(lse_s - m) (natural log)
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int sp = warp; sp < n_split; sp += kCombineWarps) {
    const float ls = __ldg(pl + sp);
    const float4 v = __ldg(po + static_cast<int64_t>(sp) * 32 + lane);
    if (ls == -INFINITY) continue;  // empty split (uniform across the warp)
    const float mn = fmaxf(m, ls);
    const float a = __expf(m - mn), b = __expf(ls - mn);
    acc.x = acc.x * a + v.x * b;
    acc.y = acc.y * a + v.y * b;
    acc.z = acc.z * a + v.z * b;
    acc.w = acc.w * a + v.w * b;
    l = l * a + b;
    m = mn;
  }
  s_acc[warp][lane] = acc;
  if (lane == 0) {
    s_m[warp] = m;
    s_l[warp] = l;
  }
  __syncthreads();
  if (warp != 0) return;
  float mt = -INFINITY;
#pragma unroll
  for (int w = 0; w < kCombineWarps; ++w) mt = fmaxf(mt, s_m[w]);
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  float lt = 0.f;
  if (mt != -INFINITY) {
#pragma unroll
    for (int w = 0; w < kCombineWarps; ++w) {
      if (s_m[w] == -INFINITY) continue;
      const float f = __expf(s_m[w] - mt);
      const float4 a = s_acc[w][lane];
      r.x += a.x * f;
      r.y += a.y * f;
      r.z += a.z * f;
      r.w += a.w * f;
      lt += s_l[w] * f;
    }
  }
  const bool has = lt > 0.f;
  const float inv = has ? 1.0f / lt : 0.f;
  reinterpret_cast<float4*>(o + row * 128)[lane] = make_float4(r.x * inv, r.y * inv, r.z * inv, r.w * inv);
  if (lane == 0) lse[row] = has ? mt + logf(lt) : -INFINITY;
}

// Keys per CTA: about 8 waves of 148 CTAs, at least 8 blocks per CTA.
// CTA-count target of the split heuristic.  148 x 8 (about 2.7 waves of the
// three CTAs per SM the 2-stage ring allows) measured best: 148 x 6 and
// 148 x 3 gave 0.79 / 0.87 ms per graphed B=4 step against 0.755 ms.
// (Round 2: 148 x 9, three full waves of 3 CTAs per SM instead of 2.65, measured
// neutral at B = 1 (0.247 vs 0.245 ms per graphed step) and 2 % slower at B = 4.)
#ifndef RCP_DEC_CTA_TARGET
#define RCP_DEC_CTA_TARGET (148 * 8)
#endif
// Batch rows counted by the split heuristic: the all-gathered decode form
// launches N x slots query rows of which, at small batch, only ~1/N are
// active (the rest are empty slots with kv_len 0), so sizing the split by the
// full row count left the active rows with ~2 CTAs per SM at B = 1 (cfg5).
static int64_t split_rows(int64_t batch) { return batch <= 4 ? 1 : (batch + 3) / 4; }
static int keys_per_cta(int64_t batch, int32_t hkv, int64_t max_kv_len) {
  const int64_t target = RCP_DEC_CTA_TARGET;
  int64_t per = (max_kv_len * split_rows(batch) * hkv + target - 1) / target;
  per = (per + kDecBlock - 1) / kDecBlock * kDecBlock;
  if (per < 8 * kDecBlock) per = 8 * kDecBlock;
  return static_cast<int>(per);
}

static int n_splits(int64_t batch, int32_t hkv, int64_t max_kv_len) {
  const int per = keys_per_cta(batch, hkv, max_kv_len);
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

static int make_kv_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t stride) {
  auto fn = dec_encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return RCP_ERR_CUDA;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(stride) * 2};
  cuuint32_t box[2] = {64, kDecBlock};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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
  const int64_t n_split = n_splits(batch, 1, max_kv_len);
  return static_cast<size_t>(batch * hq * n_split * (128 + 1) * sizeof(float));
}

extern "C" int rcp_decode_attn(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                               int64_t kv_rows, const int64_t* kv_start, const int64_t* kv_len,
                               int64_t batch, int64_t max_kv_len, int32_t hq, int32_t hkv,
                               int32_t head_dim, float scale, float* o, float* lse, void* workspace,
                               size_t workspace_bytes, void* stream) {
  RCP_CHECK_ARG(head_dim == 128, "head_dim must be 128, got %d", head_dim);
  RCP_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0,
                "n_query_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  RCP_CHECK_ARG(hq / hkv <= kDecMaxGroup, "at most %d query heads per kv head", kDecMaxGroup);
  RCP_CHECK_ARG(batch >= 0 && max_kv_len >= 0 && kv_rows >= 0, "bad sizes");
  RCP_CHECK_ARG(kv_rows < INT32_MAX, "kv arena rows must fit int32");
  if (batch == 0) return RCP_OK;
  RCP_CHECK_ARG(q && o && lse && kv_start && kv_len, "null pointer");
  const size_t need = rcp_decode_workspace_bytes(batch, hq, max_kv_len);
  RCP_CHECK_ARG(workspace && workspace_bytes >= need, "workspace too small: need %zu", need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (kv_rows == 0 || max_kv_len == 0) return rcp_fill_empty(o, lse, batch * hq, 128, stream);
  RCP_CHECK_ARG(k && v, "null kv pointer");
  RCP_CHECK_ARG(kv_row_stride % 8 == 0 && kv_row_stride >= hkv * 128, "bad kv row stride");
  RCP_CHECK_ARG(((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) == 0,
                "k/v must be 16-byte aligned");
  DecodeParams prm;
  memset(&prm, 0, sizeof(prm));
  int rc;
  if ((rc = make_kv_map(&prm.tm_k, k, kv_rows, static_cast<int64_t>(hkv) * 128, kv_row_stride)) != RCP_OK)
    return rc;
  if ((rc = make_kv_map(&prm.tm_v, v, kv_rows, static_cast<int64_t>(hkv) * 128, kv_row_stride)) != RCP_OK)
    return rc;
  const int n_split = n_splits(batch, hkv, max_kv_len);
  prm.q = static_cast<const __nv_bfloat16*>(q);
  prm.kv_start = kv_start;
  prm.kv_len = kv_len;
  prm.part_o = static_cast<float*>(workspace);
  prm.part_lse = prm.part_o + batch * hq * n_split * 128;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.group = hq / hkv;
  prm.n_split = n_split;
  prm.keys_per_cta = keys_per_cta(batch, hkv, max_kv_len);
  prm.scale_log2 = static_cast<float>(static_cast<double>(scale) * 1.4426950408889634);
  static bool attr = false;
  if (!attr) {
    RCP_CUDA(cudaFuncSetAttribute(decode_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kDecSmemBytes));
    attr = true;
  }
  dim3 grid(n_split, hkv, static_cast<unsigned>(batch));
  decode_mma_kernel<<<grid, kDecThreads, kDecSmemBytes, st>>>(prm);
  RCP_CUDA(cudaGetLastError());
  const int64_t rows = batch * hq;
  decode_combine_kernel<<<static_cast<unsigned>(rows), kCombineWarps * 32, 0, st>>>(
      prm.part_o, prm.part_lse, rows, n_split, o, lse);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}
