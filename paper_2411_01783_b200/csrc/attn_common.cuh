// Shared pieces of the attention kernels (attn_fwd.cu: active-list pre-pass,
// the 64-key v4 kernel and the C ABI; attn_fwd_n128.cu: the 128-key v12
// kernel): parameters, tile constants, trace macro, tile-summary helpers,
// packed fp32x2 math and the FMA-pipe exp2.
#pragma once

#include <climits>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace rcp {


constexpr int kD = 128;
constexpr int kQRows = 128;        // query tile rows (MMA M)
constexpr int kKRows = 64;         // key block rows  (MMA N of S, K of PV)
#ifndef RCP_KV_SLOTS
#define RCP_KV_SLOTS 8
#endif
constexpr int kSlots = RCP_KV_SLOTS;  // unified K/V TMA ring (K_j, V_j, K_j+1, ...)
constexpr int kThreads = 384;
constexpr uint32_t kQTileBytes = kQRows * kD * 2;   // 32 KB: two 16 KB SW128 boxes
constexpr uint32_t kQBoxBytes = kQTileBytes / 2;
constexpr uint32_t kKVBytes = kKRows * kD * 2;      // 16 KB: two 8 KB SW128 boxes
constexpr uint32_t kKVBoxBytes = kKVBytes / 2;
constexpr uint32_t kSmemBytes = 2 * kQTileBytes + kSlots * kKVBytes + 1024;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr uint32_t kTmemO = 0, kTmemS = 256;  // column bases

struct AttnParams {
  CUtensorMap tm_q, tm_k, tm_v;
  const int32_t* q_pos;
  const int32_t* q_seq;
  const int32_t* k_pos;
  const int32_t* k_seq;
  const TileSum* q_sum;  // per 128-row query tile
  const TileSum* k_sum;  // per 64-row key block
  const uint32_t* act;   // per query-tile pair: active key blocks, j | cls0 << 24 | cls1 << 26
  const int* act_n;      // per query-tile pair: number of active key blocks
  float* o;
  float* lse;
  int tq, tk, hq, hkv, group;
  int n_qtiles, n_qblk, n_kblocks;
  int mode;
  float scale_log2;
  const __nv_bfloat16* q;  // v7: query rows are read directly (into TMEM)
  int64_t q_stride;        // elements between consecutive query rows
  long long* trace;  // RCP_TRACE builds only: per-CTA role timestamps (clock64)
  int* item_ctr;     // v9: work-item counter (workspace, zeroed by active_list_kernel)
  int mask_shift;    // negative-control hook (RCP_FAULT=mask_diag): 1 excludes key == query; else 0
  const float* q_scale;  // e4m3 Q / K form (attn_fwd_qk8.cu): per query head / per KV head
  const float* k_scale;
};

#ifndef RCP_TRACE
#define RCP_TRACE 0
#endif
// Trace layout: CTA b < kTraceCtas, iteration it < kTraceIters, event e < kTraceEv.
constexpr int kTraceCtas = 8, kTraceIters = 64, kTraceEv = 16;
#define TRACE(e, it)                                                                    \
  do {                                                                                  \
    if (RCP_TRACE && p.trace && blockIdx.x < kTraceCtas && (it) < kTraceIters)          \
      p.trace[(blockIdx.x * kTraceIters + (it)) * kTraceEv + (e)] = clock64();          \
  } while (0)

__device__ __forceinline__ TileSum load_sum(const TileSum* p, int i, int n) {
  TileSum t;
  if (i < n) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(p + i));
    const int4 b = __ldg(reinterpret_cast<const int4*>(p + i) + 1);
    t.pmin = a.x; t.pmax = a.y; t.smin = a.z; t.smax = a.w;
    t.nvalid = b.x; t.uniform = b.y; t.pad0 = 0; t.pad1 = 0;
  } else {
    t.pmin = INT_MAX; t.pmax = INT_MIN; t.smin = INT_MAX; t.smax = INT_MIN;
    t.nvalid = 0; t.uniform = 0; t.pad0 = 0; t.pad1 = 0;
  }
  return t;
}

// Active-list entry: key block index and the class of the pair with each query tile.
__device__ __forceinline__ int act_j(uint32_t e) { return static_cast<int>(e & 0xFFFFFFu); }
__device__ __forceinline__ int act_cls(uint32_t e, int t) { return static_cast<int>((e >> (24 + 2 * t)) & 3u); }

// K-major SW128 operand (Q or K): 8-row groups 1024 B apart; k-step kk (16
// elements of D) selects box kk/4 and a 32-byte offset in the 128-byte row.
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t tile_addr, uint32_t box_bytes, int kk) {
  return make_sw128_desc(tile_addr + (kk >> 2) * box_bytes + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 V block as the B operand (N = head dim contiguous): the two
// 64-column boxes are LBO = 8 KB apart, 8-key groups SBO = 1 KB; k-step = 16 keys.
__device__ __forceinline__ uint64_t v_desc(uint32_t tile_addr, int kk) {
  return make_sw128_desc(tile_addr + kk * 2048, kKVBoxBytes, 1024);
}

// ---- packed fp32x2 (FFMA2 / FADD2) and the FMA-pipe exp2
__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 unf2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for finite x <= 8 on the FMA/ALU pipes: round-to-nearest split x = n + f,
// f in [-1/2, 1/2], cubic minimax for 2^f (max rel. error 1.0e-4, far below the
// bf16 rounding of P), exponent add.  x is clamped at -126 (result >= 2^-126).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.0f);
  const float t = __fadd_rn(x, 12582912.0f);  // 1.5 * 2^23: low mantissa bits = round(x)
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
  const float p = fmaf(fmaf(fmaf(0.05500893f, f, 0.24221097f), f, 0.69328290f), f, 1.0f);
  // (bits(t) << 23) == round(x) << 23 modulo 2^32 because 0x4B400000 << 23 == 0
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// ex2_poly on a pair with the rounding split and Horner steps on FADD2 / FFMA2
// (same IEEE operations, so bitwise equal to two ex2_poly calls).
__device__ __forceinline__ float2 ex2_poly_x2(float a, float b) {
  const uint64_t x2 = f2(fmaxf(a, -126.0f), fmaxf(b, -126.0f));
  const uint64_t t = fadd2(x2, f2(12582912.0f, 12582912.0f));
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x2), "l"(fadd2(t, f2(-12582912.0f, -12582912.0f))));
  uint64_t pp = ffma2(f2(0.05500893f, 0.05500893f), r, f2(0.24221097f, 0.24221097f));
  pp = ffma2(pp, r, f2(0.69328290f, 0.69328290f));
  pp = ffma2(pp, r, f2(1.0f, 1.0f));
  const float2 pf = unf2(pp), tf = unf2(t);
  return make_float2(__int_as_float(__float_as_int(pf.x) + (__float_as_int(tf.x) << 23)),
                     __int_as_float(__float_as_int(pf.y) + (__float_as_int(tf.y) << 23)));
}


// ---- kernel forms
// v4 (attn_fwd.cu): 64-key blocks, double-buffered S.  v12 (attn_fwd_n128.cu):
// 128-key blocks, one S buffer per tile.  v13 (attn_fwd_pair.cu): CTA pairs,
// 128-key blocks, three S buffers, block-alternating softmax groups.
// Key-block rows of a version's tile summaries:
inline int attn_key_rows(int version) { return (version == 4 || version == 15) ? 64 : 128; }
// TMA box rows of the K / V maps (v13 loads half blocks: 64 keys of K, 128 keys x 64 dims of V)
inline int attn_k_box_rows(int version) { return (version == 13 || version == 14) ? 64 : attn_key_rows(version); }
inline int attn_v_box_rows(int version) { return attn_key_rows(version); }
#ifndef RCP_DEFAULT_ATTN_VERSION
#define RCP_DEFAULT_ATTN_VERSION 4
#endif
constexpr int kDefaultAttnVersion = RCP_DEFAULT_ATTN_VERSION;
#ifndef RCP_AB_FORMS
#define RCP_AB_FORMS 0  // 1: the A/B build with the alternative kernel forms (v12-v17)
#endif
int attn_n128_launch(const AttnParams& prm, int64_t grid, cudaStream_t st, int form);
int attn_qk8_launch(const AttnParams& prm, int64_t grid, cudaStream_t st);
int attn_pair_launch(const AttnParams& prm, int64_t n_pairs_heads, cudaStream_t st, bool col_split);

}  // namespace rcp
