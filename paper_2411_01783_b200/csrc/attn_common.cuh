// Shared pieces of the attention kernels (attn_fwd.cu: active-list pre-pass,
// the default v4 kernel and the C ABI; attn_variants.cu: the A/B variants
// v5-v8): parameters, tile constants, trace macro, tile-summary helpers,
// packed fp32x2 math and the FMA-pipe exp2, and the CTA-pair primitives.
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
// Of every 8 score pairs of a FULL block, this many take exp2 on the FMA pipe
// (cubic polynomial) instead of MUFU.EX2, balancing the two pipes.  With the
// per-tile MMA issuers (v4f) the softmax waits less and the FMA pipe is the
// tighter one: 1 measured +3 % over 2 (CP1), 0 and 3 slower.
#ifndef RCP_POLY_PAIRS
#define RCP_POLY_PAIRS 1
#endif
constexpr int kPolyPairsPer8 = RCP_POLY_PAIRS;
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


// ---- CTA-pair (cta_group::2) primitives used by the v5 / v8 variants
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion is reported to the LEADER CTA's barrier (same smem offset).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                                 int c1, uint64_t hint) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)),
      "r"(b), "r"(c0), "r"(c1), "l"(hint)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ss_lo(uint32_t d, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 da, db;\nsetp.ne.b32 p, %5, 0;\nmov.b64 da, {%1, %3};\n"
      "mov.b64 db, {%2, %3};\ntcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %4, p;\n}\n" ::"r"(d),
      "r"(a_lo), "r"(b_lo), "n"(kSw128DescHi), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts_lo(uint32_t d, uint32_t a, uint32_t b_lo, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 db;\nsetp.ne.b32 p, %5, 0;\nmov.b64 db, {%2, %3};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], db, %4, p;\n}\n" ::"r"(d),
      "r"(a), "r"(b_lo), "n"(kSw128DescHi), "r"(idesc), "r"(acc)
      : "memory");
}
// Commit to the barrier at this smem offset in BOTH CTAs of the pair.
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// Remote arrive on the leader CTA's barrier.  Default .release.cta semantics
// (as CUTLASS's ClusterBarrier::arrive): the consumer of P is the leader's
// tcgen05.mma, ordered by tcgen05.fence::before_thread_sync on this side and
// fence::after_thread_sync after the wait.  A .release.cluster arrive stalled
// the arriving warp ~1000 cycles per block (tools/trace_attn.py, v5).
#ifndef RCP_ARRIVE_CLUSTER_RELEASE
#define RCP_ARRIVE_CLUSTER_RELEASE 0
#endif
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
#if RCP_ARRIVE_CLUSTER_RELEASE
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & 0xFEFFFFFFu)
               : "memory");
#else
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & 0xFEFFFFFFu) : "memory");
#endif
}


// ---- variants (attn_variants.cu)
// Key-block rows of a version's tile summaries / TMA boxes.
inline int attn_key_rows(int version) { return (version == 4 || version == 7 || version >= 9) ? 64 : 128; }
inline int attn_k_box_rows(int version) { return version == 6 ? 128 : 64; }
inline int attn_v_box_rows(int version) { return (version == 4 || version == 7 || version >= 9) ? 64 : 128; }
// Launch variant `version` (5..11) over n_pairs_heads = (query-tile pairs) x Hq.
int attn_variant_launch(int version, const AttnParams& prm, int64_t n_pairs_heads, cudaStream_t st);

}  // namespace rcp
