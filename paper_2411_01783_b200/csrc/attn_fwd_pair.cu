// K1, CTA-pair form (v13): causal-by-position GQA flash-attention forward for
// sm_100a with LSE.  Replaces ringcp.attention.gqa_attention
// (attention.py:230-282) on the ring hot path with the masking / active-list /
// epilogue contract of the 64-key v4 kernel (attn_fwd.cu).
//
// Why this shape.  Per SM, one 128 x 128 score block costs 1024 tensor cycles
// (S = Q K^T plus O += P V) and ~1000 cycles of softmax issue on the SM's four
// SMSPs, so the two must overlap almost perfectly:
//   * S must be issued with N = 128 (a 128 x 64 SS MMA needs 192 B/clk of
//     shared-memory operands against the 128 B/clk port and runs at 55 %,
//     profiles/r01_probe_mma_rate.txt);
//   * the softmax must never wait for a PV -> S round trip, i.e. S needs more
//     than one TMEM buffer per query tile;
//   * operand traffic through shared memory must stay under the port.
// One CTA with two 128-row tiles has no TMEM for a second S buffer
// (O0|O1|S0|S1 = 512 columns, v12 / attn_fwd_n128.cu); one tile per CTA needs
// ~160 B/clk of operand + TMA traffic.  A CTA pair (cta_group::2, M = 256)
// halves the per-SM B operands (each CTA holds half of every K and V block),
// ~96 B/clk, and each CTA's TMEM holds its 128 rows of O plus THREE S buffers.
//
// Cluster of 2 CTAs = one 256-row query block of one query head; CTA r owns
// query rows [128 r, 128 r + 128) of it.  Per 128-key block j the leader CTA
// issues S(j) = Q K_j^T (M256 x N128, B split by keys: CTA r holds keys
// [64 r, 64 r + 64) of the block) into S buffer j % 3, and O += P(j) V_j
// (M256 x N128 dims, A = P from TMEM, B split by dims: CTA r holds dims
// [64 r, 64 r + 64) of all 128 keys).  S(j+3) follows PV(j) in the same buffer
// (tcgen05 MMAs of one thread execute in order).
//
// Softmax: two warpgroups per CTA take ALTERNATE key blocks (group g owns
// blocks j = g mod 2) with full 128-column rows, both accumulating into the
// one O of their rows.  They share the row's running max m through shared
// memory: group g computes block j's row max, takes m(j-1) from the other
// group (handed over through a 64-thread named barrier of the two warps that
// own the same TMEM lane quarter), raises it lazily (only when it grows by
// more than 2^8), hands m(j) on, then exponentiates.  Each group keeps its own
// row sum in units of the m it last used (rescaled when m moves) and the two
// sums are combined in the epilogue.  A raise of m at block j rescales O in
// place after PV(j-1) has completed and before P(j) is published, so every PV
// accumulates with the current m.  The two groups' softmaxes run staggered by
// one block, so each SMSP always has one group in its exp phase while the
// other loads / reduces, and the tensor cores always have S queued.
//
// Warp roles (384 threads): warp 0 TMA producer (both CTAs), warp 1 MMA issuer
// (leader only), warp 2 TMEM allocator, warp 3 idle, warps 4-7 softmax group
// 0, warps 8-11 softmax group 1 (thread i of a group <-> TMEM lane / row i).
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

#include "attn_common.cuh"

namespace rcp {

constexpr int kSBufP = 3;                    // S buffers per CTA
constexpr int kKRowsP = 128;                 // keys per block
constexpr int kSlotsP = 11;                  // 16 KB half-block slots (K half, V half, ...)
constexpr uint32_t kSlotBytesP = 16384;      // K half: 64 keys x 128 dims; V half: 128 keys x 64 dims
constexpr uint32_t kSmemBytesP = kQTileBytes + kSlotsP * kSlotBytesP + 1024;
static_assert(kSmemBytesP + 8192 <= 232448, "v13 shared memory (+ static barriers / exchange arrays) exceeds 227 KB");
constexpr uint32_t kTmemOP = 0, kTmemSP = 128;
#ifndef RCP_POLY_PAIRS_P
#define RCP_POLY_PAIRS_P 2
#endif
constexpr int kPolyPairsP = RCP_POLY_PAIRS_P;  // of every 8 score pairs of a FULL block on the FMA pipe

// ---- CTA-pair primitives
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive_wait() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion is reported to the LEADER CTA's barrier (same smem offset).
__device__ __forceinline__ void tma_load_2d_to_leader(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                                      int c1, uint64_t hint) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)),
      "r"(b), "r"(c0), "r"(c1), "l"(hint)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint32_t a_lo, uint32_t b_lo, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 da, db;\nsetp.ne.b32 p, %5, 0;\nmov.b64 da, {%1, %3};\n"
      "mov.b64 db, {%2, %3};\ntcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %4, p;\n}\n" ::"r"(d),
      "r"(a_lo), "r"(b_lo), "n"(kSw128DescHi), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint32_t b_lo, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 db;\nsetp.ne.b32 p, %5, 0;\nmov.b64 db, {%2, %3};\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], db, %4, p;\n}\n" ::"r"(d),
      "r"(a), "r"(b_lo), "n"(kSw128DescHi), "r"(idesc), "r"(acc)
      : "memory");
}
// Commit to the barrier at this smem offset in BOTH CTAs of the pair.
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// Arrive on the leader CTA's barrier (the consumer is the leader's tcgen05.mma,
// ordered by tcgen05.fence::before_thread_sync here and ::after after its wait).
__device__ __forceinline__ void arrive_on_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & 0xFEFFFFFFu) : "memory");
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// The lazily raised running max: m moves only when the block max exceeds it by
// more than 2^8 (also -inf -> finite).
__device__ __forceinline__ float lazy_max(float m, float blk) { return blk > m + kRescaleThreshold ? blk : m; }
__device__ __forceinline__ float2 unpack_bf16x2(uint32_t v) {
  return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
}

// kColSplit = false (v13): the two softmax groups take alternate key blocks.
// kColSplit = true (v14): both groups take every block, group g the score
// columns [64 g, 64 g + 64) of all 128 rows (two warps per SMSP in the same
// phase, as v4's two tiles, but on N = 128 MMAs with three S buffers).
template <bool kColSplit>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_pair_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // this CTA's 128-row query tile
  uint8_t* sKV = smem + kQTileBytes;  // kSlotsP half blocks: K half / V half alternate

  __shared__ uint64_t bar_q, bar_full[kSlotsP], bar_empty[kSlotsP];
  __shared__ uint64_t bar_s[kSBufP], bar_p[kSBufP], bar_pv[2], bar_o;
  __shared__ uint32_t tmem_slot;
  __shared__ float m_xch[2][128];  // [producing group][row]: m(it) handed to the other group
  __shared__ float l_xch[2][128];  // epilogue: each group's row sum
  __shared__ float mx2[2][2][128];  // v14: [block parity][group][row] half-block max

  const int warp = static_cast<int>(warp_id());
  // Pair order as v4: KV-head major, heavy (late) query blocks first, then the
  // GQA group.  Recomputed inside each role (after its setmaxnreg) so nothing
  // from here is live across a register-limit change.
  auto coords = [&](int& rank, int& qblk, int& head, int& kvh, int& n, const uint32_t*& act) {
    rank = static_cast<int>(cluster_ctarank());
    const int pair = static_cast<int>(blockIdx.x) >> 1;
    const int per_kv = p.n_qblk * p.group;
    kvh = pair / per_kv;
    const int rem = pair - kvh * per_kv;
    qblk = p.n_qblk - 1 - rem / p.group;
    head = kvh * p.group + rem % p.group;
    n = __ldg(p.act_n + qblk);
    act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
  };

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kSlotsP; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int b = 0; b < kSBufP; ++b) {
      mbar_init(&bar_s[b], 1);
      // v13: the four warps of the block's softmax group; v14: all eight; in both CTAs
      mbar_init(&bar_p[b], kColSplit ? 2 * 8 : 2 * 4);
    }
    mbar_init(&bar_pv[0], 1);  // PV(it) completions, it even / odd
    mbar_init(&bar_pv[1], 1);
    mbar_init(&bar_o, 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_arrive_wait();
  tc_fence_after();

  // Registers: the softmax rows hold 128 scores, the TMA / MMA / TMEM
  // warpgroup needs few.  setmaxnreg.inc can only take what .dec released
  // from the launch allocation (384 x 168 = 64512, not the 65536 of the
  // file: 128 x 32 + 256 x 240 hangs the increase), so 128 x 40 + 256 x 232.
  if (warp < 4) {
    setmaxnreg_dec<40>();
    int rank, qblk, head, kvh, n;
    const uint32_t* act;
    coords(rank, qblk, head, kvh, n, act);
    const uint32_t tmem = tmem_slot;
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer (both CTAs)
      if (elect_one() && n > 0) {
        tma_prefetch_desc(&p.tm_q);
        tma_prefetch_desc(&p.tm_k);
        tma_prefetch_desc(&p.tm_v);
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        if (rank == 0) mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes);
        for (int h = 0; h < 2; ++h)
          tma_load_2d_to_leader(sQ + h * kQBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                                (2 * qblk + rank) * kQRows, pol_q);
        uint32_t ld = 0;  // K_j half is load 2 it, V_j half load 2 it + 1
        uint32_t e_next = __ldg(act);
        for (int it = 0; it < n; ++it) {
          const int j = act_j(e_next);
          if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++ld) {
            const uint32_t slot = ld % kSlotsP, ph = (ld / kSlotsP) & 1;
            mbar_wait(&bar_empty[slot], ph ^ 1);
            TRACE(6 + kv, it);
            if (rank == 0) mbar_arrive_expect_tx(&bar_full[slot], 2 * kSlotBytesP);
            uint8_t* dst = sKV + slot * kSlotBytesP;
            if (kv == 0) {  // K half: keys [128 j + 64 r, +64), all 128 dims (two 8 KB boxes)
              for (int h = 0; h < 2; ++h)
                tma_load_2d_to_leader(dst + h * 8192, &p.tm_k, &bar_full[slot], kvh * kD + h * 64,
                                      j * kKRowsP + rank * 64, pol_kv);
            } else {        // V half: all 128 keys, dims [64 r, 64 r + 64)
              tma_load_2d_to_leader(dst, &p.tm_v, &bar_full[slot], kvh * kD + rank * 64, j * kKRowsP, pol_kv);
            }
          }
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer (leader CTA, one lane)
      if (rank == 0 && n > 0 && elect_one()) {
        const uint32_t idesc_s = make_idesc_bf16_f32(256, kKRowsP, 0, 0);
        const uint32_t idesc_o = make_idesc_bf16_f32(256, kD, 0, 1);
        const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
        const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
        const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kSlotBytesP);
        auto wait_load = [&](uint32_t ld) {
          mbar_wait(&bar_full[ld % kSlotsP], (ld / kSlotsP) & 1);
          tc_fence_after();
        };
        auto issue_s = [&](int buf, uint32_t ld) {
          const uint32_t ka = k_lo + (((ld % kSlotsP) * kSlotBytesP) >> 4);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk)
            mma2_ss(tmem + kTmemSP + buf * 128, q_lo + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                    ka + (((kk >> 2) * 8192 + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
        };
        auto issue_pv = [&](int buf, uint32_t ld, bool acc) {
          const uint32_t va = v_lo + (((ld % kSlotsP) * kSlotBytesP) >> 4);
#pragma unroll
          for (int kk = 0; kk < kKRowsP / 16; ++kk) {
            // P columns of keys [16 kk, 16 kk + 16): v13 packs all 128 keys over the first 64
            // columns of the S buffer; v14's groups each pack theirs over the first 32 of
            // their own 64 S columns
            const uint32_t pcol = kColSplit ? (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8) : kk * 8;
            mma2_ts(tmem + kTmemOP, tmem + kTmemSP + buf * 128 + pcol, va + ((kk * 2048) >> 4), idesc_o,
                    (acc || kk > 0) ? 1u : 0u);
          }
        };
        mbar_wait(&bar_q, 0);
        for (int b = 0; b < kSBufP && b < n; ++b) {
          wait_load(2 * b);
          issue_s(b, 2 * b);
          commit2(&bar_s[b]);
          commit2(&bar_empty[(2 * b) % kSlotsP]);
        }
        int buf = 0;
        uint32_t ph = 0;
        for (int it = 0; it < n; ++it) {
          const bool last = it + 1 == n;
          const uint32_t ldv = 2 * it + 1, ldk = 2 * (it + kSBufP);
          wait_load(ldv);
          mbar_wait(&bar_p[buf], ph);
          tc_fence_after();
          TRACE(0, it);
          issue_pv(buf, ldv, it > 0);
          commit2(last ? &bar_o : &bar_pv[it & 1]);
          commit2(&bar_empty[ldv % kSlotsP]);
          if (it + kSBufP < n) {
            wait_load(ldk);
            issue_s(buf, ldk);
            TRACE(1, it);
            commit2(&bar_s[buf]);
            commit2(&bar_empty[ldk % kSlotsP]);
          }
          if (++buf == kSBufP) {
            buf = 0;
            ph ^= 1u;
          }
        }
      }
      __syncwarp();
    }
  } else {
    setmaxnreg_inc<232>();
    int rank, qblk, head, kvh, n;
    const uint32_t* act;
    coords(rank, qblk, head, kvh, n, act);
    const uint32_t tmem = tmem_slot;
    // ------------------------------------------------------------ softmax + epilogue (both CTAs)
    const int g = (warp - 4) >> 2;                                // softmax group: blocks it = g mod 2
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * g;  // row inside this CTA's tile
    const int q4 = warp & 3;                                      // TMEM lane quarter / SMSP
    const int row = (2 * qblk + rank) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) - p.mask_shift : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemOP;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    // Named barriers (64 threads = the two warps of this lane quarter):
    // 1 + q4 + 4 g hands m from group g to the other group; 9 + q4 is the
    // epilogue's.
    const uint32_t bar_give = 1 + q4 + 4 * g, bar_take = 1 + q4 + 4 * (g ^ 1);
    float m = -INFINITY;   // m (log2 units) after the last block this group processed
    float mg = -INFINITY;  // the m this group's row sum lg is expressed in
    float lg = 0.f;
    if constexpr (!kColSplit) {
      int it = g;
      for (; it < n; it += 2) {
        const int buf = it % kSBufP;
        const uint32_t s_addr = lane_base + kTmemSP + buf * 128;
        const uint32_t e = __ldg(act + it);
        const int j = act_j(e);
        const int cls = act_cls(e, rank);
        // mask bits of a PARTIAL block (bit c: key c admitted), before S is live
        uint32_t mbits[4] = {~0u, ~0u, ~0u, ~0u};
        if (cls == kTilePartial) {
          const int base = j * kKRowsP;
          if (base + kKRowsP <= p.tk) {
            const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
            const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
  #pragma unroll 1
            for (int gq = 0; gq < 4; ++gq) {  // (not unrolled: 8 int4 pairs in flight, not 64)
              uint32_t bits = 0;
  #pragma unroll
              for (int c4 = 0; c4 < 8; ++c4) {
                const int4 kp = __ldg(kp4 + 8 * gq + c4), kq = __ldg(ks4 + 8 * gq + c4);
                bits |= static_cast<uint32_t>(kq.x == my_seq && kp.x <= my_pos) << (4 * c4 + 0);
                bits |= static_cast<uint32_t>(kq.y == my_seq && kp.y <= my_pos) << (4 * c4 + 1);
                bits |= static_cast<uint32_t>(kq.z == my_seq && kp.z <= my_pos) << (4 * c4 + 2);
                bits |= static_cast<uint32_t>(kq.w == my_seq && kp.w <= my_pos) << (4 * c4 + 3);
              }
  #pragma unroll
              for (int x = 0; x < 4; ++x) mbits[x] = gq == x ? bits : mbits[x];
            }
          } else {
  #pragma unroll
            for (int gq = 0; gq < 4; ++gq) {  // (unrolled: mbits stays in registers)
              uint32_t bits = 0;
  #pragma unroll 1
              for (int c = 0; c < 32; ++c) {
                const int kidx = base + 32 * gq + c;
                const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq && __ldg(p.k_pos + kidx) <= my_pos;
                bits |= static_cast<uint32_t>(ok) << c;
              }
              mbits[gq] = bits;
            }
          }
        }
        mbar_wait(&bar_s[buf], (it / kSBufP) & 1);
        tc_fence_after();
        if (t == 0) TRACE(2 + 2 * g, it >> 1);
        // The running max m(it) = lazy(m(it-1), max of block it) chains the
        // blocks of both groups: group g takes m(it-1) from the other group and
        // hands m(it) on.  The exps run first, with the provisional m of the
        // group's own chain, so they never wait; the exact m(it) is settled after
        // them, and in the rare case it differs (the other group raised m at
        // it-1) this row's P and block sum are rescaled by the exact power of two.
        uint32_t s[128];  // scores (fp32 bits) of this row
        float mx = -INFINITY;
        if (cls != kTileEmpty) {  // uniform across the CTA
          tmem_ld64(s_addr, s);
          tmem_ld64(s_addr + 64, s + 64);
          tmem_ld_wait();
          if (cls == kTilePartial) {
  #pragma unroll
            for (int c = 0; c < 128; ++c)
              if (!((mbits[c >> 5] >> (c & 31)) & 1u)) s[c] = 0xFF800000u;  // -inf
          }
          float m8[8];
  #pragma unroll
          for (int k = 0; k < 8; ++k)
            m8[k] = fmax3(__uint_as_float(s[k]), __uint_as_float(s[8 + k]), __uint_as_float(s[16 + k]));
  #pragma unroll
          for (int c = 24; c < 120; c += 16)
  #pragma unroll
            for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], __uint_as_float(s[c + k]), __uint_as_float(s[c + 8 + k]));
  #pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], __uint_as_float(s[120 + k]));
          mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
        }
        if (t == 0 && g == 0) TRACE(8, it >> 1);
        const float mx_l2 = mx * sl2;
        // provisional m of this block from this group's own chain (m holds m(it-2)):
        // the exps never wait for the other group
        const float m_prov = lazy_max(m, mx_l2);  // m: this group's m after its previous block
        float bsum = 0.f;
        if (cls != kTileEmpty) {
          const float m_use = (m_prov == -INFINITY) ? 0.f : m_prov;
          const uint64_t negm2 = f2(-m_use, -m_use);
          uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
          auto exp_chunks = [&](auto full) {
  #pragma unroll
            for (int q = 0; q < 4; ++q) {  // 32 keys -> 16 packed P columns per chunk
              uint32_t pk[16];
  #pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int ip = 16 * q + i;
                const float2 x =
                    unf2(ffma2(f2(__uint_as_float(s[2 * ip]), __uint_as_float(s[2 * ip + 1])), sl2x2, negm2));
                float p0, p1;
                if (decltype(full)::value && (ip & 7) < kPolyPairsP) {
                  const float2 pp = ex2_poly_x2(x.x, x.y);
                  p0 = pp.x;
                  p1 = pp.y;
                } else {
                  p0 = ex2_approx(x.x);
                  p1 = ex2_approx(x.y);
                }
                acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
                pk[i] = pack_bf16x2(p0, p1);
              }
              tmem_st16(s_addr + 16 * q, pk);
            }
          };
          if (cls == kTileFull) {
            exp_chunks(std::true_type{});
          } else {
            exp_chunks(std::false_type{});
          }
          const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
          const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
          bsum = (a01.x + a01.y) + (a23.x + a23.y);
        } else {
          uint32_t pk[32];
  #pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = 0u;
          tmem_st32(s_addr, pk);
          tmem_st32(s_addr + 32, pk);
        }
        if (t == 0 && g == 0) TRACE(9, it >> 1);
        // settle m(it): take m(it-1) from the other group, hand m(it) on
        const float m_in = it > 0 ? (named_bar_sync(bar_take, 64), m_xch[g ^ 1][t]) : -INFINITY;
        const float m_fin = lazy_max(m_in, mx_l2);
        if (it + 1 < n) {
          m_xch[g][t] = m_fin;
          named_bar_arrive(bar_give, 64);
        }
        if (t == 0 && g == 0) TRACE(10, it >> 1);
        // rare: P was made with a different m (the other group raised m at it-1)
        // -> rescale this row's P and block sum by the exact power of two
        const bool fix_p = m_prov != m_fin && m_prov != -INFINITY && cls != kTileEmpty;
        if (__any_sync(0xffffffffu, fix_p)) {
          const float fp = fix_p ? ex2_approx(m_prov - m_fin) : 1.0f;
          tmem_st_wait();
  #pragma unroll 1
          for (int c = 0; c < 64; c += 8) {
            uint32_t pk[8];
            tmem_ld8(s_addr + c, pk);
            tmem_ld_wait();
  #pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float2 v2 = unpack_bf16x2(pk[i]);
              pk[i] = pack_bf16x2(v2.x * fp, v2.y * fp);
            }
            tmem_st8(s_addr + c, pk);
          }
          bsum *= fp;
        }
        // O rescale when block it raised m over a non-empty O: after PV(it-1)
        // completed (PV(it) waits for this group's P)
        const bool raised = m_fin != m_in && m_in != -INFINITY;
        if (__any_sync(0xffffffffu, raised)) {
          const float f = raised ? ex2_approx(m_in - m_fin) : 1.0f;
          // PV(it-1) is phase (it-1)/2 of bar_pv[(it-1)&1]; PV(it-3) (same barrier,
          // one phase earlier) completed before S(it) was issued and PV(it+1)
          // cannot start before this group's P(it), so the parity is unambiguous
          mbar_wait(&bar_pv[(it - 1) & 1], ((it - 1) >> 1) & 1);
          tc_fence_after();
  #pragma unroll 1
          for (int c = 0; c < kD; c += 8) {
            uint32_t r[8];
            tmem_ld8(o_addr + c, r);
            tmem_ld_wait();
  #pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st8(o_addr + c, r);
          }
        }
        m = m_fin;
        // this group's row sum, in units of the current m
        if (m != mg) {
          lg = (mg == -INFINITY) ? 0.f : lg * ex2_approx(mg - m);
          mg = m;
        }
        lg += bsum;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) arrive_on_leader(&bar_p[buf]);
        if (t == 0) TRACE(3 + 2 * g, it >> 1);
      }
    } else {
      // ---- v14: every block, this group's 64 score columns
      const uint32_t bar_x = 1 + q4;  // symmetric exchange of the half-block max (this quarter's 2 warps)
      for (int it = 0; it < n; ++it) {
        const int buf = it % kSBufP;
        const uint32_t s_addr = lane_base + kTmemSP + buf * 128 + 64 * g;
        const uint32_t e = __ldg(act + it);
        const int j = act_j(e);
        const int cls = act_cls(e, rank);
        uint32_t mbits[2] = {~0u, ~0u};
        if (cls == kTilePartial) {
          const int base = j * kKRowsP + 64 * g;
#pragma unroll
          for (int gq = 0; gq < 2; ++gq) {
            uint32_t bits = 0;
#pragma unroll 4
            for (int c = 0; c < 32; ++c) {
              const int kidx = base + 32 * gq + c;
              const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq && __ldg(p.k_pos + kidx) <= my_pos;
              bits |= static_cast<uint32_t>(ok) << c;
            }
            mbits[gq] = bits;
          }
        }
        mbar_wait(&bar_s[buf], (it / kSBufP) & 1);
        tc_fence_after();
        if (t == 0) TRACE(2 + 2 * g, it);
        uint32_t s[64];
        float mx = -INFINITY;
        if (cls != kTileEmpty) {
          tmem_ld64(s_addr, s);
          tmem_ld_wait();
          if (cls == kTilePartial) {
#pragma unroll
            for (int c = 0; c < 64; ++c)
              if (!((mbits[c >> 5] >> (c & 31)) & 1u)) s[c] = 0xFF800000u;
          }
          float m8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            m8[k] = fmax3(__uint_as_float(s[k]), __uint_as_float(s[8 + k]), __uint_as_float(s[16 + k]));
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], __uint_as_float(s[24 + k]), __uint_as_float(s[32 + k]));
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], __uint_as_float(s[40 + k]), __uint_as_float(s[48 + k]));
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], __uint_as_float(s[56 + k]));
          mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
        }
        const float mx_l2 = mx * sl2;
        // exps with the provisional m from this half's max; the exact m (both
        // halves) is settled after them and differs only when just one half
        // raises the lazy max (rare): then this half's P and sum are rescaled
        const float m_prov = lazy_max(m, mx_l2);
        float bsum = 0.f;
        if (cls != kTileEmpty) {
          const float m_use = (m_prov == -INFINITY) ? 0.f : m_prov;
          const uint64_t negm2 = f2(-m_use, -m_use);
          uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
          auto exp_chunks = [&](auto full) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int ip = 16 * q + i;
                const float2 x =
                    unf2(ffma2(f2(__uint_as_float(s[2 * ip]), __uint_as_float(s[2 * ip + 1])), sl2x2, negm2));
                float p0, p1;
                if (decltype(full)::value && (ip & 7) < kPolyPairsP) {
                  const float2 pp = ex2_poly_x2(x.x, x.y);
                  p0 = pp.x;
                  p1 = pp.y;
                } else {
                  p0 = ex2_approx(x.x);
                  p1 = ex2_approx(x.y);
                }
                acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
                pk[i] = pack_bf16x2(p0, p1);
              }
              tmem_st16(s_addr + 16 * q, pk);
            }
          };
          if (cls == kTileFull) {
            exp_chunks(std::true_type{});
          } else {
            exp_chunks(std::false_type{});
          }
          const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
          const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
          bsum = (a01.x + a01.y) + (a23.x + a23.y);
        } else {
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = 0u;
          tmem_st32(s_addr, pk);
        }
        if (t == 0 && g == 0) TRACE(9, it);
        mx2[it & 1][g][t] = mx_l2;
        named_bar_sync(bar_x, 64);
        const float m_fin = lazy_max(m, fmaxf(mx_l2, mx2[it & 1][g ^ 1][t]));
        const bool fix_p = m_prov != m_fin && m_prov != -INFINITY && cls != kTileEmpty;
        if (__any_sync(0xffffffffu, fix_p)) {
          const float fp = fix_p ? ex2_approx(m_prov - m_fin) : 1.0f;
          tmem_st_wait();
#pragma unroll 1
          for (int c = 0; c < 32; c += 8) {
            uint32_t pk[8];
            tmem_ld8(s_addr + c, pk);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float2 v2 = unpack_bf16x2(pk[i]);
              pk[i] = pack_bf16x2(v2.x * fp, v2.y * fp);
            }
            tmem_st8(s_addr + c, pk);
          }
          bsum *= fp;
        }
        // O rescale when block it raised m over a non-empty O: this group's 64
        // O columns, after PV(it-1) completed
        const bool raised = m_fin != m && m != -INFINITY;
        if (__any_sync(0xffffffffu, raised)) {
          const float f = raised ? ex2_approx(m - m_fin) : 1.0f;
          mbar_wait(&bar_pv[(it - 1) & 1], ((it - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 64; c += 8) {
            uint32_t r[8];
            tmem_ld8(o_addr + 64 * g + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st8(o_addr + 64 * g + c, r);
          }
        }
        m = m_fin;
        if (m != mg) {
          lg = (mg == -INFINITY) ? 0.f : lg * ex2_approx(mg - m);
          mg = m;
        }
        lg += bsum;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) arrive_on_leader(&bar_p[buf]);
        if (t == 0) TRACE(3 + 2 * g, it);
      }
    }

    // epilogue: combine the groups' sums in the final m, O / l, LSE, optional merge
    if (n > 0) {
      mbar_wait(&bar_o, 0);
      tc_fence_after();
    }
    const bool merge = p.mode == RCP_MODE_MERGE;
    if (!(merge && n == 0)) {
      m_xch[g][t] = mg;
      l_xch[g][t] = lg;
      named_bar_sync(9 + q4, 64);
      const float mo = m_xch[g ^ 1][t], lo = l_xch[g ^ 1][t];
      const float mf = fmaxf(mg, mo);
      float l = 0.f;
      if (mf != -INFINITY) {
        l = (mg == -INFINITY ? 0.f : lg * ex2_approx(mg - mf)) + (mo == -INFINITY ? 0.f : lo * ex2_approx(mo - mf));
      }
      const bool has = l > 0.f;
      const float inv = has ? 1.0f / l : 0.f;
      const float lse_new = has ? (mf + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD + g * 64;
      float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
      MergeW mw;
      mw.lse = lse_new;
      mw.wa = 0.f;
      mw.wb = 1.f;
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
      for (int c = 0; c < 64; c += 32) {  // group g stores O columns [64 g, 64 g + 64)
        uint32_t r[32];
        if (n > 0) {
          tmem_ld32(o_addr + 64 * g + c, r);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        if (row_ok) {
          float4* dst = reinterpret_cast<float4*>(orow + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 v = make_float4(__uint_as_float(r[4 * i]) * inv, __uint_as_float(r[4 * i + 1]) * inv,
                                   __uint_as_float(r[4 * i + 2]) * inv, __uint_as_float(r[4 * i + 3]) * inv);
            if (merge) {
              const float4 a = dst[i];
              v = make_float4(merge_val(a.x, v.x, mw), merge_val(a.y, v.y, mw), merge_val(a.z, v.z, mw),
                              merge_val(a.w, v.w, mw));
            }
            dst[i] = v;
          }
        }
      }
      if (merge) named_bar_sync(9 + q4, 64);  // both groups read the old LSE before it is overwritten
      if (row_ok && g == 0) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_arrive_wait();  // the peer's TMEM / smem stay live until the leader's MMAs are done
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_slot), "n"(512) : "memory");
  }
}

int attn_pair_launch(const AttnParams& prm, int64_t n_pairs_heads, cudaStream_t st, bool col_split) {
  static bool attr_set[2] = {false, false};
  auto kern = col_split ? attn_fwd_pair_kernel<true> : attn_fwd_pair_kernel<false>;
  if (!attr_set[col_split]) {
    RCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytesP));
    attr_set[col_split] = true;
  }
  kern<<<static_cast<unsigned>(2 * n_pairs_heads), kThreads, kSmemBytesP, st>>>(prm);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

}  // namespace rcp
