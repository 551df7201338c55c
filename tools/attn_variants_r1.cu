// A/B variants of the attention forward kernel (selected with
// RCP_ATTN_VERSION=5..8; the default v4 lives in attn_fwd.cu).  Each passes
// the same parity tests; DESIGN.md ("Attention kernel versions") has the
// measured comparison and why v4 stays the default.
#include "attn_common.cuh"

namespace rcp {
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



// Key-block rows of the round-1 variants (5-11).
inline int attn_key_rows_r1(int version) { return (version == 7 || version >= 9) ? 64 : 128; }
inline int attn_k_box_rows(int version) { return version == 6 ? 128 : 64; }
inline int attn_v_box_rows(int version) { return (version == 7 || version >= 9) ? 64 : 128; }
int attn_variant_launch(int version, const AttnParams& prm, int64_t n_pairs_heads, cudaStream_t st);
}  // namespace rcp


namespace rcp {

// ======================================================================
// v6: 1-CTA, 128-key blocks (default).  Same warp roles as v4, but S = Q K^T
// is issued with N = 128: a 128 x 64 SS MMA needs 6 KB of shared-memory
// operands per 32 tensor cycles (192 B/clk > the 128 B/clk smem port) and
// measures at 55% of the tensor rate, while N = 128 runs at 100%
// (tools/probe_mma_rate.cu).  TMEM: O0 [0,128) | O1 [128,256) | S0 [256,384)
// | S1 [384,512): one S buffer per query tile, P_t(j) packed over the first
// 64 columns of S_t.  The MMA warp issues PV_0(j), S_0(j+1), PV_1(j),
// S_1(j+1): while the softmax of one tile runs, the tensor cores work on the
// other tile, and in-order tcgen05 execution makes S_t(j+1) land after
// PV_t(j) has read P_t(j).  K/V ring: 5 slots of 32 KB (K_j, V_j, ...).
//
// The softmax of a 128-column row costs ~1050 SMSP cycles per warp whatever
// the MUFU / FMA-pipe split (tools/probe_softmax_rate.cu), so two tiles'
// softmaxes running at once each take twice as long.  The two softmax
// warpgroups therefore take turns on their exp phase (named-barrier
// ping-pong), and each publishes P in four 32-key chunks with one barrier per
// chunk: the MMA warp issues PV k-steps as chunks land, so PV_t(j) overlaps
// the exps and S_t(j+1) follows right after the last chunk.
// ======================================================================
constexpr int kKRows6 = 128;
constexpr int kSlots6 = 4;
constexpr uint32_t kKV6Bytes = kKRows6 * kD * 2;   // 32 KB: two 16 KB SW128 boxes
constexpr uint32_t kKV6BoxBytes = kKV6Bytes / 2;
constexpr uint32_t kSmem6Bytes = 2 * kQTileBytes + kSlots6 * kKV6Bytes + 1024;
static_assert(kSmem6Bytes <= 232448, "v6 shared memory exceeds 227 KB");

constexpr int kThreads6 = 640;  // warpgroup 0: TMA / MMA / TMEM; 4 softmax warpgroups
// Exp-phase ping-pong between the two tiles' softmax warpgroups (measured
// slower than letting the warp schedulers interleave them; off by default).
#ifndef RCP_PINGPONG
#define RCP_PINGPONG 0
#endif

__global__ void __launch_bounds__(kThreads6, 1) attn_fwd_v6_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // 2 query tiles
  uint8_t* sKV = smem + 2 * kQTileBytes;      // kSlots6 K/V blocks

  __shared__ uint64_t bar_q, bar_full[kSlots6], bar_empty[kSlots6];
  __shared__ uint64_t bar_s[2], bar_p[2][4], bar_o[2];
  __shared__ uint32_t tmem_slot;
  __shared__ float xch6[2][2][kQRows];  // [tile][half][row]: row max / row sum exchange

  const int warp = static_cast<int>(warp_id());
  const int per_kv = p.n_qblk * p.group;
  const int kvh = static_cast<int>(blockIdx.x) / per_kv;
  const int rem = static_cast<int>(blockIdx.x) - kvh * per_kv;
  const int qblk = p.n_qblk - 1 - rem / p.group;
  const int head = kvh * p.group + rem % p.group;
  const int n = __ldg(p.act_n + qblk);
  const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kSlots6; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t], 1);
      for (int q = 0; q < 4; ++q) mbar_init(&bar_p[t][q], 128);
      mbar_init(&bar_o[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one() && n > 0) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes);
      for (int t = 0; t < 2; ++t)
        for (int h = 0; h < 2; ++h)
          tma_load_2d(sQ + t * kQTileBytes + h * kQBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                      (2 * qblk + t) * kQRows, pol_q);
      uint32_t ld = 0;  // K_j is load 2*it, V_j load 2*it + 1
      uint32_t e_next = __ldg(act);
      for (int it = 0; it < n; ++it) {
        const int j = act_j(e_next);
        if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++ld) {
          const uint32_t slot = ld % kSlots6, ph = (ld / kSlots6) & 1;
          mbar_wait(&bar_empty[slot], ph ^ 1);
          TRACE(6 + kv, it);
          mbar_arrive_expect_tx(&bar_full[slot], kKV6Bytes);
          const CUtensorMap* map = kv ? &p.tm_v : &p.tm_k;
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sKV + slot * kKV6Bytes + h * kKV6BoxBytes, map, &bar_full[slot], kvh * kD + h * 64,
                        j * kKRows6, pol_kv);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (one elected lane)
    if (elect_one() && n > 0) {
      const uint32_t idesc_s = make_idesc_bf16_f32(kQRows, kKRows6, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(kQRows, kD, 0, 1);
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kKV6BoxBytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots6], (ld / kSlots6) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int t, uint32_t ld) {
        const uint32_t qa = q_lo + ((t * kQTileBytes) >> 4);
        const uint32_t ka = k_lo + (((ld % kSlots6) * kKV6Bytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma_ss_lo(tmem + kTmemS + t * kKRows6, qa + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                    ka + (((kk >> 2) * kKV6BoxBytes + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      // PV_t(it) in four 32-key chunks, each issued once its P chunk is in TMEM.
      auto issue_pv = [&](int t, uint32_t ld, int it) {
        const uint32_t va = v_lo + (((ld % kSlots6) * kKV6Bytes) >> 4);
        const uint32_t pa = tmem + kTmemS + t * kKRows6;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          mbar_wait(&bar_p[t][q], it & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 2 * q; kk < 2 * q + 2; ++kk)
            mma_ts_lo(tmem + kTmemO + t * kD, pa + kk * 8, va + ((kk * 2048) >> 4), idesc_o,
                      (it > 0 || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(&bar_q, 0);
      wait_load(0);
      issue_s(0, 0);
      mma_commit(&bar_s[0]);
      issue_s(1, 0);
      mma_commit(&bar_s[1]);
      mma_commit(&bar_empty[0]);
      for (int it = 0; it < n; ++it) {
        const bool last = it + 1 == n;
        const uint32_t ldv = 2 * it + 1, ldk1 = 2 * it + 2;
        wait_load(ldv);
        TRACE(12, it);
        // tile 0: PV_0(it), then S_0(it+1) over the same TMEM columns
        issue_pv(0, ldv, it);
        TRACE(0, it);
        if (last) mma_commit(&bar_o[0]);
        if (!last) {
          wait_load(ldk1);
          issue_s(0, ldk1);
          mma_commit(&bar_s[0]);
        }
        // tile 1
        issue_pv(1, ldv, it);
        TRACE(1, it);
        if (last) mma_commit(&bar_o[1]);
        mma_commit(&bar_empty[ldv % kSlots6]);
        TRACE(13, it);
        if (!last) {
          issue_s(1, ldk1);
          mma_commit(&bar_s[1]);
          mma_commit(&bar_empty[ldk1 % kSlots6]);
        }
        TRACE(14, it);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    // Warpgroup g = warp/4 - 1: query tile w = g >> 1, column half h = g & 1.
    // Half h owns keys [32h, 32h+32) and [64+32h, 96+32h) of every block, i.e.
    // P chunks h and h+2, and O columns [64h, 64h+64) in the epilogue.
    const int g = (warp - 4) >> 2;
    const int w = g >> 1, h = g & 1;
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * g;  // row inside the tile
    const int row = (2 * qblk + w) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO + w * kD + h * 64;
    const uint32_t s_addr = lane_base + kTmemS + w * kKRows6;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;  // l: this half's partial row sum
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    // Named barriers: 1 + w pairs the two halves of tile w (row-max exchange);
    // 3 + w is tile w's exp-phase turn, arrived on by the other tile's 256
    // threads when their exp phase ends (tile 0 goes first).
    const uint32_t pair_bar = 1 + w, my_turn = 3 + w, their_turn = 4 - w;
    if (RCP_PINGPONG && w == 1 && n > 0) named_bar_arrive(their_turn, 512);
    int it = 0;
    for (; it < n; ++it) {
      const uint32_t e = e_next;
      if (it + 1 < n) e_next = __ldg(act + it + 1);
      const int j = act_j(e);
      const int cls = act_cls(e, w);
      // S_t(it) complete also means PV_t(it-1) is (one commit tracks all
      // earlier MMAs), so O_t may be rescaled in place below.
      mbar_wait(&bar_s[w], it & 1);
      tc_fence_after();
      if (t == 0 && h == 0) TRACE(2 + 2 * w, it);
      const bool hand_over = !(w == 1 && it + 1 == n);
      if (cls != kTileEmpty) {  // uniform over both halves of the tile
        float s[64];
        {
          uint32_t sr[64];
          tmem_ld32(s_addr + 32 * h, sr);
          tmem_ld32(s_addr + 64 + 32 * h, sr + 32);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
        }
        if (t == 0 && w == 0 && h == 0) TRACE(8, it);
        if (cls == kTilePartial) {
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const int base = j * kKRows6 + 64 * part + 32 * h;
            if (base + 32 <= p.tk) {
              const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
              const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll
              for (int c4 = 0; c4 < 8; ++c4) {
                const int4 kp = __ldg(kp4 + c4), kq = __ldg(ks4 + c4);
                float* sp = s + 32 * part + 4 * c4;
                if (!(kq.x == my_seq && kp.x <= my_pos)) sp[0] = -INFINITY;
                if (!(kq.y == my_seq && kp.y <= my_pos)) sp[1] = -INFINITY;
                if (!(kq.z == my_seq && kp.z <= my_pos)) sp[2] = -INFINITY;
                if (!(kq.w == my_seq && kp.w <= my_pos)) sp[3] = -INFINITY;
              }
            } else {
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                const int kidx = base + c;
                const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq &&
                                __ldg(p.k_pos + kidx) <= my_pos;
                if (!ok) s[32 * part + c] = -INFINITY;
              }
            }
          }
        }
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = fmaxf(s[k], s[8 + k]);
#pragma unroll
        for (int c = 16; c < 64; c += 8)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
        float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        // Row max over both halves.  Both halves have read all their S columns
        // once this barrier passes, so P chunks may overwrite S from here on.
        xch6[w][h][t] = mx;
        named_bar_sync(pair_bar, 256);
        mx = fmaxf(mx, xch6[w][h ^ 1][t]);
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;  // also true for -inf -> finite
        if (need) m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
          // Rescale this half's O_t columns in place (PV_t(it-1) has landed,
          // PV_t(it) waits for P).
#pragma unroll 1
          for (int c = 0; c < 64; c += 16) {
            uint32_t r[16];
            tmem_ld16(o_addr + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st16(o_addr + c, r);
          }
        }
        if (RCP_PINGPONG) named_bar_sync(my_turn, 512);
        if (t == 0 && w == 0 && h == 0) TRACE(9, it);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int part = 0; part < 2; ++part) {  // P chunk q = 2*part + h: 32 keys, 16 columns
          const int q = 2 * part + h;
          uint32_t pk[16];
          if (cls == kTileFull) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int ip = 16 * part + i;
              const float2 x = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
              float p0, p1;
              if ((ip & 7) < kPolyPairsPer8) {
                {
                  const float2 pp_ = ex2_poly_x2(x.x, x.y);
                  p0 = pp_.x;
                  p1 = pp_.y;
                }
              } else {
                p0 = ex2_approx(x.x);
                p1 = ex2_approx(x.y);
              }
              acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              pk[i] = pack_bf16x2(p0, p1);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int ip = 16 * part + i;
              const float2 x = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
              const float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
              acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              pk[i] = pack_bf16x2(p0, p1);
            }
          }
          tmem_st16(s_addr + 16 * q, pk);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bar_p[w][q]);
        }
        if (RCP_PINGPONG && hand_over) named_bar_arrive(their_turn, 512);
        if (t == 0 && w == 0 && h == 0) TRACE(10, it);
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
      } else {
        if (RCP_PINGPONG) named_bar_sync(my_turn, 512);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = 0u;
        tmem_st16(s_addr + 16 * h, pk);
        tmem_st16(s_addr + 16 * (h + 2), pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bar_p[w][h]);
        mbar_arrive(&bar_p[w][h + 2]);
        if (RCP_PINGPONG && hand_over) named_bar_arrive(their_turn, 512);
      }
      if (t == 0 && w == 0 && h == 0) TRACE(11, it);
      if (t == 0 && h == 0) TRACE(3 + 2 * w, it);
    }

    // epilogue: combine the halves' sums, O / l, LSE, optional merge
    if (it > 0) {
      mbar_wait(&bar_o[w], 0);
      tc_fence_after();
    }
    const bool merge = p.mode == RCP_MODE_MERGE;
    if (!(merge && it == 0)) {
      xch6[w][h][t] = l;
      named_bar_sync(pair_bar, 256);
      l += xch6[w][h ^ 1][t];
      const bool has = l > 0.f;
      const float inv = has ? 1.0f / l : 0.f;
      const float lse_new = has ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD + h * 64;
      float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
      MergeW mw;
      mw.lse = lse_new;
      mw.wa = 0.f;
      mw.wb = 1.f;
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t r[32];
        if (it > 0) {
          tmem_ld32(o_addr + c, r);
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
                                   __uint_as_float(r[4 * i + 2]) * inv,
                                   __uint_as_float(r[4 * i + 3]) * inv);
            if (merge) {
              const float4 a = dst[i];
              v = make_float4(merge_val(a.x, v.x, mw), merge_val(a.y, v.y, mw),
                              merge_val(a.z, v.z, mw), merge_val(a.w, v.w, mw));
            }
            dst[i] = v;
          }
        }
      }
      if (merge) named_bar_sync(pair_bar, 256);  // both halves read the old LSE before it is overwritten
      if (row_ok && h == 0) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ======================================================================
// v7: 1-CTA, 64-key blocks, Q in TMEM.  S = Q K^T is a TS MMA (A = the query
// tile from TMEM, B = K from shared memory): a 128x64 SS MMA needs 6 KB of
// shared-memory operands per 32 tensor cycles (192 B/clk, runs at 55 %),
// the TS form only K's 2 KB (64 B/clk, full rate).  TMEM (512 columns):
// O0 [0,128) | O1 [128,256) | Q0 [256,320) | Q1 [320,384) | S0 [384,448) |
// S1 [448,512): one S buffer per tile, P_t(j) packed over its first 32
// columns in two 32-key chunks (PV overlaps the exps), S_t(j+1) issued right
// after PV_t(j).  The softmax warps write their query rows into TMEM once;
// Q never touches shared memory, which leaves room for a 14-slot K/V ring.
// ======================================================================
constexpr int kSlots7 = 14;
constexpr uint32_t kSmem7Bytes = kSlots7 * kKVBytes + 1024;
constexpr uint32_t kTmemO7 = 0, kTmemQ7 = 256, kTmemS7 = 384;
static_assert(kSmem7Bytes <= 232448, "v7 shared memory exceeds 227 KB");

__global__ void __launch_bounds__(kThreads, 1) attn_fwd_v7_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sKV = smem;  // kSlots7 K/V blocks (16 KB each)

  __shared__ uint64_t bar_full[kSlots7], bar_empty[kSlots7];
  __shared__ uint64_t bar_qt[2], bar_s[2], bar_p[2][2], bar_o[2];
  __shared__ uint32_t tmem_slot;

  const int warp = static_cast<int>(warp_id());
  const int per_kv = p.n_qblk * p.group;
  const int kvh = static_cast<int>(blockIdx.x) / per_kv;
  const int rem = static_cast<int>(blockIdx.x) - kvh * per_kv;
  const int qblk = p.n_qblk - 1 - rem / p.group;
  const int head = kvh * p.group + rem % p.group;
  const int n = __ldg(p.act_n + qblk);
  const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots7; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_qt[t], 128);
      mbar_init(&bar_s[t], 1);
      mbar_init(&bar_p[t][0], 128);
      mbar_init(&bar_p[t][1], 128);
      mbar_init(&bar_o[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (K_j, V_j)
    if (elect_one() && n > 0) {
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      const uint64_t pol_kv = policy_evict_last();
      uint32_t ld = 0;
      uint32_t e_next = __ldg(act);
      for (int it = 0; it < n; ++it) {
        const int j = act_j(e_next);
        if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++ld) {
          const uint32_t slot = ld % kSlots7, ph = (ld / kSlots7) & 1;
          mbar_wait(&bar_empty[slot], ph ^ 1);
          TRACE(6 + kv, it);
          mbar_arrive_expect_tx(&bar_full[slot], kKVBytes);
          const CUtensorMap* map = kv ? &p.tm_v : &p.tm_k;
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sKV + slot * kKVBytes + h * kKVBoxBytes, map, &bar_full[slot], kvh * kD + h * 64,
                        j * kKRows, pol_kv);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (one elected lane)
    if (elect_one() && n > 0) {
      const uint32_t idesc_s = make_idesc_bf16_f32(kQRows, kKRows, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(kQRows, kD, 0, 1);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kKVBoxBytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots7], (ld / kSlots7) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int t, uint32_t ld) {  // TS: A = Q_t in TMEM, B = K (K-major)
        const uint32_t ka = k_lo + (((ld % kSlots7) * kKVBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma_ts_lo(tmem + kTmemS7 + t * kKRows, tmem + kTmemQ7 + t * 64 + kk * 8,
                    ka + (((kk >> 2) * kKVBoxBytes + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int t, uint32_t ld, int it) {  // two 32-key chunks as P lands
        const uint32_t va = v_lo + (((ld % kSlots7) * kKVBytes) >> 4);
        const uint32_t pa = tmem + kTmemS7 + t * kKRows;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          mbar_wait(&bar_p[t][q], it & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 2 * q; kk < 2 * q + 2; ++kk)
            mma_ts_lo(tmem + kTmemO7 + t * kD, pa + kk * 8, va + ((kk * 2048) >> 4), idesc_o,
                      (it > 0 || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(&bar_qt[0], 0);
      mbar_wait(&bar_qt[1], 0);
      tc_fence_after();
      wait_load(0);
      issue_s(0, 0);
      mma_commit(&bar_s[0]);
      issue_s(1, 0);
      mma_commit(&bar_s[1]);
      mma_commit(&bar_empty[0]);
      for (int it = 0; it < n; ++it) {
        const bool last = it + 1 == n;
        const uint32_t ldv = 2 * it + 1, ldk1 = 2 * it + 2;
        wait_load(ldv);
        issue_pv(0, ldv, it);
        TRACE(0, it);
        if (last) mma_commit(&bar_o[0]);
        if (!last) {
          wait_load(ldk1);
          issue_s(0, ldk1);
          mma_commit(&bar_s[0]);
        }
        issue_pv(1, ldv, it);
        TRACE(1, it);
        if (last) mma_commit(&bar_o[1]);
        mma_commit(&bar_empty[ldv % kSlots7]);
        if (!last) {
          issue_s(1, ldk1);
          mma_commit(&bar_s[1]);
          mma_commit(&bar_empty[ldk1 % kSlots7]);
        }
        TRACE(14, it);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int w = (warp - 4) >> 2;                                 // query tile 0 / 1
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * w;  // row inside the tile
    const int row = (2 * qblk + w) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO7 + w * kD;
    const uint32_t s_addr = lane_base + kTmemS7 + w * kKRows;
    // this row of Q into TMEM (A operand layout: column c holds dims 2c, 2c+1)
    {
      const uint4* src = reinterpret_cast<const uint4*>(p.q + static_cast<int64_t>(row) * p.q_stride + head * kD);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 v = row_ok && n > 0 ? __ldg(src + half * 8 + i) : make_uint4(0, 0, 0, 0);
          r[4 * i] = v.x;
          r[4 * i + 1] = v.y;
          r[4 * i + 2] = v.z;
          r[4 * i + 3] = v.w;
        }
        tmem_st32(lane_base + kTmemQ7 + w * 64 + half * 32, r);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bar_qt[w]);
    }
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    int it = 0;
    for (; it < n; ++it) {
      const uint32_t e = e_next;
      if (it + 1 < n) e_next = __ldg(act + it + 1);
      const int j = act_j(e);
      const int cls = act_cls(e, w);
      // S_t(it) complete also means PV_t(it-1) is: O_t may be rescaled in place.
      mbar_wait(&bar_s[w], it & 1);
      tc_fence_after();
      if (t == 0) TRACE(2 + 2 * w, it);
      if (cls != kTileEmpty) {  // warp-uniform
        uint32_t sr[64];
        tmem_ld32(s_addr, sr);
        tmem_ld32(s_addr + 32, sr + 32);
        tmem_ld_wait();
        float s[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
        if (cls == kTilePartial) {
          const int base = j * kKRows;
          if (base + kKRows <= p.tk) {
            const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
            const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
              const int4 kp = __ldg(kp4 + c4), kq = __ldg(ks4 + c4);
              if (!(kq.x == my_seq && kp.x <= my_pos)) s[4 * c4 + 0] = -INFINITY;
              if (!(kq.y == my_seq && kp.y <= my_pos)) s[4 * c4 + 1] = -INFINITY;
              if (!(kq.z == my_seq && kp.z <= my_pos)) s[4 * c4 + 2] = -INFINITY;
              if (!(kq.w == my_seq && kp.w <= my_pos)) s[4 * c4 + 3] = -INFINITY;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 64; ++c) {
              const int kidx = base + c;
              const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq &&
                              __ldg(p.k_pos + kidx) <= my_pos;
              if (!ok) s[c] = -INFINITY;
            }
          }
        }
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = fmaxf(s[k], s[8 + k]);
#pragma unroll
        for (int c = 16; c < 64; c += 8)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;  // also true for -inf -> finite
        if (need) m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
#pragma unroll 1
          for (int c = 0; c < kD; c += 32) {
            uint32_t r[32];
            tmem_ld32(o_addr + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st32(o_addr + c, r);
          }
        }
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int q = 0; q < 2; ++q) {  // P chunk q: keys [32q, 32q+32) -> columns [16q, 16q+16)
          uint32_t pk[16];
          if (cls == kTileFull) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int ip = 16 * q + i;
              const float2 x = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
              float p0, p1;
              if ((ip & 7) < kPolyPairsPer8) {
                {
                  const float2 pp_ = ex2_poly_x2(x.x, x.y);
                  p0 = pp_.x;
                  p1 = pp_.y;
                }
              } else {
                p0 = ex2_approx(x.x);
                p1 = ex2_approx(x.y);
              }
              acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              pk[i] = pack_bf16x2(p0, p1);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int ip = 16 * q + i;
              const float2 x = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
              const float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
              acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              pk[i] = pack_bf16x2(p0, p1);
            }
          }
          tmem_st16(s_addr + 16 * q, pk);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bar_p[w][q]);
        }
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
      } else {
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
        tmem_st32(s_addr, pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bar_p[w][0]);
        mbar_arrive(&bar_p[w][1]);
      }
      if (t == 0) TRACE(3 + 2 * w, it);
    }

    // epilogue: O / l, LSE, optional merge into the running (O, LSE)
    if (it > 0) {
      mbar_wait(&bar_o[w], 0);
      tc_fence_after();
    }
    const bool merge = p.mode == RCP_MODE_MERGE;
    if (!(merge && it == 0)) {
      const bool has = l > 0.f;
      const float inv = has ? 1.0f / l : 0.f;
      const float lse_new = has ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD;
      float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
      MergeW mw;
      mw.lse = lse_new;
      mw.wa = 0.f;
      mw.wb = 1.f;
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
      for (int c = 0; c < kD; c += 32) {
        uint32_t r[32];
        if (it > 0) {
          tmem_ld32(o_addr + c, r);
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
                                   __uint_as_float(r[4 * i + 2]) * inv,
                                   __uint_as_float(r[4 * i + 3]) * inv);
            if (merge) {
              const float4 a = dst[i];
              v = make_float4(merge_val(a.x, v.x, mw), merge_val(a.y, v.y, mw),
                              merge_val(a.z, v.z, mw), merge_val(a.w, v.w, mw));
            }
            dst[i] = v;
          }
        }
      }
      if (row_ok) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ======================================================================
// v5: CTA-pair (cta_group::2) variant.  Cluster of 2 CTAs = 2 x 128 query rows
// of one query head (CTA r owns query tile 2*qblk + r).  Key blocks are 128
// keys; the leader CTA issues M=256 MMAs: S = Q K^T (N=128 keys, B split by
// keys: CTA r holds keys [64r, 64r+64) of the block) and O += P V (N=128 dims,
// B split by dims: CTA r holds dims [64r, 64r+64) of all 128 keys).  Per SM
// this halves the operand traffic through shared memory (~94 B/clk at full
// tensor rate instead of ~156 for the 1-CTA N=64 form).  TMEM per CTA: O
// [0,128) | S0 [128,256) | S1 [256,384); S double-buffered as in v4.  Two
// softmax warpgroups per CTA split the 128 score columns (64 each) and
// exchange the row max through shared memory once per block.
// ======================================================================
// S/P buffers of v5: three 128-column TMEM buffers after O (O 128 + 3 x 128 =
// 512 columns), so S(j+3) is issued after PV(j) and the softmax of block j+1
// finds S(j+1) ready even when P(j) of the slowest of the 16 softmax warps
// (two SMs) is late.
// Softmax column groups of v5: each of kSmWG2 warpgroups per CTA owns
// 128 / kSmWG2 score columns of every row (4 -> 4 softmax warps per SMSP to
// hide MUFU / TMEM latency: measured slower, 1050 vs 1114 TF/s; 2 -> 384 threads, the default).
#ifndef RCP_V5_GROUPS
#define RCP_V5_GROUPS 2
#endif
constexpr int kSmWG2 = RCP_V5_GROUPS;
constexpr int kCols2 = 128 / kSmWG2;
constexpr int kThreads2 = 128 + 128 * kSmWG2;
static_assert(kSmWG2 == 2 || kSmWG2 == 4, "v5 softmax groups must be 2 or 4");
constexpr int kSBuf2 = 3;
constexpr int kKRows2 = 128;
constexpr int kSlots2 = 11;
constexpr uint32_t kSlot2Bytes = 16384;  // K half: 64 keys x 128 dims; V half: 128 keys x 64 dims
constexpr uint32_t kSmem2Bytes = kQTileBytes + kSlots2 * kSlot2Bytes + 1024;
constexpr uint32_t kTmemO2 = 0, kTmemS2 = 128;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    attn_fwd_2cta_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // this CTA's 128-row query tile
  uint8_t* sKV = smem + kQTileBytes;   // kSlots2 half blocks (K half / V half alternate)

  __shared__ uint64_t bar_q, bar_full[kSlots2], bar_empty[kSlots2];
  __shared__ uint64_t bar_s[kSBuf2], bar_p[kSBuf2], bar_pv, bar_o;
  __shared__ uint32_t tmem_slot;
  __shared__ float xch[kSmWG2][128];

  const int warp = static_cast<int>(warp_id());
  const int rank = static_cast<int>(cluster_rank());
  const int pair = static_cast<int>(blockIdx.x) >> 1;
  const int per_kv = p.n_qblk * p.group;
  const int kvh = pair / per_kv;
  const int rem = pair - kvh * per_kv;
  const int qblk = p.n_qblk - 1 - rem / p.group;
  const int head = kvh * p.group + rem % p.group;
  const int n = __ldg(p.act_n + qblk);
  const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kSlots2; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int b = 0; b < kSBuf2; ++b) {
      mbar_init(&bar_s[b], 1);
      mbar_init(&bar_p[b], 2 * 4 * kSmWG2);  // every softmax warp of both CTAs
    }
    mbar_init(&bar_pv, 1);
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
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one() && n > 0) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      if (rank == 0) mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes);
      for (int h = 0; h < 2; ++h)
        tma_load_2d_pair(sQ + h * kQBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                         (2 * qblk + rank) * kQRows, pol_q);
      uint32_t ld = 0;
      uint32_t e_next = __ldg(act);
      for (int it = 0; it < n; ++it) {
        const int j = act_j(e_next);
        if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++ld) {
          const uint32_t slot = ld % kSlots2, ph = (ld / kSlots2) & 1;
          mbar_wait(&bar_empty[slot], ph ^ 1);
          TRACE(6 + kv, it);
          if (rank == 0) mbar_arrive_expect_tx(&bar_full[slot], 2 * kSlot2Bytes);
          uint8_t* dst = sKV + slot * kSlot2Bytes;
          if (kv == 0) {  // K half: keys [j*128 + 64 r, +64), all 128 dims (two 8 KB boxes)
            for (int h = 0; h < 2; ++h)
              tma_load_2d_pair(dst + h * 8192, &p.tm_k, &bar_full[slot], kvh * kD + h * 64,
                               j * kKRows2 + rank * 64, pol_kv);
          } else {        // V half: all 128 keys, dims [64 r, 64 r + 64)
            tma_load_2d_pair(dst, &p.tm_v, &bar_full[slot], kvh * kD + rank * 64, j * kKRows2, pol_kv);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA, one elected lane)
    if (rank == 0 && n > 0 && elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16_f32(256, kKRows2, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(256, kD, 0, 1);
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kSlot2Bytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots2], (ld / kSlots2) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int buf, uint32_t ld) {
        const uint32_t ka = k_lo + (((ld % kSlots2) * kSlot2Bytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma2_ss_lo(tmem + kTmemS2 + buf * 128, q_lo + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                     ka + (((kk >> 2) * 8192 + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int buf, uint32_t ld, bool acc) {
        const uint32_t va = v_lo + (((ld % kSlots2) * kSlot2Bytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kKRows2 / 16; ++kk)
          mma2_ts_lo(tmem + kTmemO2, tmem + kTmemS2 + buf * 128 + kk * 8, va + ((kk * 2048) >> 4), idesc_o,
                     (acc || kk > 0) ? 1u : 0u);
      };
      mbar_wait(&bar_q, 0);
      for (int b = 0; b < kSBuf2 && b < n; ++b) {
        wait_load(2 * b);
        issue_s(b, 2 * b);
        commit2_mc(&bar_s[b]);
        commit2_mc(&bar_empty[(2 * b) % kSlots2]);
      }
      int buf = 0;
      uint32_t ph = 0;
      for (int it = 0; it < n; ++it) {
        const bool last = it + 1 == n;
        const uint32_t ldv = 2 * it + 1, ldk2 = 2 * (it + kSBuf2);
        wait_load(ldv);
        mbar_wait(&bar_p[buf], ph);
        tc_fence_after();
        TRACE(0, it);
        issue_pv(buf, ldv, it > 0);
        TRACE(8, it);
        commit2_mc(last ? &bar_o : &bar_pv);
        commit2_mc(&bar_empty[ldv % kSlots2]);
        if (it + kSBuf2 < n) {
          wait_load(ldk2);
          TRACE(9, it);
          issue_s(buf, ldk2);
          TRACE(10, it);
          commit2_mc(&bar_s[buf]);
          commit2_mc(&bar_empty[ldk2 % kSlots2]);
        }
        TRACE(1, it);
        if (++buf == kSBuf2) {
          buf = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
#if RCP_TRACE && !defined(RCP_TRACE_PERWARP)
  } else if (warp == 3) {
    // trace builds: an idle warp timestamps S and PV completions (MMA latency)
    if (elect_one() && p.trace && n > 0) {
      // completion order: S(0..kSBuf2-1), then PV(j), S(j+kSBuf2), PV(j+1), ...
      for (int it = 0; it < kSBuf2 && it < n; ++it) {
        mbar_wait(&bar_s[it], 0);
        TRACE(11, it);
      }
      for (int it = 0; it + 1 < n; ++it) {
        mbar_wait(&bar_pv, it & 1);
        TRACE(14, it);
        if (it + kSBuf2 < n) {
          mbar_wait(&bar_s[it % kSBuf2], ((it + kSBuf2) / kSBuf2) & 1);
          TRACE(11, it + kSBuf2);
        }
      }
    }
    __syncwarp();
#endif
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue (both CTAs)
    const int h = (warp - 4) >> 2;                                // column group of the 128-key block
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * h;  // row inside this CTA's tile
    const int row = (2 * qblk + rank) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO2 + h * kCols2;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;  // l: this group's partial row sum
    const uint32_t row_bar = 1 + (warp & 3), row_bar_threads = 32 * kSmWG2;  // warps of this row quarter
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    int it = 0;
    for (; it < n; ++it) {
      const int buf = it % kSBuf2;
      const uint32_t s_addr = lane_base + kTmemS2 + buf * 128 + h * kCols2;
      const uint32_t p_addr = lane_base + kTmemS2 + buf * 128 + h * (kCols2 / 2);
      const uint32_t e = e_next;
      if (it + 1 < n) e_next = __ldg(act + it + 1);
      const int j = act_j(e);
      const int cls = act_cls(e, rank);
      mbar_wait(&bar_s[buf], (it / kSBuf2) & 1);
      tc_fence_after();
      if (t == 0 && h == 0) TRACE(2 + 2 * rank, it);
#if RCP_TRACE
      if ((threadIdx.x & 31) == 0 && p.trace && blockIdx.x < kTraceCtas && it < kTraceIters)
        (void)0;
#endif
      if (cls != kTileEmpty) {  // uniform across the CTA
        uint32_t sr[kCols2];
#pragma unroll
        for (int c = 0; c < kCols2; c += 32) tmem_ld32(s_addr + c, sr + c);
        tmem_ld_wait();
        float s[kCols2];
#pragma unroll
        for (int c = 0; c < kCols2; ++c) s[c] = __uint_as_float(sr[c]);
        if (cls == kTilePartial) {
          const int base = j * kKRows2 + h * kCols2;
          if (j * kKRows2 + kKRows2 <= p.tk) {
            const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
            const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll
            for (int c4 = 0; c4 < kCols2 / 4; ++c4) {
              const int4 kp = __ldg(kp4 + c4), kq = __ldg(ks4 + c4);
              if (!(kq.x == my_seq && kp.x <= my_pos)) s[4 * c4 + 0] = -INFINITY;
              if (!(kq.y == my_seq && kp.y <= my_pos)) s[4 * c4 + 1] = -INFINITY;
              if (!(kq.z == my_seq && kp.z <= my_pos)) s[4 * c4 + 2] = -INFINITY;
              if (!(kq.w == my_seq && kp.w <= my_pos)) s[4 * c4 + 3] = -INFINITY;
            }
          } else {
#pragma unroll
            for (int c = 0; c < kCols2; ++c) {
              const int kidx = base + c;
              const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq &&
                              __ldg(p.k_pos + kidx) <= my_pos;
              if (!ok) s[c] = -INFINITY;
            }
          }
        }
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
        for (int c = 8; c < kCols2; c += 8)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
        float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        // Row max over the groups (same order everywhere -> identical m).  All
        // groups have read their S columns once this barrier passes, so P
        // (the first 64 columns of the buffer) may overwrite S from here on.
        xch[h][t] = mx;
        named_bar_sync(row_bar, row_bar_threads);
        mx = xch[0][t];
#pragma unroll
        for (int g = 1; g < kSmWG2; ++g) mx = fmaxf(mx, xch[g][t]);
        if (t == 0 && h == 0) TRACE(12 + rank, it);
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;
        if (need) m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
        uint32_t pk[kCols2 / 2];
        if (cls == kTileFull) {
#pragma unroll
          for (int i = 0; i < kCols2 / 2; ++i) {
            const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
            float p0, p1;
            if ((i & 7) < kPolyPairsPer8) {
              {
                const float2 pp_ = ex2_poly_x2(x.x, x.y);
                p0 = pp_.x;
                p1 = pp_.y;
              }
            } else {
              p0 = ex2_approx(x.x);
              p1 = ex2_approx(x.y);
            }
            acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
            pk[i] = pack_bf16x2(p0, p1);
          }
        } else {
#pragma unroll
          for (int i = 0; i < kCols2 / 2; ++i) {
            const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
            const float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
            acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
            pk[i] = pack_bf16x2(p0, p1);
          }
        }
        if (kCols2 == 64) tmem_st32(p_addr, pk);
        else tmem_st16(p_addr, pk);
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
          mbar_wait(&bar_pv, (it - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < kCols2; c += 32) {
            uint32_t r[32];
            tmem_ld32(o_addr + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st32(o_addr + c, r);
          }
        }
      } else {
        uint32_t pk[kCols2 / 2];
#pragma unroll
        for (int i = 0; i < kCols2 / 2; ++i) pk[i] = 0u;
        if (kCols2 == 64) tmem_st32(p_addr, pk);
        else tmem_st16(p_addr, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      if (t == 0 && h == 0) TRACE(3 + 2 * rank, it);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) arrive_leader(&bar_p[buf]);
      if (t == 0 && h == 0 && rank == 0) TRACE(15, it);
#if RCP_TRACE && defined(RCP_TRACE_PERWARP)
      if ((threadIdx.x & 31) == 0 && p.trace && blockIdx.x < kTraceCtas && it < kTraceIters)
        p.trace[(blockIdx.x * kTraceIters + it) * kTraceEv + 8 + (warp - 4)] = clock64();
#endif
    }
    // epilogue: combine the halves' sums, O / l, LSE, optional merge
    if (it > 0) {
      mbar_wait(&bar_o, 0);
      tc_fence_after();
    }
    const bool merge = p.mode == RCP_MODE_MERGE;
    if (!(merge && it == 0)) {
      xch[h][t] = l;
      named_bar_sync(row_bar, row_bar_threads);
      l = xch[0][t];
#pragma unroll
      for (int g = 1; g < kSmWG2; ++g) l += xch[g][t];
      const bool has = l > 0.f;
      const float inv = has ? 1.0f / l : 0.f;
      const float lse_new = has ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD + h * kCols2;
      float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
      MergeW mw;
      mw.lse = lse_new;
      mw.wa = 0.f;
      mw.wb = 1.f;
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
      for (int c = 0; c < kCols2; c += 32) {
        uint32_t r[32];
        if (it > 0) {
          tmem_ld32(o_addr + c, r);
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
      if (merge) named_bar_sync(row_bar, row_bar_threads);  // every group read the old LSE before it is overwritten
      if (row_ok && h == 0) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's TMEM / smem stay live until the leader's MMAs are done
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
  }
}

// ======================================================================
// v8: CTA pairs (as v5: M=256 MMAs, 128-key blocks, B split across the
// pair), but the two softmax warpgroups of a CTA take ALTERNATE key blocks
// instead of splitting every block's columns: group x owns blocks it ≡ x
// (mod 2) with full 128-column rows (no per-block row-max exchange), its own
// S buffer and its own O accumulator and (m, l); the two partials are folded
// once in the epilogue with the exact LSE merge.  TMEM per CTA: O_a [0,128) |
// O_b [128,256) | S_a [256,384) | S_b [384,512).  While one group's
// PV -> S(next) chain runs on the tensor cores, the other group's softmax
// keeps the SMSPs busy.
// ======================================================================
constexpr uint32_t kTmemO8 = 0, kTmemS8 = 256;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_v8_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // this CTA's 128-row query tile
  uint8_t* sKV = smem + kQTileBytes;   // kSlots2 half blocks (K half / V half alternate)

  __shared__ uint64_t bar_q, bar_full[kSlots2], bar_empty[kSlots2];
  __shared__ uint64_t bar_s[2], bar_p[2], bar_o[2];
  __shared__ uint32_t tmem_slot;
  __shared__ float xch8[2][2][128];  // [group][m | l][row]

  const int warp = static_cast<int>(warp_id());
  const int rank = static_cast<int>(cluster_rank());
  const int pair = static_cast<int>(blockIdx.x) >> 1;
  const int per_kv = p.n_qblk * p.group;
  const int kvh = pair / per_kv;
  const int rem = pair - kvh * per_kv;
  const int qblk = p.n_qblk - 1 - rem / p.group;
  const int head = kvh * p.group + rem % p.group;
  const int n = __ldg(p.act_n + qblk);
  const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kSlots2; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&bar_s[x], 1);
      mbar_init(&bar_p[x], 2 * 4);  // the 4 warps of group x in both CTAs
      mbar_init(&bar_o[x], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one() && n > 0) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      if (rank == 0) mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes);
      for (int h = 0; h < 2; ++h)
        tma_load_2d_pair(sQ + h * kQBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                         (2 * qblk + rank) * kQRows, pol_q);
      uint32_t ld = 0;
      uint32_t e_next = __ldg(act);
      for (int it = 0; it < n; ++it) {
        const int j = act_j(e_next);
        if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++ld) {
          const uint32_t slot = ld % kSlots2, ph = (ld / kSlots2) & 1;
          mbar_wait(&bar_empty[slot], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&bar_full[slot], 2 * kSlot2Bytes);
          uint8_t* dst = sKV + slot * kSlot2Bytes;
          if (kv == 0) {  // K half: keys [j*128 + 64 r, +64), all 128 dims (two 8 KB boxes)
            for (int h = 0; h < 2; ++h)
              tma_load_2d_pair(dst + h * 8192, &p.tm_k, &bar_full[slot], kvh * kD + h * 64,
                               j * kKRows2 + rank * 64, pol_kv);
          } else {        // V half: all 128 keys, dims [64 r, 64 r + 64)
            tma_load_2d_pair(dst, &p.tm_v, &bar_full[slot], kvh * kD + rank * 64, j * kKRows2, pol_kv);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA, one elected lane)
    if (rank == 0 && n > 0 && elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16_f32(256, kKRows2, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(256, kD, 0, 1);
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kSlot2Bytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots2], (ld / kSlots2) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int x, uint32_t ld) {
        const uint32_t ka = k_lo + (((ld % kSlots2) * kSlot2Bytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma2_ss_lo(tmem + kTmemS8 + x * 128, q_lo + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                     ka + (((kk >> 2) * 8192 + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int x, uint32_t ld, bool acc) {
        const uint32_t va = v_lo + (((ld % kSlots2) * kSlot2Bytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kKRows2 / 16; ++kk)
          mma2_ts_lo(tmem + kTmemO8 + x * kD, tmem + kTmemS8 + x * 128 + kk * 8, va + ((kk * 2048) >> 4),
                     idesc_o, (acc || kk > 0) ? 1u : 0u);
      };
      mbar_wait(&bar_q, 0);
      for (int b = 0; b < 2 && b < n; ++b) {
        wait_load(2 * b);
        issue_s(b, 2 * b);
        commit2_mc(&bar_s[b]);
        commit2_mc(&bar_empty[(2 * b) % kSlots2]);
      }
      for (int it = 0; it < n; ++it) {
        const int x = it & 1;
        const uint32_t ldv = 2 * it + 1, ldk2 = 2 * (it + 2);
        wait_load(ldv);
        mbar_wait(&bar_p[x], (it >> 1) & 1);
        tc_fence_after();
        TRACE(0, it);
        issue_pv(x, ldv, it >= 2);
        if (it + 2 >= n) commit2_mc(&bar_o[x]);  // last block of group x
        commit2_mc(&bar_empty[ldv % kSlots2]);
        if (it + 2 < n) {
          wait_load(ldk2);
          issue_s(x, ldk2);
          commit2_mc(&bar_s[x]);
          commit2_mc(&bar_empty[ldk2 % kSlots2]);
        }
        TRACE(1, it);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax (group x: blocks x, x+2, ...)
    const int x = (warp - 4) >> 2;
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * x;  // row inside this CTA's tile
    const int row = (2 * qblk + rank) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t s_addr = lane_base + kTmemS8 + x * 128;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    int cnt = 0;  // blocks processed by this group
    for (int it = x; it < n; it += 2, ++cnt) {
      const uint32_t e = __ldg(act + it);
      const int j = act_j(e);
      const int cls = act_cls(e, rank);
      // S_x(it) complete also means PV_x(it-2) is: O_x may be rescaled in place.
      mbar_wait(&bar_s[x], cnt & 1);
      tc_fence_after();
      if (t == 0) TRACE(2 + 2 * x, it);
      if (cls != kTileEmpty) {  // uniform across the pair for this block
        float s[128];
        {
          uint32_t sr[128];
#pragma unroll
          for (int c = 0; c < 128; c += 32) tmem_ld32(s_addr + c, sr + c);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 128; ++c) s[c] = __uint_as_float(sr[c]);
        }
        if (cls == kTilePartial) {
          const int base = j * kKRows2;
          if (base + kKRows2 <= p.tk) {
            const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
            const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll
            for (int c4 = 0; c4 < 32; ++c4) {
              const int4 kp = __ldg(kp4 + c4), kq = __ldg(ks4 + c4);
              if (!(kq.x == my_seq && kp.x <= my_pos)) s[4 * c4 + 0] = -INFINITY;
              if (!(kq.y == my_seq && kp.y <= my_pos)) s[4 * c4 + 1] = -INFINITY;
              if (!(kq.z == my_seq && kp.z <= my_pos)) s[4 * c4 + 2] = -INFINITY;
              if (!(kq.w == my_seq && kp.w <= my_pos)) s[4 * c4 + 3] = -INFINITY;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 128; ++c) {
              const int kidx = base + c;
              const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq &&
                              __ldg(p.k_pos + kidx) <= my_pos;
              if (!ok) s[c] = -INFINITY;
            }
          }
        }
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = fmaxf(s[k], s[8 + k]);
#pragma unroll
        for (int c = 16; c < 128; c += 8)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;  // also true for -inf -> finite
        if (need) m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        if (__any_sync(0xffffffffu, f != 1.0f && cnt > 0)) {
          const uint32_t o_x = lane_base + kTmemO8 + x * kD;
#pragma unroll 1
          for (int c = 0; c < kD; c += 16) {
            uint32_t r[16];
            tmem_ld16(o_x + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st16(o_x + c, r);
          }
        }
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // 32 keys -> 16 packed columns per chunk
          uint32_t pk[16];
          if (cls == kTileFull) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int ip = 16 * q + i;
              const float2 xx = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
              float p0, p1;
              if ((ip & 7) < kPolyPairsPer8) {
                {
                  const float2 pp_ = ex2_poly_x2(xx.x, xx.y);
                  p0 = pp_.x;
                  p1 = pp_.y;
                }
              } else {
                p0 = ex2_approx(xx.x);
                p1 = ex2_approx(xx.y);
              }
              acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              pk[i] = pack_bf16x2(p0, p1);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int ip = 16 * q + i;
              const float2 xx = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
              const float p0 = ex2_approx(xx.x), p1 = ex2_approx(xx.y);
              acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              pk[i] = pack_bf16x2(p0, p1);
            }
          }
          tmem_st16(s_addr + 16 * q, pk);
        }
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
      } else {
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
        tmem_st32(s_addr, pk);
        tmem_st32(s_addr + 32, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      if (t == 0) TRACE(3 + 2 * x, it);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) arrive_leader(&bar_p[x]);
    }

    // epilogue: fold the two groups' partials (exact LSE merge), O / l, LSE, optional merge
    const bool has_a = n > 0, has_b = n > 1;
    if (has_a) {
      mbar_wait(&bar_o[0], 0);
      if (has_b) mbar_wait(&bar_o[1], 0);
      tc_fence_after();
    }
    const bool merge = p.mode == RCP_MODE_MERGE;
    xch8[x][0][t] = m;
    xch8[x][1][t] = l;
    named_bar_sync(1 + (warp & 3), 64);  // warps w and w+4 share rows
    const float ma = xch8[0][0][t], la = xch8[0][1][t];
    const float mb = xch8[1][0][t], lb = xch8[1][1][t];
    if (!(merge && n == 0)) {
      const float mt = fmaxf(ma, mb);
      const float fa = (ma == -INFINITY) ? 0.f : ex2_approx(ma - mt);
      const float fb = (mb == -INFINITY) ? 0.f : ex2_approx(mb - mt);
      const float lt = la * fa + lb * fb;
      const bool has = lt > 0.f;
      const float inv = has ? 1.0f / lt : 0.f;
      const float lse_new = has ? (mt + __log2f(lt)) * 0.69314718055994530942f : -INFINITY;
      // group x writes output columns [64x, 64x + 64)
      float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD + x * 64;
      float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
      MergeW mw;
      mw.lse = lse_new;
      mw.wa = 0.f;
      mw.wb = 1.f;
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
      const float wa = fa * inv, wb = fb * inv;
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t ra[32], rb[32];
        if (has_a) {
          tmem_ld32(lane_base + kTmemO8 + x * 64 + c, ra);
          if (has_b) tmem_ld32(lane_base + kTmemO8 + kD + x * 64 + c, rb);
          tmem_ld_wait();
        }
        if (!has_a) {
#pragma unroll
          for (int i = 0; i < 32; ++i) ra[i] = 0u;
        }
        if (!has_b) {
#pragma unroll
          for (int i = 0; i < 32; ++i) rb[i] = 0u;
        }
        if (row_ok) {
          float4* dst = reinterpret_cast<float4*>(orow + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 v;
            v.x = __uint_as_float(ra[4 * i]) * wa + __uint_as_float(rb[4 * i]) * wb;
            v.y = __uint_as_float(ra[4 * i + 1]) * wa + __uint_as_float(rb[4 * i + 1]) * wb;
            v.z = __uint_as_float(ra[4 * i + 2]) * wa + __uint_as_float(rb[4 * i + 2]) * wb;
            v.w = __uint_as_float(ra[4 * i + 3]) * wa + __uint_as_float(rb[4 * i + 3]) * wb;
            if (merge) {
              const float4 a = dst[i];
              v = make_float4(merge_val(a.x, v.x, mw), merge_val(a.y, v.y, mw), merge_val(a.z, v.z, mw),
                              merge_val(a.w, v.w, mw));
            }
            dst[i] = v;
          }
        }
      }
      if (merge) named_bar_sync(1 + (warp & 3), 64);  // both groups read the old LSE before it is overwritten
      if (row_ok && x == 0) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's TMEM / smem stay live until the leader's MMAs are done
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
  }
}



// ======================================================================
// v9: persistent v4.  One CTA per SM streams (query block, head) items in
// v4's heavy-first order, claimed dynamically: the producer lane takes the
// next item from a global counter and hands it to the MMA and softmax warps
// through a 4-deep shared-memory ring (full / empty mbarriers); the roles keep
// their barrier phases across items — S/P/K/V phases from a global block
// counter, Q / O phases from the count of non-empty items — so the next
// item's Q load, first K/V loads and first two S MMAs overlap the current
// item's drain and epilogue, and TMEM allocation, barrier init and descriptor
// prefetch happen once per CTA.  Two extra hand-offs: bar_qfree (MMA commit
// after an item's last S: Q smem may be reloaded) and bar_ofree (the tile's
// softmax threads read O out: the next item's first PV may overwrite it).
// ======================================================================
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_v9_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + 2 * kQTileBytes;

  __shared__ uint64_t bar_q, bar_qfree, bar_full[kSlots], bar_empty[kSlots];
  __shared__ uint64_t bar_s[2][2], bar_p[2][2], bar_pv[2], bar_o[2], bar_ofree[2];
  constexpr int kItemSlots = 4;
  __shared__ uint64_t bar_item_full[kItemSlots], bar_item_empty[kItemSlots];
  __shared__ int item_buf[kItemSlots];
  __shared__ uint32_t tmem_slot;

  const int warp = static_cast<int>(warp_id());
  const int per_kv = p.n_qblk * p.group;
  // consumer side of the item ring: k-th item of this CTA (>= n_items: done)
  // (whole_warp: all 32 lanes call, lane 0 releases the slot after every
  // lane has read it; otherwise a single elected lane reads and releases)
  auto next_item = [&](uint32_t k, bool whole_warp) -> int {
    const uint32_t sl = k % kItemSlots;
    mbar_wait(&bar_item_full[sl], (k / kItemSlots) & 1);
    const int item = reinterpret_cast<volatile int*>(item_buf)[sl];
    if (whole_warp) __syncwarp();
    if (!whole_warp || (threadIdx.x & 31) == 0) mbar_arrive(&bar_item_empty[sl]);
    return item;
  };
  const int n_items = per_kv * p.hkv;
  auto item_coords = [&](int item, int& qblk, int& head, int& kvh) {
    kvh = item / per_kv;
    const int rem = item - kvh * per_kv;
    qblk = p.n_qblk - 1 - rem / p.group;
    head = kvh * p.group + rem % p.group;
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    mbar_init(&bar_qfree, 1);
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t][0], 1);
      mbar_init(&bar_s[t][1], 1);
      mbar_init(&bar_p[t][0], 128);
      mbar_init(&bar_p[t][1], 128);
      mbar_init(&bar_pv[t], 1);
      mbar_init(&bar_o[t], 1);
      mbar_init(&bar_ofree[t], 128);
    }
    for (int i = 0; i < kItemSlots; ++i) {
      mbar_init(&bar_item_full[i], 1);
      mbar_init(&bar_item_empty[i], 1 + 8);  // MMA lane + lane 0 of each softmax warp
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t ld = 0, qi = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t sl = k % kItemSlots;
        mbar_wait(&bar_item_empty[sl], ((k / kItemSlots) & 1) ^ 1);
        const int item = atomicAdd(p.item_ctr, 1);
        reinterpret_cast<volatile int*>(item_buf)[sl] = item;
        mbar_arrive(&bar_item_full[sl]);
        if (item >= n_items) break;
        int qblk, head, kvh;
        item_coords(item, qblk, head, kvh);
        const int n = __ldg(p.act_n + qblk);
        if (n == 0) continue;
        const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
        if (qi > 0) mbar_wait(&bar_qfree, (qi - 1) & 1);  // previous item's S MMAs read Q
        mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes);
        for (int t = 0; t < 2; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sQ + t * kQTileBytes + h * kQBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                        (2 * qblk + t) * kQRows, pol_q);
        uint32_t e_next = __ldg(act);
        for (int it = 0; it < n; ++it) {
          const int j = act_j(e_next);
          if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++ld) {
            const uint32_t slot = ld % kSlots, ph = (ld / kSlots) & 1;
            mbar_wait(&bar_empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&bar_full[slot], kKVBytes);
            const CUtensorMap* map = kv ? &p.tm_v : &p.tm_k;
            for (int h = 0; h < 2; ++h)
              tma_load_2d(sKV + slot * kKVBytes + h * kKVBoxBytes, map, &bar_full[slot],
                          kvh * kD + h * 64, j * kKRows, pol_kv);
          }
        }
        ++qi;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16_f32(kQRows, kKRows, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(kQRows, kD, 0, 1);
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kKVBoxBytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots], (ld / kSlots) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int t, int buf, uint32_t ld) {
        const uint32_t qa = q_lo + ((t * kQTileBytes) >> 4);
        const uint32_t ka = k_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t d = tmem + kTmemS + (2 * t + buf) * kKRows;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma_ss_lo(d, qa + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                    ka + (((kk >> 2) * kKVBoxBytes + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int t, int buf, uint32_t ld, bool acc) {
        const uint32_t va = v_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t pa = tmem + kTmemS + (2 * t + buf) * kKRows;
#pragma unroll
        for (int kk = 0; kk < kKRows / 16; ++kk)
          mma_ts_lo(tmem + kTmemO + t * kD, pa + kk * 8, va + ((kk * 2048) >> 4), idesc_o,
                    (acc || kk > 0) ? 1u : 0u);
      };
      uint32_t g0 = 0, qi = 0;  // global index of the item's first block; non-empty items so far
      for (uint32_t k = 0;; ++k) {
        const int item = next_item(k, false);
        if (item >= n_items) break;
        int qblk, head, kvh;
        item_coords(item, qblk, head, kvh);
        const int n = __ldg(p.act_n + qblk);
        if (n == 0) continue;
        mbar_wait(&bar_q, qi & 1);
        tc_fence_after();
        // prologue: S(g0), S(g0 + 1) for both tiles
        {
          const int b0 = g0 & 1;
          wait_load(2 * g0);
          issue_s(0, b0, 2 * g0);
          mma_commit(&bar_s[0][b0]);
          issue_s(1, b0, 2 * g0);
          mma_commit(&bar_s[1][b0]);
          mma_commit(&bar_empty[(2 * g0) % kSlots]);
          if (n > 1) {
            const int b1 = (g0 + 1) & 1;
            wait_load(2 * (g0 + 1));
            issue_s(0, b1, 2 * (g0 + 1));
            mma_commit(&bar_s[0][b1]);
            issue_s(1, b1, 2 * (g0 + 1));
            mma_commit(&bar_s[1][b1]);
            mma_commit(&bar_empty[(2 * (g0 + 1)) % kSlots]);
          }
          if (n <= 2) mma_commit(&bar_qfree);  // every S of this item issued
        }
        for (int it = 0; it < n; ++it) {
          const uint32_t g = g0 + it;
          const int buf = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          const bool last = it + 1 == n, has2 = it + 2 < n;
          const uint32_t ldv = 2 * g + 1, ldk2 = 2 * (g + 2);
          wait_load(ldv);
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&bar_p[t][buf], ph);
            tc_fence_after();
            if (it == 0 && qi > 0) {  // the previous item's epilogue has read O_t
              mbar_wait(&bar_ofree[t], (qi - 1) & 1);
              tc_fence_after();
            }
            issue_pv(t, buf, ldv, it > 0);
            mma_commit(last ? &bar_o[t] : &bar_pv[t]);
            if (t == 1) mma_commit(&bar_empty[ldv % kSlots]);
            if (has2) {
              if (t == 0) wait_load(ldk2);
              issue_s(t, buf, ldk2);
              mma_commit(&bar_s[t][buf]);
              if (t == 1) {
                mma_commit(&bar_empty[ldk2 % kSlots]);
                if (it + 3 == n) mma_commit(&bar_qfree);  // S(g0 + n - 1) was the item's last S
              }
            }
          }
        }
        g0 += n;
        ++qi;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int w = (warp - 4) >> 2;
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * w;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO + w * kD;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    const bool merge = p.mode == RCP_MODE_MERGE;
    uint32_t g0 = 0, qi = 0, pvb = 0;  // global block base, non-empty items, bar_pv commits so far
    for (uint32_t k = 0;; ++k) {
      const int item = next_item(k, true);
      if (item >= n_items) break;
      int qblk, head, kvh;
      item_coords(item, qblk, head, kvh);
      const int row = (2 * qblk + w) * kQRows + t;
      const bool row_ok = row < p.tq;
      const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
      const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
      float m = -INFINITY, l = 0.f;
      const int n = __ldg(p.act_n + qblk);
      const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
      uint32_t e_next = n > 0 ? __ldg(act) : 0u;
      int it = 0;
      for (; it < n; ++it) {
        const uint32_t g = g0 + it;
        const int buf = g & 1;
        const uint32_t s_addr = lane_base + kTmemS + (2 * w + buf) * kKRows;
        const uint32_t e = e_next;
        if (it + 1 < n) e_next = __ldg(act + it + 1);
        const int j = act_j(e);
        const int cls = act_cls(e, w);
        mbar_wait(&bar_s[w][buf], (g >> 1) & 1);
        tc_fence_after();
        if (cls != kTileEmpty) {
          uint32_t sr[64];
          tmem_ld64(s_addr, sr);
          tmem_ld_wait();
          float s[64];
#pragma unroll
          for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
          if (cls == kTilePartial) {
            const int base = j * kKRows;
            if (base + kKRows <= p.tk) {
              const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
              const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll
              for (int c4 = 0; c4 < 16; ++c4) {
                const int4 kp = __ldg(kp4 + c4), kq = __ldg(ks4 + c4);
                if (!(kq.x == my_seq && kp.x <= my_pos)) s[4 * c4 + 0] = -INFINITY;
                if (!(kq.y == my_seq && kp.y <= my_pos)) s[4 * c4 + 1] = -INFINITY;
                if (!(kq.z == my_seq && kp.z <= my_pos)) s[4 * c4 + 2] = -INFINITY;
                if (!(kq.w == my_seq && kp.w <= my_pos)) s[4 * c4 + 3] = -INFINITY;
              }
            } else {
#pragma unroll
              for (int c = 0; c < 64; ++c) {
                const int kidx = base + c;
                const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq &&
                                __ldg(p.k_pos + kidx) <= my_pos;
                if (!ok) s[c] = -INFINITY;
              }
            }
          }
          float m8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
          for (int c = 8; c < 64; c += 8)
#pragma unroll
            for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
          const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                                 fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          const float m_old = m;
          const float m_new = fmaxf(m, mx * sl2);
          const bool need = m_new > m + kRescaleThreshold;
          if (need) m = m_new;
          const float m_use = (m == -INFINITY) ? 0.f : m;
          const uint64_t negm2 = f2(-m_use, -m_use);
          uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
          uint32_t pk[32];
          if (cls == kTileFull) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
              float p0, p1;
              if ((i & 7) < kPolyPairsPer8) {
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
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
              const float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
              acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              pk[i] = pack_bf16x2(p0, p1);
            }
          }
          tmem_st32(s_addr, pk);
          const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
          const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
          const float sum = (a01.x + a01.y) + (a23.x + a23.y);
          const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
          l = (m_old == -INFINITY ? 0.f : l * f) + sum;
          if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
            mbar_wait(&bar_pv[w], (pvb + it - 1) & 1);  // PV_t of the previous block landed
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < kD; c += 32) {
              uint32_t r[32];
              tmem_ld32(o_addr + c, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
              tmem_st32(o_addr + c, r);
            }
          }
        } else {
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = 0u;
          tmem_st32(s_addr, pk);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bar_p[w][buf]);
      }

      // epilogue: O / l, LSE, optional merge into the running (O, LSE)
      if (n > 0) {
        mbar_wait(&bar_o[w], qi & 1);
        tc_fence_after();
      }
      if (!(merge && n == 0)) {
        const bool has = l > 0.f;
        const float inv = has ? 1.0f / l : 0.f;
        const float lse_new = has ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
        float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD;
        float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
        MergeW mw;
        mw.lse = lse_new;
        mw.wa = 0.f;
        mw.wb = 1.f;
        if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
        for (int c = 0; c < kD; c += 32) {
          uint32_t r[32];
          if (n > 0) {
            tmem_ld32(o_addr + c, r);
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
                                     __uint_as_float(r[4 * i + 2]) * inv,
                                     __uint_as_float(r[4 * i + 3]) * inv);
              if (merge) {
                const float4 a = dst[i];
                v = make_float4(merge_val(a.x, v.x, mw), merge_val(a.y, v.y, mw),
                                merge_val(a.z, v.z, mw), merge_val(a.w, v.w, mw));
              }
              dst[i] = v;
            }
          }
        }
        if (row_ok) *lrow = merge ? mw.lse : lse_new;
      }
      if (n > 0) {
        tc_fence_before();
        mbar_arrive(&bar_ofree[w]);  // O_t read out: the next item's first PV may overwrite it
        g0 += n;
        pvb += n - 1;
        ++qi;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}


// ======================================================================
// v10: v4 with S decoupled from P.  In v4, S_t(j+2) shares a TMEM buffer
// with P_t(j), so it can only be issued after PV_t(j) — and the N = 64 S
// MMAs run at ~55 % of the tensor rate — so the softmax waits for its next
// S (20 % of all warp samples in the v4e ncu capture sit on that wait).
// Here each tile has ONE S buffer, released by the softmax as soon as it has
// loaded S(j) into registers (bar_sfree), so the MMA issues S(j+1) at the
// start of softmax block j and it computes under the exps; P goes to its own
// double buffer (2 x 32 columns per tile), reused once the PV that read it
// is done (bar_pvd, also the "PV(j-1) landed" signal of the O rescale).
// TMEM: O0 [0,128) | O1 [128,256) | S0 [256,320) | S1 [320,384) |
//       P0 [384,416) [416,448) | P1 [448,480) [480,512).
// ======================================================================
constexpr uint32_t kTmemS10 = 256, kTmemP10 = 384;

__global__ void __launch_bounds__(kThreads, 1) attn_fwd_v10_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + 2 * kQTileBytes;

  __shared__ uint64_t bar_q, bar_full[kSlots], bar_empty[kSlots];
  __shared__ uint64_t bar_s[2], bar_sfree[2], bar_p[2][2], bar_pvd[2][2], bar_o[2];
  __shared__ uint32_t tmem_slot;

  const int warp = static_cast<int>(warp_id());
  const int per_kv = p.n_qblk * p.group;
  const int kvh = static_cast<int>(blockIdx.x) / per_kv;
  const int rem = static_cast<int>(blockIdx.x) - kvh * per_kv;
  const int qblk = p.n_qblk - 1 - rem / p.group;
  const int head = kvh * p.group + rem % p.group;
  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t], 1);
      mbar_init(&bar_sfree[t], 128);
      mbar_init(&bar_o[t], 1);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&bar_p[t][b], 128);
        mbar_init(&bar_pvd[t][b], 1);
      }
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (as v4)
    if (elect_one()) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      const int n = __ldg(p.act_n + qblk);
      const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
      if (n > 0) {
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes);
        for (int t = 0; t < 2; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sQ + t * kQTileBytes + h * kQBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                        (2 * qblk + t) * kQRows, pol_q);
        uint32_t ld = 0;
        uint32_t e_next = __ldg(act);
        for (int it = 0; it < n; ++it) {
          const int j = act_j(e_next);
          if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++ld) {
            const uint32_t slot = ld % kSlots, ph = (ld / kSlots) & 1;
            mbar_wait(&bar_empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&bar_full[slot], kKVBytes);
            const CUtensorMap* map = kv ? &p.tm_v : &p.tm_k;
            for (int h = 0; h < 2; ++h)
              tma_load_2d(sKV + slot * kKVBytes + h * kKVBoxBytes, map, &bar_full[slot],
                          kvh * kD + h * 64, j * kKRows, pol_kv);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16_f32(kQRows, kKRows, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(kQRows, kD, 0, 1);
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kKVBoxBytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots], (ld / kSlots) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int t, uint32_t ld) {
        const uint32_t qa = q_lo + ((t * kQTileBytes) >> 4);
        const uint32_t ka = k_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t d = tmem + kTmemS10 + t * kKRows;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma_ss_lo(d, qa + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                    ka + (((kk >> 2) * kKVBoxBytes + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int t, int b, uint32_t ld, bool acc) {
        const uint32_t va = v_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t pa = tmem + kTmemP10 + 64 * t + 32 * b;
#pragma unroll
        for (int kk = 0; kk < kKRows / 16; ++kk)
          mma_ts_lo(tmem + kTmemO + t * kD, pa + kk * 8, va + ((kk * 2048) >> 4), idesc_o,
                    (acc || kk > 0) ? 1u : 0u);
      };
      const int n = __ldg(p.act_n + qblk);
      if (n > 0) {
        mbar_wait(&bar_q, 0);
        tc_fence_after();
        wait_load(0);
        issue_s(0, 0);
        mma_commit(&bar_s[0]);
        issue_s(1, 0);
        mma_commit(&bar_s[1]);
        mma_commit(&bar_empty[0]);
        for (int it = 0; it < n; ++it) {
          const int b = it & 1;
          const uint32_t pph = (it >> 1) & 1;
          const bool last = it + 1 == n;
          if (!last) {  // S(it + 1) into the buffer each tile's softmax has just read
            const uint32_t ldk = 2 * (it + 1);
            wait_load(ldk);
            for (int t = 0; t < 2; ++t) {
              mbar_wait(&bar_sfree[t], it & 1);
              tc_fence_after();
              issue_s(t, ldk);
              mma_commit(&bar_s[t]);
            }
            mma_commit(&bar_empty[ldk % kSlots]);
          }
          const uint32_t ldv = 2 * it + 1;
          wait_load(ldv);
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&bar_p[t][b], pph);
            tc_fence_after();
            issue_pv(t, b, ldv, it > 0);
            mma_commit(&bar_pvd[t][b]);
            if (last) mma_commit(&bar_o[t]);
          }
          mma_commit(&bar_empty[ldv % kSlots]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int w = (warp - 4) >> 2;
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * w;
    const int row = (2 * qblk + w) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO + w * kD;
    const uint32_t s_addr = lane_base + kTmemS10 + w * kKRows;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    const int n = __ldg(p.act_n + qblk);
    const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    int it = 0;
    for (; it < n; ++it) {
      const int b = it & 1;
      const uint32_t p_addr = lane_base + kTmemP10 + 64 * w + 32 * b;
      const uint32_t e = e_next;
      if (it + 1 < n) e_next = __ldg(act + it + 1);
      const int j = act_j(e);
      const int cls = act_cls(e, w);
      mbar_wait(&bar_s[w], it & 1);
      tc_fence_after();
      uint32_t pk[32];
      if (cls != kTileEmpty) {  // warp-uniform
        uint32_t sr[64];
        tmem_ld64(s_addr, sr);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bar_sfree[w]);  // S buffer free: the MMA may issue S(it + 1)
        float s[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
        if (cls == kTilePartial) {
          const int base = j * kKRows;
          if (base + kKRows <= p.tk) {
            const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
            const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
              const int4 kp = __ldg(kp4 + c4), kq = __ldg(ks4 + c4);
              if (!(kq.x == my_seq && kp.x <= my_pos)) s[4 * c4 + 0] = -INFINITY;
              if (!(kq.y == my_seq && kp.y <= my_pos)) s[4 * c4 + 1] = -INFINITY;
              if (!(kq.z == my_seq && kp.z <= my_pos)) s[4 * c4 + 2] = -INFINITY;
              if (!(kq.w == my_seq && kp.w <= my_pos)) s[4 * c4 + 3] = -INFINITY;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 64; ++c) {
              const int kidx = base + c;
              const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq &&
                              __ldg(p.k_pos + kidx) <= my_pos;
              if (!ok) s[c] = -INFINITY;
            }
          }
        }
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
        for (int c = 8; c < 64; c += 8)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;
        if (need) m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
        if (cls == kTileFull) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
            float p0, p1;
            if ((i & 7) < kPolyPairsPer8) {
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
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
            const float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
            acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
            pk[i] = pack_bf16x2(p0, p1);
          }
        }
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
          // rescale O_t in place once PV_t(it - 1) has landed
          mbar_wait(&bar_pvd[w][(it - 1) & 1], ((it - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < kD; c += 32) {
            uint32_t r[32];
            tmem_ld32(o_addr + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st32(o_addr + c, r);
          }
        }
      } else {
        tc_fence_before();
        mbar_arrive(&bar_sfree[w]);
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      }
      if (it >= 2) {  // P buffer b was read by PV(it - 2)
        mbar_wait(&bar_pvd[w][b], ((it >> 1) - 1) & 1);
        tc_fence_after();
      }
      tmem_st32(p_addr, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bar_p[w][b]);
    }

    // epilogue (as v4)
    if (it > 0) {
      mbar_wait(&bar_o[w], 0);
      tc_fence_after();
    }
    const bool merge = p.mode == RCP_MODE_MERGE;
    if (!(merge && it == 0)) {
      const bool has = l > 0.f;
      const float inv = has ? 1.0f / l : 0.f;
      const float lse_new = has ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD;
      float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
      MergeW mw;
      mw.lse = lse_new;
      mw.wa = 0.f;
      mw.wb = 1.f;
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
      for (int c = 0; c < kD; c += 32) {
        uint32_t r[32];
        if (it > 0) {
          tmem_ld32(o_addr + c, r);
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
                                   __uint_as_float(r[4 * i + 2]) * inv,
                                   __uint_as_float(r[4 * i + 3]) * inv);
            if (merge) {
              const float4 a = dst[i];
              v = make_float4(merge_val(a.x, v.x, mw), merge_val(a.y, v.y, mw),
                              merge_val(a.z, v.z, mw), merge_val(a.w, v.w, mw));
            }
            dst[i] = v;
          }
        }
      }
      if (row_ok) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ======================================================================
// v11: v10 with one MMA-issuing warp per query tile (warp 1: tile 0, warp 3:
// tile 1).  tcgen05.commit tracks the issuing thread's MMAs, so each tile's
// S / PV stream is ordered only by its own barriers — a tile's next S is no
// longer held behind the other tile's P.  K/V slots are read by both tiles:
// their "empty" barriers take one commit from each issuer.
// (v10 text follows.)
// v10: v4 with S decoupled from P.  In v4, S_t(j+2) shares a TMEM buffer
// with P_t(j), so it can only be issued after PV_t(j) — and the N = 64 S
// MMAs run at ~55 % of the tensor rate — so the softmax waits for its next
// S (20 % of all warp samples in the v4e ncu capture sit on that wait).
// Here each tile has ONE S buffer, released by the softmax as soon as it has
// loaded S(j) into registers (bar_sfree), so the MMA issues S(j+1) at the
// start of softmax block j and it computes under the exps; P goes to its own
// double buffer (2 x 32 columns per tile), reused once the PV that read it
// is done (bar_pvd, also the "PV(j-1) landed" signal of the O rescale).
// TMEM: O0 [0,128) | O1 [128,256) | S0 [256,320) | S1 [320,384) |
//       P0 [384,416) [416,448) | P1 [448,480) [480,512).
// ======================================================================

__global__ void __launch_bounds__(kThreads, 1) attn_fwd_v11_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + 2 * kQTileBytes;

  __shared__ uint64_t bar_q, bar_full[kSlots], bar_empty[kSlots];
  __shared__ uint64_t bar_s[2], bar_sfree[2], bar_p[2][2], bar_pvd[2][2], bar_o[2];
  __shared__ uint32_t tmem_slot;

  const int warp = static_cast<int>(warp_id());
  const int per_kv = p.n_qblk * p.group;
  const int kvh = static_cast<int>(blockIdx.x) / per_kv;
  const int rem = static_cast<int>(blockIdx.x) - kvh * per_kv;
  const int qblk = p.n_qblk - 1 - rem / p.group;
  const int head = kvh * p.group + rem % p.group;
  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 2);  // one commit per tile's MMA issuer
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t], 1);
      mbar_init(&bar_sfree[t], 128);
      mbar_init(&bar_o[t], 1);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&bar_p[t][b], 128);
        mbar_init(&bar_pvd[t][b], 1);
      }
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (as v4)
    if (elect_one()) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      const int n = __ldg(p.act_n + qblk);
      const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
      if (n > 0) {
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes);
        for (int t = 0; t < 2; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sQ + t * kQTileBytes + h * kQBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                        (2 * qblk + t) * kQRows, pol_q);
        uint32_t ld = 0;
        uint32_t e_next = __ldg(act);
        for (int it = 0; it < n; ++it) {
          const int j = act_j(e_next);
          if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++ld) {
            const uint32_t slot = ld % kSlots, ph = (ld / kSlots) & 1;
            mbar_wait(&bar_empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&bar_full[slot], kKVBytes);
            const CUtensorMap* map = kv ? &p.tm_v : &p.tm_k;
            for (int h = 0; h < 2; ++h)
              tma_load_2d(sKV + slot * kKVBytes + h * kKVBoxBytes, map, &bar_full[slot],
                          kvh * kD + h * 64, j * kKRows, pol_kv);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuer of tile tt
    const int tt = warp == 1 ? 0 : 1;
    if (elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16_f32(kQRows, kKRows, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(kQRows, kD, 0, 1);
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kKVBoxBytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots], (ld / kSlots) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](uint32_t ld) {
        const uint32_t qa = q_lo + ((tt * kQTileBytes) >> 4);
        const uint32_t ka = k_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t d = tmem + kTmemS10 + tt * kKRows;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma_ss_lo(d, qa + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                    ka + (((kk >> 2) * kKVBoxBytes + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int b, uint32_t ld, bool acc) {
        const uint32_t va = v_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t pa = tmem + kTmemP10 + 64 * tt + 32 * b;
#pragma unroll
        for (int kk = 0; kk < kKRows / 16; ++kk)
          mma_ts_lo(tmem + kTmemO + tt * kD, pa + kk * 8, va + ((kk * 2048) >> 4), idesc_o,
                    (acc || kk > 0) ? 1u : 0u);
      };
      const int n = __ldg(p.act_n + qblk);
      if (n > 0) {
        mbar_wait(&bar_q, 0);
        tc_fence_after();
        wait_load(0);
        issue_s(0);
        mma_commit(&bar_s[tt]);
        mma_commit(&bar_empty[0]);
        for (int it = 0; it < n; ++it) {
          const int b = it & 1;
          const bool last = it + 1 == n;
          if (!last) {  // S(it + 1) into the buffer this tile's softmax has just read
            const uint32_t ldk = 2 * (it + 1);
            wait_load(ldk);
            mbar_wait(&bar_sfree[tt], it & 1);
            tc_fence_after();
            issue_s(ldk);
            mma_commit(&bar_s[tt]);
            mma_commit(&bar_empty[ldk % kSlots]);
          }
          const uint32_t ldv = 2 * it + 1;
          wait_load(ldv);
          mbar_wait(&bar_p[tt][b], (it >> 1) & 1);
          tc_fence_after();
          issue_pv(b, ldv, it > 0);
          mma_commit(&bar_pvd[tt][b]);
          if (last) mma_commit(&bar_o[tt]);
          mma_commit(&bar_empty[ldv % kSlots]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int w = (warp - 4) >> 2;
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * w;
    const int row = (2 * qblk + w) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO + w * kD;
    const uint32_t s_addr = lane_base + kTmemS10 + w * kKRows;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    const int n = __ldg(p.act_n + qblk);
    const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    int it = 0;
    for (; it < n; ++it) {
      const int b = it & 1;
      const uint32_t p_addr = lane_base + kTmemP10 + 64 * w + 32 * b;
      const uint32_t e = e_next;
      if (it + 1 < n) e_next = __ldg(act + it + 1);
      const int j = act_j(e);
      const int cls = act_cls(e, w);
      mbar_wait(&bar_s[w], it & 1);
      tc_fence_after();
      uint32_t pk[32];
      if (cls != kTileEmpty) {  // warp-uniform
        uint32_t sr[64];
        tmem_ld64(s_addr, sr);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bar_sfree[w]);  // S buffer free: the MMA may issue S(it + 1)
        float s[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
        if (cls == kTilePartial) {
          const int base = j * kKRows;
          if (base + kKRows <= p.tk) {
            const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
            const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
              const int4 kp = __ldg(kp4 + c4), kq = __ldg(ks4 + c4);
              if (!(kq.x == my_seq && kp.x <= my_pos)) s[4 * c4 + 0] = -INFINITY;
              if (!(kq.y == my_seq && kp.y <= my_pos)) s[4 * c4 + 1] = -INFINITY;
              if (!(kq.z == my_seq && kp.z <= my_pos)) s[4 * c4 + 2] = -INFINITY;
              if (!(kq.w == my_seq && kp.w <= my_pos)) s[4 * c4 + 3] = -INFINITY;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 64; ++c) {
              const int kidx = base + c;
              const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq &&
                              __ldg(p.k_pos + kidx) <= my_pos;
              if (!ok) s[c] = -INFINITY;
            }
          }
        }
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
        for (int c = 8; c < 64; c += 8)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;
        if (need) m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
        if (cls == kTileFull) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
            float p0, p1;
            if ((i & 7) < kPolyPairsPer8) {
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
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
            const float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
            acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
            pk[i] = pack_bf16x2(p0, p1);
          }
        }
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
          // rescale O_t in place once PV_t(it - 1) has landed
          mbar_wait(&bar_pvd[w][(it - 1) & 1], ((it - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < kD; c += 32) {
            uint32_t r[32];
            tmem_ld32(o_addr + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st32(o_addr + c, r);
          }
        }
      } else {
        tc_fence_before();
        mbar_arrive(&bar_sfree[w]);
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      }
      if (it >= 2) {  // P buffer b was read by PV(it - 2)
        mbar_wait(&bar_pvd[w][b], ((it >> 1) - 1) & 1);
        tc_fence_after();
      }
      tmem_st32(p_addr, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bar_p[w][b]);
    }

    // epilogue (as v4)
    if (it > 0) {
      mbar_wait(&bar_o[w], 0);
      tc_fence_after();
    }
    const bool merge = p.mode == RCP_MODE_MERGE;
    if (!(merge && it == 0)) {
      const bool has = l > 0.f;
      const float inv = has ? 1.0f / l : 0.f;
      const float lse_new = has ? (m + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      float* orow = p.o + (static_cast<int64_t>(row) * p.hq + head) * kD;
      float* lrow = p.lse + static_cast<int64_t>(row) * p.hq + head;
      MergeW mw;
      mw.lse = lse_new;
      mw.wa = 0.f;
      mw.wb = 1.f;
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
      for (int c = 0; c < kD; c += 32) {
        uint32_t r[32];
        if (it > 0) {
          tmem_ld32(o_addr + c, r);
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
                                   __uint_as_float(r[4 * i + 2]) * inv,
                                   __uint_as_float(r[4 * i + 3]) * inv);
            if (merge) {
              const float4 a = dst[i];
              v = make_float4(merge_val(a.x, v.x, mw), merge_val(a.y, v.y, mw),
                              merge_val(a.z, v.z, mw), merge_val(a.w, v.w, mw));
            }
            dst[i] = v;
          }
        }
      }
      if (row_ok) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}



int attn_variant_launch(int version, const AttnParams& prm, int64_t grid, cudaStream_t st) {
  const unsigned g = static_cast<unsigned>(grid);
  if (version == 5) {
    static bool attr = false;
    if (!attr) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_2cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmem2Bytes));
      attr = true;
    }
    attn_fwd_2cta_kernel<<<2 * g, kThreads2, kSmem2Bytes, st>>>(prm);
  } else if (version == 6) {
    static bool attr = false;
    if (!attr) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_v6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmem6Bytes));
      attr = true;
    }
    attn_fwd_v6_kernel<<<g, kThreads6, kSmem6Bytes, st>>>(prm);
  } else if (version == 7) {
    static bool attr = false;
    if (!attr) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_v7_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmem7Bytes));
      attr = true;
    }
    attn_fwd_v7_kernel<<<g, kThreads, kSmem7Bytes, st>>>(prm);
  } else if (version == 8) {
    static bool attr = false;
    if (!attr) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_v8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmem2Bytes));
      attr = true;
    }
    attn_fwd_v8_kernel<<<2 * g, kThreads, kSmem2Bytes, st>>>(prm);
  } else if (version == 9) {
    static bool attr = false;
    static int n_sm = 0;
    if (!attr) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_v9_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmemBytes));
      int dev = 0;
      RCP_CUDA(cudaGetDevice(&dev));
      RCP_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
      attr = true;
    }
    const unsigned gp = static_cast<unsigned>(grid < n_sm ? grid : n_sm);
    attn_fwd_v9_kernel<<<gp, kThreads, kSmemBytes, st>>>(prm);
  } else if (version == 10) {
    static bool attr = false;
    if (!attr) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_v10_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmemBytes));
      attr = true;
    }
    attn_fwd_v10_kernel<<<g, kThreads, kSmemBytes, st>>>(prm);
  } else if (version == 11) {
    static bool attr = false;
    if (!attr) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_v11_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmemBytes));
      attr = true;
    }
    attn_fwd_v11_kernel<<<g, kThreads, kSmemBytes, st>>>(prm);
  } else {
    set_error("unknown attention kernel version %d", version);
    return RCP_ERR_INVALID;
  }
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

}  // namespace rcp
