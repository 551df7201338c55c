// K1: causal-by-position GQA flash-attention forward for sm_100a with LSE.
//
// Replaces ringcp.attention.gqa_attention (attention.py:230-282) on the ring
// hot path.  One CTA = two 128-row query tiles of one query head; the tiles
// share every 64-key K/V block the TMA producer streams through an 8-slot ring.
//
// Warp roles (384 threads):
//   warp 0      TMA producer (one elected lane): Q once, then K_j / V_j
//   warps 1, 3  MMA issuers of tiles 0 / 1 (one elected lane each):
//                                                S_t(j) = Q_t K_j^T   (SS, K-major)
//                                                O_t   += P_t(j) V_j  (TS, P in TMEM)
//   warp 2      TMEM allocator
//   warps 4-7   softmax for query tile 0 (thread i owns TMEM lane / row i)
//   warps 8-11  softmax for query tile 1
//
// TMEM (512 columns): O0 [0,128) | O1 [128,256) | S0 buffers [256,320) [320,384)
// | S1 buffers [384,448) [448,512).  S is double-buffered per query tile and
// P(j) (packed bf16) is written over the first 32 columns of the buffer S(j)
// came from.  The MMA warp issues S_t(j+2) into a buffer right after PV_t(j)
// (tcgen05 ops complete in issue order), so while the softmax works on block j
// the tensor cores already hold S(j+1): the softmax never waits for a PV->S
// round trip and both pipes stay busy.  The (rare) in-place rescale of O waits
// for a per-tile "PV done" barrier first.
//
// Masking: per-tile summaries (min/max position and sequence over valid rows,
// 128-row query tiles, 64-row key blocks) classify every (query tile, key
// block) pair as EMPTY (skipped: no TMA, no MMA), FULL (no per-element mask) or
// PARTIAL (per-element seq/pos test), which keeps the general position-based
// mask of the reference off the dense path.  Softmax runs in the exp2 domain
// with a lazily raised running max (rescale only when it grows by > 2^8), part
// of the exp2 on the FMA pipe (cubic polynomial) to relieve MUFU; LSE =
// (m + log2 l) * ln 2 (natural log, attention.py:274-277); rows that admit
// nothing give O = 0, LSE = -inf.
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

#include "attn_common.cuh"

// exp2 polynomial of the FULL-block softmax on packed f32x2 ops (bitwise equal
// to the scalar form; fewer issued instructions).
#ifndef RCP_PACKED_POLY
#define RCP_PACKED_POLY 1
#endif

namespace rcp {

// Pre-pass: for every query-tile pair (one CTA of 256 threads each), the
// ascending list of key blocks that are non-empty for either tile, with both
// classes, compacted with a block-wide ballot scan.
__global__ void __launch_bounds__(256) active_list_kernel(const TileSum* __restrict__ q_sum,
                                                          const TileSum* __restrict__ k_sum,
                                                          int n_qtiles, int n_kblocks,
                                                          uint32_t* __restrict__ act,
                                                          int* __restrict__ act_n, int drop_last) {
  __shared__ int warp_cnt[8];
  __shared__ int base;
  const int qb = blockIdx.x;
  const TileSum q0 = load_sum(q_sum, 2 * qb, n_qtiles), q1 = load_sum(q_sum, 2 * qb + 1, n_qtiles);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  uint32_t* out = act + static_cast<int64_t>(qb) * n_kblocks;
  for (int j0 = 0; j0 < n_kblocks; j0 += 256) {
    const int j = j0 + threadIdx.x;
    uint32_t e = 0;
    bool on = false;
    if (j < n_kblocks) {
      const TileSum k = load_sum(k_sum, j, n_kblocks);
      const int c0 = classify_tile(q0, k), c1 = classify_tile(q1, k);
      on = (c0 | c1) != kTileEmpty;
      e = static_cast<uint32_t>(j) | (static_cast<uint32_t>(c0) << 24) | (static_cast<uint32_t>(c1) << 26);
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0) warp_cnt[wid] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int w2 = 0; w2 < wid; ++w2) off += warp_cnt[w2];
    if (on) out[off + __popc(bal & ((1u << lane) - 1u))] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w2 = 0; w2 < 8; ++w2) tot += warp_cnt[w2];
      base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) act_n[qb] = (drop_last && base > 0) ? base - 1 : base;  // drop_last: negative control
  if (qb == 0 && threadIdx.x == 0) act_n[gridDim.x] = 0;  // v9's work-item counter (workspace slack)
}

// Bound-finding knobs (tools/dbg_builds.sh builds them into separate .so
// files; never set in the product build): RCP_DBG_S_STEPS < 8 computes S over
// fewer K-dim steps, RCP_DBG_NO_EXP replaces the exponentials by a copy.
#ifndef RCP_DBG_S_STEPS
#define RCP_DBG_S_STEPS (kD / 16)
#endif
#ifndef RCP_DBG_NO_EXP
#define RCP_DBG_NO_EXP 0
#endif
// exp2 split of a FULL block: score pair i (of 32) takes the FMA-pipe
// polynomial when bit i of RCP_POLY_MASK is set.  Round 2 A/B
// (profiles/r02_k1_ab.txt, same box): pairs {0,1,2,16,17,18} (18.75 %) run
// +1.5 % over round 1's 1 of 8 ({0,8,16,24}, 12.5 %); the same share spread
// differently ({0,5,10,16,21,26}: -5 %; {0..5}: -3 %) or 12.5 / 25 % at the
// half starts ({0,1,16,17}: -2 %; {0..3,16..19}: 0 %) are not — the position
// of the polynomial pairs in the unrolled loop sets how well the FMA work
// interleaves with the MUFU stream.
#ifndef RCP_POLY_MASK
#define RCP_POLY_MASK 0x00070007u
#endif
constexpr uint32_t kPolyMask = RCP_POLY_MASK;

// kPhase (v15, RCP_ATTN_VERSION=15): the two tiles' softmax warps that share
// an SMSP (warps 4+s and 8+s) run half a block apart — tile 1 starts block j
// once tile 0 has its block-j max, tile 0 starts block j+1 once tile 1 has its
// block-j max (two named barriers per SMSP pair) — so one warp's TMEM load,
// row max and P store overlap the other's exps instead of coinciding.
template <int kPhase>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // 2 query tiles
  uint8_t* sKV = smem + 2 * kQTileBytes;      // kSlots K/V blocks

  __shared__ uint64_t bar_q, bar_full[kSlots], bar_empty[kSlots];
  __shared__ uint64_t bar_s[2][2], bar_p[2][2], bar_pv[2], bar_o[2];
  __shared__ uint32_t tmem_slot;

  const int warp = static_cast<int>(warp_id());
  // CTA order: KV-head major (consecutive CTAs share one KV head, so a wave of
  // ~148 CTAs streams that head's K/V once from DRAM and later waves find it in
  // the 126 MB L2), heavy (late) query blocks first inside a head, then the
  // query heads of the GQA group.
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
      mbar_init(&bar_s[t][0], 1);
      mbar_init(&bar_s[t][1], 1);
      mbar_init(&bar_p[t][0], 128);
      mbar_init(&bar_p[t][1], 128);
      mbar_init(&bar_pv[t], 1);
      mbar_init(&bar_o[t], 1);
    }
#ifdef RCP_TRACE_BUILD
    if (blockIdx.x == 0 && p.trace) {
      p.trace[kTraceCtas * kTraceIters * kTraceEv + 0] = smem_u32(&bar_q);
      p.trace[kTraceCtas * kTraceIters * kTraceEv + 1] = smem_u32(&bar_full[0]);
      p.trace[kTraceCtas * kTraceIters * kTraceEv + 2] = smem_u32(&bar_empty[0]);
      p.trace[kTraceCtas * kTraceIters * kTraceEv + 3] = smem_u32(&bar_s[0][0]);
      p.trace[kTraceCtas * kTraceIters * kTraceEv + 4] = smem_u32(&bar_p[0][0]);
      p.trace[kTraceCtas * kTraceIters * kTraceEv + 5] = smem_u32(&bar_pv[0]);
      p.trace[kTraceCtas * kTraceIters * kTraceEv + 6] = smem_u32(&bar_o[0]);
    }
#endif
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
        uint32_t ld = 0;  // load counter: K_j is load 2*it, V_j load 2*it + 1
        uint32_t e_next = __ldg(act);
        for (int it = 0; it < n; ++it) {
          const int j = act_j(e_next);
          if (it + 1 < n) e_next = __ldg(act + it + 1);
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++ld) {
            const uint32_t slot = ld % kSlots, ph = (ld / kSlots) & 1;
            mbar_wait(&bar_empty[slot], ph ^ 1);
            TRACE(6 + kv, ld / 2);
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
    // ------------------------------------------------------------ MMA issuers: warp 1 tile 0, warp 3 tile 1
    // Each tile's PV(j), S(j+2) stream is ordered only by its own P barriers,
    // so one tile's next S is never held behind the other tile's P (a single
    // issuer measured 2-3.5 % slower).  tcgen05.commit tracks the issuing
    // thread's MMAs; K/V slots, read by both tiles, take one commit from each.
    const int tt = warp == 1 ? 0 : 1;
    if (elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16_f32(kQRows, kKRows, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(kQRows, kD, 0, 1);
      // Descriptor low words (see sm100.cuh): Q / K K-major (LBO field 1), V MN-major (LBO = box).
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ), 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kKVBoxBytes);
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlots], (ld / kSlots) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int buf, uint32_t ld) {
        const uint32_t qa = q_lo + ((tt * kQTileBytes) >> 4);
        const uint32_t ka = k_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t d = tmem + kTmemS + (2 * tt + buf) * kKRows;
#pragma unroll
        for (int kk = 0; kk < RCP_DBG_S_STEPS; ++kk)
          mma_ss_lo(d, qa + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                    ka + (((kk >> 2) * kKVBoxBytes + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int buf, uint32_t ld, bool acc) {
        const uint32_t va = v_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t pa = tmem + kTmemS + (2 * tt + buf) * kKRows;
#pragma unroll
        for (int kk = 0; kk < kKRows / 16; ++kk)
          mma_ts_lo(tmem + kTmemO + tt * kD, pa + kk * 8, va + ((kk * 2048) >> 4), idesc_o,
                    (acc || kk > 0) ? 1u : 0u);
      };
      const int n = __ldg(p.act_n + qblk);
      if (n > 0) {
        mbar_wait(&bar_q, 0);
        // prologue: S(0) and S(1) of this tile
        wait_load(0);
        issue_s(0, 0);
        mma_commit(&bar_s[tt][0]);
        mma_commit(&bar_empty[0]);
        if (n > 1) {
          wait_load(2);
          issue_s(1, 2);
          mma_commit(&bar_s[tt][1]);
          mma_commit(&bar_empty[2 % kSlots]);
        }
        for (int it = 0; it < n; ++it) {
          const int buf = it & 1;
          const bool last = it + 1 == n, has2 = it + 2 < n;
          const uint32_t ldv = 2 * it + 1, ldk2 = 2 * it + 4;
          wait_load(ldv);
          if (tt == 0) TRACE(12, it);
          // PV(it), then into the same buffer S(it+2) (tcgen05 ops complete in issue order)
          mbar_wait(&bar_p[tt][buf], (it >> 1) & 1);
          tc_fence_after();
          TRACE(tt, it);
          issue_pv(buf, ldv, it > 0);
          mma_commit(last ? &bar_o[tt] : &bar_pv[tt]);
          mma_commit(&bar_empty[ldv % kSlots]);
          if (tt == 1) TRACE(13, it);
          if (has2) {
            wait_load(ldk2);
            issue_s(buf, ldk2);
            mma_commit(&bar_s[tt][buf]);
            mma_commit(&bar_empty[ldk2 % kSlots]);
          }
          if (tt == 1) TRACE(14, it);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int w = (warp - 4) >> 2;                                 // query tile 0 / 1
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * w;  // row inside the tile
    const int row = (2 * qblk + w) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) - p.mask_shift : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO + w * kD;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    const int n = __ldg(p.act_n + qblk);
    const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    const uint32_t id_ab = 1 + (warp & 3), id_ba = 5 + (warp & 3);  // kPhase: tile 0 -> 1, 1 -> 0
    int it = 0;
    for (; it < n; ++it) {
      const int buf = it & 1;
      const uint32_t s_addr = lane_base + kTmemS + (2 * w + buf) * kKRows;
      if constexpr (kPhase != 0) {
        if (w == 1)
          named_bar_sync(id_ab, 64);  // tile 0 has the max of block it
        else if (it > 0)
          named_bar_sync(id_ba, 64);  // tile 1 has the max of block it - 1
      }
      const uint32_t e = e_next;
      if (it + 1 < n) e_next = __ldg(act + it + 1);
      const int j = act_j(e);
      const int cls = act_cls(e, w);
      mbar_wait(&bar_s[w][buf], (it >> 1) & 1);
      tc_fence_after();
      if (t == 0) TRACE(2 + 2 * w, it);
      if (cls != kTileEmpty) {  // warp-uniform
        uint32_t sr[64];
        tmem_ld64(s_addr, sr);  // one 64-column load + one wait (vs 2 x 32: +0.8 % CP1, +2 % CP8 shapes)
        tmem_ld_wait();
        float s[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
        if (t == 0 && w == 0) TRACE(8, it);
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
        const bool need = m_new > m + kRescaleThreshold;  // also true for -inf -> finite
        if (need) m = m_new;
        // Rows that have admitted nothing yet keep m = -inf: their scores are all
        // -inf, so exp2(s - 0) = 0.  Everything below is warp-uniform (the
        // tcgen05.ld/st are .sync.aligned).
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        if constexpr (kPhase != 0) named_bar_arrive(w == 0 ? id_ab : id_ba, 64);
        if (t == 0 && w == 0) TRACE(9, it);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
        uint32_t pk[32];
        if (cls == kTileFull) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = unf2(ffma2(f2(s[2 * i], s[2 * i + 1]), sl2x2, negm2));
            float p0, p1;
            if (RCP_DBG_NO_EXP) {  // bound-finding builds only (tools/dbg_builds.sh)
              p0 = x.x;
              p1 = x.y;
            } else if (kPolyMask & (1u << i)) {
#if RCP_PACKED_POLY
              const float2 pp = ex2_poly_x2(x.x, x.y);
              p0 = pp.x;
              p1 = pp.y;
#else
              p0 = ex2_poly(x.x);
              p1 = ex2_poly(x.y);
#endif
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
        if (t == 0 && w == 0) TRACE(10, it);
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
          // Rescale O_t rows in place once PV_t(it-1) has landed in TMEM.
          mbar_wait(&bar_pv[w], (it - 1) & 1);
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
        if constexpr (kPhase != 0) named_bar_arrive(w == 0 ? id_ab : id_ba, 64);
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
        tmem_st32(s_addr, pk);
      }
      if (t == 0 && w == 0) TRACE(11, it);
      tmem_st_wait();
      tc_fence_before();
      if (t == 0) TRACE(3 + 2 * w, it);
      // One P barrier per S buffer: a warp may run one block ahead of the rest
      // of its warpgroup (S(it+1) is already computed), so arrivals of
      // consecutive blocks must not share a barrier phase.
      mbar_arrive(&bar_p[w][buf]);
    }

    if constexpr (kPhase != 0) {
      if (w == 0 && n > 0) named_bar_sync(id_ba, 64);  // consume tile 1's last arrival
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

// ------------------------------------------------------------------ host side
// Kernel form.  The product library has one: v4 (64-key blocks, this file).
// The A/B build (-DRCP_AB_FORMS=1, _ringcp_b200_ab.so, with attn_fwd_n128.cu
// and attn_fwd_pair.cu) also carries the measured alternatives v12-v17,
// selected by RCP_ATTN_VERSION (read once); DESIGN.md §3 has their A/B.
static int attn_version() {
#if RCP_AB_FORMS
  static int version = -1;
  if (version < 0) {
    const char* e = getenv("RCP_ATTN_VERSION");
    const int v = e ? atoi(e) : kDefaultAttnVersion;
    version = (v == 4 || (v >= 12 && v <= 17)) ? v : kDefaultAttnVersion;
  }
  return version;
#else
  return kDefaultAttnVersion;
#endif
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 2-D map over a token-major [rows, heads*128] bf16 array; box = box_rows x 64 cols, SW128.
// (e4m3 = true: a [rows, heads*128] e4m3 array, box = box_rows x 128 cols.)
static int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols,
                    int64_t row_stride_elems, uint32_t box_rows, bool e4m3 = false) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return RCP_ERR_CUDA;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_elems) * (e4m3 ? 1 : 2)};
  cuuint32_t box[2] = {e4m3 ? 128u : 64u, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, e4m3 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld stride=%lld", (int)r,
              (long long)rows, (long long)cols, (long long)row_stride_elems);
    return RCP_ERR_CUDA;
  }
  return RCP_OK;
}

}  // namespace rcp

using namespace rcp;

static long long* g_trace = nullptr;
// Debug hook (RCP_TRACE builds): device buffer of kTraceCtas*kTraceIters*kTraceEv int64.
extern "C" void rcp_debug_set_trace(long long* buf) { g_trace = buf; }
#ifdef RCP_TRACE_BUILD
// Debug hook: {1 + block, thread, barrier smem address, parity} of the first hung wait.
extern "C" void rcp_debug_hang_info(int* out) {
  cudaMemcpyFromSymbol(out, g_hang_info, sizeof(int) * 4);
}
#endif

int rcp::rcp_fault_flags() {
  static int flags = -1;
  if (flags < 0) {
    const char* e = getenv("RCP_FAULT");
    flags = 0;
    if (e) {
      if (strstr(e, "drop_block")) flags |= kFaultDropBlock;
      if (strstr(e, "mask_diag")) flags |= kFaultMaskDiag;
      if (strstr(e, "reverse_merge")) flags |= kFaultReverseMerge;
    }
  }
  return flags;
}

// Workspace: tile summaries | active lists (n_qblk x n_kblocks) | list lengths.
extern "C" size_t rcp_attn_workspace_bytes(int64_t tq, int64_t tk) {
  const int64_t nq = (tq + kQRows - 1) / kQRows, nk = (tk + kKRows - 1) / kKRows;
  const int64_t nqb = (nq + 1) / 2;
  return static_cast<size_t>((nq + nk) * sizeof(TileSum) + nqb * nk * 4 + nqb * 4 + 256);
}

// Shared host side of rcp_attn_fwd and rcp_attn_fwd_qk8 (q_scale non-null:
// q / k are e4m3 with per-head scales, the attn_fwd_qk8.cu kernel runs).
static int attn_fwd_host(const void* q, int64_t q_row_stride, const void* k, int64_t k_row_stride, const void* v,
                         int64_t v_row_stride, const int32_t* q_pos, const int32_t* q_seq, const int32_t* k_pos,
                         const int32_t* k_seq, int64_t tq, int64_t tk, int32_t hq, int32_t hkv, int32_t head_dim,
                         float scale, const float* q_scale, const float* k_scale, float* o, float* lse,
                         int32_t mode, void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool qk8 = q_scale != nullptr;
  RCP_CHECK_ARG(head_dim == kD, "head_dim must be 128, got %d", head_dim);
  RCP_CHECK_ARG(hq >= 1 && hkv >= 1, "head counts must be positive");
  RCP_CHECK_ARG(hq % hkv == 0, "n_query_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  RCP_CHECK_ARG(tq >= 0 && tk >= 0, "token counts must be >= 0");
  RCP_CHECK_ARG(tq < INT32_MAX && tk < INT32_MAX, "token counts must fit int32");
  RCP_CHECK_ARG(mode == RCP_MODE_OVERWRITE || mode == RCP_MODE_MERGE, "bad mode %d", mode);
  if (tq == 0) return RCP_OK;
  RCP_CHECK_ARG(o && lse && q_pos && q_seq, "null query-side pointer");
  if (tk == 0) {
    if (mode == RCP_MODE_MERGE) return RCP_OK;  // merging an empty partial is the identity
    return rcp_fill_empty(o, lse, tq * hq, head_dim, stream);
  }
  RCP_CHECK_ARG(q && k && v && k_pos && k_seq, "null pointer");
  RCP_CHECK_ARG(q_row_stride % (qk8 ? 16 : 8) == 0 && k_row_stride % (qk8 ? 16 : 8) == 0 && v_row_stride % 8 == 0,
                "row strides must be multiples of 8 elements (16 for e4m3 q / k)");
  RCP_CHECK_ARG(!qk8 || k_scale, "e4m3 q / k need both scale arrays");
  RCP_CHECK_ARG(q_row_stride >= hq * kD && k_row_stride >= hkv * kD && v_row_stride >= hkv * kD,
                "row stride smaller than heads*head_dim");
  RCP_CHECK_ARG(((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
                  reinterpret_cast<uintptr_t>(v)) & 15) == 0,
                "q/k/v must be 16-byte aligned");
  RCP_CHECK_ARG(((reinterpret_cast<uintptr_t>(k_pos) | reinterpret_cast<uintptr_t>(k_seq)) & 15) == 0,
                "key metadata must be 16-byte aligned");
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(o) & 15) == 0, "o must be 16-byte aligned");
  const size_t need = rcp_attn_workspace_bytes(tq, tk);
  RCP_CHECK_ARG(workspace != nullptr && workspace_bytes >= need,
                "workspace too small: need %zu bytes", need);
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(workspace) & 31) == 0, "workspace must be 32-byte aligned");

  const int version = qk8 ? kDefaultAttnVersion : attn_version();
  const int krows = attn_key_rows(version);
  AttnParams prm;
  memset(&prm, 0, sizeof(prm));
  int rc;
  if ((rc = make_map(&prm.tm_q, q, tq, static_cast<int64_t>(hq) * kD, q_row_stride, kQRows, qk8)) != RCP_OK)
    return rc;
  if ((rc = make_map(&prm.tm_k, k, tk, static_cast<int64_t>(hkv) * kD, k_row_stride,
                     attn_k_box_rows(version), qk8)) != RCP_OK)
    return rc;
  prm.q_scale = q_scale;
  prm.k_scale = k_scale;
  if ((rc = make_map(&prm.tm_v, v, tk, static_cast<int64_t>(hkv) * kD, v_row_stride,
                     attn_v_box_rows(version))) != RCP_OK)
    return rc;
  prm.q = static_cast<const __nv_bfloat16*>(q);
  prm.q_stride = q_row_stride;
  TileSum* qsum = static_cast<TileSum*>(workspace);
  const int n_qtiles = static_cast<int>((tq + kQRows - 1) / kQRows);
  const int n_kblocks = static_cast<int>((tk + krows - 1) / krows);
  TileSum* ksum = qsum + n_qtiles;
  if ((rc = launch_tile_summary(q_pos, q_seq, tq, RCP_SEQ_PAD_Q, kQRows, qsum, st)) != RCP_OK)
    return rc;
  if ((rc = launch_tile_summary(k_pos, k_seq, tk, RCP_SEQ_PAD_K, krows, ksum, st)) != RCP_OK)
    return rc;
  uint32_t* act = reinterpret_cast<uint32_t*>(ksum + n_kblocks);
  const int n_qblk = (n_qtiles + 1) / 2;
  int* act_n = reinterpret_cast<int*>(act + static_cast<int64_t>(n_qblk) * n_kblocks);
  const int fault = rcp_fault_flags();
  active_list_kernel<<<n_qblk, 256, 0, st>>>(qsum, ksum, n_qtiles, n_kblocks, act, act_n,
                                             (fault & kFaultDropBlock) ? 1 : 0);
  RCP_CUDA(cudaGetLastError());
  prm.act = act;
  prm.act_n = act_n;
  prm.item_ctr = act_n + n_qblk;
  prm.q_pos = q_pos;
  prm.q_seq = q_seq;
  prm.k_pos = k_pos;
  prm.k_seq = k_seq;
  prm.q_sum = qsum;
  prm.k_sum = ksum;
  prm.o = o;
  prm.lse = lse;
  prm.tq = static_cast<int>(tq);
  prm.tk = static_cast<int>(tk);
  prm.hq = hq;
  prm.hkv = hkv;
  prm.group = hq / hkv;
  prm.n_qtiles = n_qtiles;
  prm.n_qblk = (n_qtiles + 1) / 2;
  prm.n_kblocks = n_kblocks;
  prm.mode = mode;
  prm.scale_log2 = static_cast<float>(static_cast<double>(scale) * 1.4426950408889634);
  prm.mask_shift = (fault & kFaultMaskDiag) ? 1 : 0;
  prm.trace = g_trace;

  const int64_t grid = static_cast<int64_t>(prm.n_qblk) * hq;
  RCP_CHECK_ARG(grid < (1ll << 30), "grid too large");
  if (qk8) return attn_qk8_launch(prm, grid, st);
#if RCP_AB_FORMS
  if (version == 13 || version == 14) {
    if ((rc = attn_pair_launch(prm, grid, st, version == 14)) != RCP_OK) return rc;
    return RCP_OK;
  }
  if (version == 12 || version == 16 || version == 17) {
    if ((rc = attn_n128_launch(prm, grid, st, version == 16 ? 1 : version == 17 ? 2 : 0)) != RCP_OK) return rc;
    return RCP_OK;
  }
  if (version == 15) {
    static bool attr15 = false;
    if (!attr15) {
      RCP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmemBytes));
      attr15 = true;
    }
    attn_fwd_kernel<1><<<static_cast<unsigned>(grid), kThreads, kSmemBytes, st>>>(prm);
    RCP_CUDA(cudaGetLastError());
    return RCP_OK;
  }
#endif
  static bool attr_set = false;
  if (!attr_set) {
    RCP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBytes));
    attr_set = true;
  }
  attn_fwd_kernel<0><<<static_cast<unsigned>(grid), kThreads, kSmemBytes, st>>>(prm);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

extern "C" int rcp_attn_fwd(const void* q, int64_t q_row_stride, const void* k,
                            int64_t k_row_stride, const void* v, int64_t v_row_stride,
                            const int32_t* q_pos, const int32_t* q_seq, const int32_t* k_pos,
                            const int32_t* k_seq, int64_t tq, int64_t tk, int32_t hq,
                            int32_t hkv, int32_t head_dim, float scale, float* o, float* lse,
                            int32_t mode, void* workspace, size_t workspace_bytes, void* stream) {
  return attn_fwd_host(q, q_row_stride, k, k_row_stride, v, v_row_stride, q_pos, q_seq, k_pos, k_seq, tq, tk, hq,
                       hkv, head_dim, scale, nullptr, nullptr, o, lse, mode, workspace, workspace_bytes, stream);
}

extern "C" int rcp_attn_fwd_qk8(const void* q8, int64_t q_row_stride, const void* k8, int64_t k_row_stride,
                                const void* v, int64_t v_row_stride, const int32_t* q_pos, const int32_t* q_seq,
                                const int32_t* k_pos, const int32_t* k_seq, int64_t tq, int64_t tk, int32_t hq,
                                int32_t hkv, int32_t head_dim, float scale, const float* q_scale,
                                const float* k_scale, float* o, float* lse, int32_t mode, void* workspace,
                                size_t workspace_bytes, void* stream) {
  RCP_CHECK_ARG(q_scale && k_scale, "null q / k scale arrays");
  return attn_fwd_host(q8, q_row_stride, k8, k_row_stride, v, v_row_stride, q_pos, q_seq, k_pos, k_seq, tq, tk, hq,
                       hkv, head_dim, scale, q_scale, k_scale, o, lse, mode, workspace, workspace_bytes, stream);
}

extern "C" int rcp_attn_version(void) { return rcp::attn_version(); }
