// K1, 128-key-block form (v12): causal-by-position GQA flash-attention
// forward for sm_100a with LSE.  Replaces ringcp.attention.gqa_attention
// (attention.py:230-282) on the ring hot path, like the 64-key v4 kernel in
// attn_fwd.cu, whose masking / active-list / epilogue contract it keeps.
//
// Why 128-key blocks: S = Q K^T issued as a 128 x 64 SS MMA needs 6 KB of
// shared-memory operands per 32 tensor cycles (192 B/clk against the 128 B/clk
// port) and runs at 55 % of the tensor rate; as 128 x 128 it needs 8 KB per 64
// cycles and runs at the full rate (profiles/r01_probe_mma_rate.txt).  That
// N = 64 ceiling (~1447 of 1024 ideal cycles per 16384 scores) is what bounds v4.
//
// One CTA = two 128-row query tiles of one query head sharing each 128-key
// K / V block, streamed by TMA through a 5-slot ring (Q 64 KB + 5 x 32 KB).
//
// Warp roles (384 threads):
//   warp 0      TMA producer (one elected lane): Q once, then K_j / V_j
//   warps 1, 3  MMA issuers of tiles 0 / 1 (one elected lane each):
//                 O_t += P_t(j) V_j        (TS, P in TMEM, V MN-major)
//                 S_t(j+1) = Q_t K_{j+1}^T (SS, K-major, N = 128)
//   warp 2      TMEM allocator
//   warps 4-7   softmax of query tile 0 (thread i owns TMEM lane / row i)
//   warps 8-11  softmax of query tile 1
//
// TMEM (512 columns): O0 [0,128) | O1 [128,256) | S0 [256,384) | S1 [384,512).
// One S buffer per tile; P_t(j) (packed bf16, 64 columns) is written over the
// first half of S_t once the softmax holds S_t(j) in registers.  The issuer of
// tile t issues S_t(j+1) right after PV_t(j) (tcgen05 MMAs of one thread
// execute in order, so S_t(j+1) overwrites P_t(j) only after PV_t(j) read it).
// A tile's chain is softmax -> PV -> S; the two tiles alternate on the tensor
// cores, so while one tile's softmax runs the other tile's PV and S execute.
// Because S_t(j) is issued after PV_t(j-1), a completed S_t(j) also means O_t
// is final up to block j-1: the (rare) lazy O rescale needs no extra wait.
//
// Masking, the exp2-domain softmax with a lazily raised running max, the FMA-
// pipe polynomial share of exp2, LSE = (m + log2 l) ln 2 and the overwrite /
// merge epilogue are those of v4 (attn_fwd.cu).
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

#include "attn_common.cuh"

namespace rcp {

constexpr int kKRowsN = 128;                               // key block rows (N of S, K of PV)
constexpr int kSlotsN = 5;                                 // K/V ring slots (K_j, V_j, K_j+1, ...)
constexpr uint32_t kKVBytesN = kKRowsN * kD * 2;           // 32 KB: two 16 KB SW128 boxes
constexpr uint32_t kKVBoxBytesN = kKVBytesN / 2;
constexpr uint32_t kSmemBytesN = 2 * kQTileBytes + kSlotsN * kKVBytesN + 1024;
static_assert(kSmemBytesN <= 232448, "v12 shared memory exceeds 227 KB");
// Of every 8 score pairs of a FULL block, this many take exp2 on the FMA pipe.
#ifndef RCP_POLY_PAIRS_N
#define RCP_POLY_PAIRS_N 2
#endif
constexpr int kPolyPairsN = RCP_POLY_PAIRS_N;

// kTurn (v16, RCP_ATTN_VERSION=16): the two tiles' softmax warps that share an
// SMSP take turns on the exponentials (tile 0 block j, tile 1 block j, tile 0
// block j+1, ...; two named barriers per SMSP pair), so the MUFU / FMA pipes
// serve one warp at a time and the tiles settle half a period apart — one
// tile's exps run while the other tile's PV and next S occupy the tensor cores.
// kSplit (v17, RCP_ATTN_VERSION=17; FA4's split P arrive): the softmax
// signals P in two parts — keys 0-95 once they are stored, keys 96-127 at the
// end — and the issuer starts PV on the first part, so the tensor cores run
// under the tail of the exps; the row sum moves after the final arrive.
template <bool kTurn, bool kSplit>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_n128_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                     // 2 query tiles
  uint8_t* sKV = smem + 2 * kQTileBytes;  // kSlotsN K/V blocks

  __shared__ uint64_t bar_q, bar_full[kSlotsN], bar_empty[kSlotsN];
  __shared__ uint64_t bar_s[2], bar_p[2], bar_o[2], bar_p2[2];
  __shared__ uint32_t tmem_slot;

  const int warp = static_cast<int>(warp_id());
  // CTA order as v4: KV-head major (a wave's K/V stays L2-resident), heavy
  // (late) query blocks first inside a head, then the GQA group's query heads.
  const int per_kv = p.n_qblk * p.group;
  const int kvh = static_cast<int>(blockIdx.x) / per_kv;
  const int rem = static_cast<int>(blockIdx.x) - kvh * per_kv;
  const int qblk = p.n_qblk - 1 - rem / p.group;
  const int head = kvh * p.group + rem % p.group;
  const int n = __ldg(p.act_n + qblk);
  const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kSlotsN; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 2);  // one commit per tile's MMA issuer
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t], 1);
      mbar_init(&bar_p[t], 128);
      mbar_init(&bar_p2[t], 128);
      mbar_init(&bar_o[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  // Registers: the softmax rows hold 128 scores; the TMA / MMA / TMEM warpgroup
  // needs few.  128 x 56 + 256 x 224 = 64512 = the launch allocation 384 x 168
  // (.inc can only take what .dec released; setmaxnreg at the head of each
  // warpgroup's branch, so every role's code sits under one register limit).
  if (warp < 4) {
   setmaxnreg_dec<56>();
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
          const uint32_t slot = ld % kSlotsN, ph = (ld / kSlotsN) & 1;
          mbar_wait(&bar_empty[slot], ph ^ 1);
          TRACE(6 + kv, it);
          mbar_arrive_expect_tx(&bar_full[slot], kKVBytesN);
          const CUtensorMap* map = kv ? &p.tm_v : &p.tm_k;
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sKV + slot * kKVBytesN + h * kKVBoxBytesN, map, &bar_full[slot], kvh * kD + h * 64,
                        j * kKRowsN, pol_kv);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuers: warp 1 tile 0, warp 3 tile 1
    const int tt = warp == 1 ? 0 : 1;
    if (elect_one() && n > 0) {
      const uint32_t idesc_s = make_idesc_bf16_f32(kQRows, kKRowsN, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(kQRows, kD, 0, 1);
      const uint32_t q_lo = sw128_desc_lo(smem_u32(sQ) + tt * kQTileBytes, 16);
      const uint32_t k_lo = sw128_desc_lo(smem_u32(sKV), 16);
      const uint32_t v_lo = sw128_desc_lo(smem_u32(sKV), kKVBoxBytesN);
      const uint32_t s_t = tmem + kTmemS + tt * kKRowsN;  // S_t / P_t columns
      const uint32_t o_t = tmem + kTmemO + tt * kD;
      auto wait_load = [&](uint32_t ld) {
        mbar_wait(&bar_full[ld % kSlotsN], (ld / kSlotsN) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](uint32_t ld) {
        const uint32_t ka = k_lo + (((ld % kSlotsN) * kKVBytesN) >> 4);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma_ss_lo(s_t, q_lo + (((kk >> 2) * kQBoxBytes + (kk & 3) * 32) >> 4),
                    ka + (((kk >> 2) * kKVBoxBytesN + (kk & 3) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv = [&](uint32_t ld, bool acc, int kk0, int kk1) {
        const uint32_t va = v_lo + (((ld % kSlotsN) * kKVBytesN) >> 4);
#pragma unroll
        for (int kk = kk0; kk < kk1; ++kk)
          mma_ts_lo(o_t, s_t + kk * 8, va + ((kk * 2048) >> 4), idesc_o, (acc || kk > 0) ? 1u : 0u);
      };
      mbar_wait(&bar_q, 0);
      wait_load(0);
      issue_s(0);
      mma_commit(&bar_s[tt]);
      mma_commit(&bar_empty[0]);
      for (int it = 0; it < n; ++it) {
        const bool last = it + 1 == n;
        const uint32_t ldv = 2 * it + 1, ldk = 2 * it + 2;
        wait_load(ldv);
        mbar_wait(&bar_p[tt], it & 1);
        tc_fence_after();
        if constexpr (kSplit) {
          issue_pv(ldv, it > 0, 0, 6);  // keys 0-95 of P are stored
          mbar_wait(&bar_p2[tt], it & 1);
          tc_fence_after();
          issue_pv(ldv, it > 0, 6, 8);
        } else {
          issue_pv(ldv, it > 0, 0, 8);
        }
        TRACE(tt, it);
        if (last) mma_commit(&bar_o[tt]);
        mma_commit(&bar_empty[ldv % kSlotsN]);
        if (!last) {
          wait_load(ldk);
          issue_s(ldk);
          TRACE(12 + tt, it);
          mma_commit(&bar_s[tt]);
          mma_commit(&bar_empty[ldk % kSlotsN]);
        }
      }
    }
    __syncwarp();
   }
  } else {
    setmaxnreg_inc<224>();
    // ------------------------------------------------------------ softmax + epilogue
    const int w = (warp - 4) >> 2;                                 // query tile 0 / 1
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * w;  // row inside the tile
    const int row = (2 * qblk + w) * kQRows + t;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) - p.mask_shift : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_base + kTmemO + w * kD;
    const uint32_t s_addr = lane_base + kTmemS + w * kKRowsN;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    const uint32_t id_ab = 1 + (warp & 3), id_ba = 5 + (warp & 3);  // kTurn: tile 0 -> 1, 1 -> 0
    auto turn_begin = [&](int i) {
      if constexpr (kTurn) {
        if (w == 1)
          named_bar_sync(id_ab, 64);  // tile 0 finished its exps of block i
        else if (i > 0)
          named_bar_sync(id_ba, 64);  // tile 1 finished its exps of block i - 1
      }
    };
    auto turn_end = [&]() {
      if constexpr (kTurn) named_bar_arrive(w == 0 ? id_ab : id_ba, 64);
    };
    int it = 0;
    for (; it < n; ++it) {
      const uint32_t e = e_next;
      if (it + 1 < n) e_next = __ldg(act + it + 1);
      const int j = act_j(e);
      const int cls = act_cls(e, w);
      // Mask bits of a PARTIAL block (bit c: key c admitted for this row),
      // computed before S is live in registers.
      uint32_t mbits[4] = {~0u, ~0u, ~0u, ~0u};
      if (cls == kTilePartial) {
        const int base = j * kKRowsN;
        if (base + kKRowsN <= p.tk) {
          const int4* kp4 = reinterpret_cast<const int4*>(p.k_pos + base);
          const int4* ks4 = reinterpret_cast<const int4*>(p.k_seq + base);
#pragma unroll 1
          for (int g = 0; g < 4; ++g) {  // (not unrolled: 8 int4 pairs in flight, not 64)
            uint32_t bits = 0;
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const int4 kp = __ldg(kp4 + 8 * g + c4), kq = __ldg(ks4 + 8 * g + c4);
              bits |= static_cast<uint32_t>(kq.x == my_seq && kp.x <= my_pos) << (4 * c4 + 0);
              bits |= static_cast<uint32_t>(kq.y == my_seq && kp.y <= my_pos) << (4 * c4 + 1);
              bits |= static_cast<uint32_t>(kq.z == my_seq && kp.z <= my_pos) << (4 * c4 + 2);
              bits |= static_cast<uint32_t>(kq.w == my_seq && kp.w <= my_pos) << (4 * c4 + 3);
            }
#pragma unroll
            for (int x = 0; x < 4; ++x) mbits[x] = g == x ? bits : mbits[x];
          }
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) {  // (unrolled: mbits stays in registers)
            uint32_t bits = 0;
#pragma unroll 1
            for (int c = 0; c < 32; ++c) {
              const int kidx = base + 32 * g + c;
              const bool ok = kidx < p.tk && __ldg(p.k_seq + kidx) == my_seq && __ldg(p.k_pos + kidx) <= my_pos;
              bits |= static_cast<uint32_t>(ok) << c;
            }
            mbits[g] = bits;
          }
        }
      }
      mbar_wait(&bar_s[w], it & 1);
      tc_fence_after();
      if (t == 0) TRACE(2 + 2 * w, it);
      if (cls != kTileEmpty) {  // warp-uniform
        float s[128];
        {
          uint32_t sr[64];
          tmem_ld64(s_addr, sr);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 64; ++c) s[c] = __uint_as_float(sr[c]);
          tmem_ld64(s_addr + 64, sr);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 64; ++c) s[64 + c] = __uint_as_float(sr[c]);
        }
        if (t == 0 && w == 0) TRACE(8, it);
        if (cls == kTilePartial) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (!((mbits[c >> 5] >> (c & 31)) & 1u)) s[c] = -INFINITY;
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
        if (t == 0 && w == 0) TRACE(9, it);
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;  // also true for -inf -> finite
        if (need) m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const uint64_t negm2 = f2(-m_use, -m_use);
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
          // S_t(it) complete => PV_t(it-1) complete (issued before it): rescale O_t in place.
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
        // 32 keys -> 16 packed P columns per chunk, stored as they are made
        auto exp_chunks = [&](auto full) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int ip = 16 * q + i;
              const float2 x = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
              float p0, p1;
              if (decltype(full)::value && (ip & 7) < kPolyPairsN) {
                const float2 pp = ex2_poly_x2(x.x, x.y);
                p0 = pp.x;
                p1 = pp.y;
              } else {
                p0 = ex2_approx(x.x);
                p1 = ex2_approx(x.y);
              }
              if constexpr (kSplit) {
                s[2 * ip] = p0;  // summed after P is handed over
                s[2 * ip + 1] = p1;
              } else {
                acc2[i & 3] = fadd2(acc2[i & 3], f2(p0, p1));
              }
              pk[i] = pack_bf16x2(p0, p1);
            }
            tmem_st16(s_addr + 16 * q, pk);
            if constexpr (kSplit) {
              if (q == 2) {  // keys 0-95 stored: PV may start on them
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&bar_p[w]);
              }
            }
          }
        };
        turn_begin(it);
        if (t == 0 && w == 0) TRACE(11, it);
        if (cls == kTileFull) {
          exp_chunks(std::true_type{});
        } else {
          exp_chunks(std::false_type{});
        }
        turn_end();
        if (t == 0 && w == 0) TRACE(10, it);
        if constexpr (kSplit) {
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bar_p2[w]);
#pragma unroll
          for (int i = 0; i < 64; ++i) acc2[i & 3] = fadd2(acc2[i & 3], f2(s[2 * i], s[2 * i + 1]));
        }
        const float2 a01 = unf2(fadd2(acc2[0], acc2[1]));
        const float2 a23 = unf2(fadd2(acc2[2], acc2[3]));
        const float sum = (a01.x + a01.y) + (a23.x + a23.y);
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
      } else {
        turn_begin(it);
        turn_end();
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
        tmem_st32(s_addr, pk);
        tmem_st32(s_addr + 32, pk);
        if constexpr (kSplit) {
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bar_p[w]);
          mbar_arrive(&bar_p2[w]);
        }
      }
      if constexpr (!kSplit) {
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bar_p[w]);
      }
      if (t == 0) TRACE(3 + 2 * w, it);
    }

    if constexpr (kTurn) {
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
      if (row_ok) *lrow = merge ? mw.lse : lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

int attn_n128_launch(const AttnParams& prm, int64_t grid, cudaStream_t st, int form) {
  // form 0: v12, 1: v16 (exp turn-taking), 2: v17 (split P arrive)
  static bool attr_set = false;
  if (!attr_set) {
    RCP_CUDA(cudaFuncSetAttribute(attn_fwd_n128_kernel<false, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytesN));
    RCP_CUDA(cudaFuncSetAttribute(attn_fwd_n128_kernel<true, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytesN));
    RCP_CUDA(cudaFuncSetAttribute(attn_fwd_n128_kernel<false, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytesN));
    attr_set = true;
  }
  const unsigned g = static_cast<unsigned>(grid);
  if (form == 1)
    attn_fwd_n128_kernel<true, false><<<g, kThreads, kSmemBytesN, st>>>(prm);
  else if (form == 2)
    attn_fwd_n128_kernel<false, true><<<g, kThreads, kSmemBytesN, st>>>(prm);
  else
    attn_fwd_n128_kernel<false, false><<<g, kThreads, kSmemBytesN, st>>>(prm);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

}  // namespace rcp
