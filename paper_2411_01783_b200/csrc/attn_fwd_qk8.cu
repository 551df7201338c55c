// K1 with FP8 (e4m3) Q and K: S = Q K^T on the tensor cores' 8-bit path
// (tcgen05.mma kind::f8f6f4, K = 32 per instruction: half the S MMAs and half
// the shared-memory operand bytes of the bf16 form), P and V stay bf16.  An
// opt-in mode outside the bf16 parity
// contract: Q / K are quantised per head (rcp_kv_quantize_e4m3), the
// dequantisation scales fold into the softmax scale, and parity is checked
// against the oracle on the DEQUANTISED Q / K.
//
// Generated from the v4g kernel in attn_fwd.cu (same roles, TMEM layout,
// pipeline, masking and epilogue); only the Q / K staging and the S MMAs
// differ: Q tiles are one 16 KB SW128 box (128 rows x 128 bytes), a K block
// one 8 KB box in the first half of its 16 KB ring slot.
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

#include "attn_common.cuh"

#ifndef RCP_PACKED_POLY
#define RCP_PACKED_POLY 1
#endif

namespace rcp {

constexpr uint32_t kQTileBytes8 = kQRows * kD;    // 16 KB: 128 rows x 128 e4m3 (one SW128 box)
constexpr uint32_t kKBytes8 = kKRows * kD;        // 8 KB
constexpr uint32_t kSmemBytesQK8 = 2 * kQTileBytes8 + kSlots * kKVBytes + 1024;
#ifndef RCP_POLY_MASK
#define RCP_POLY_MASK 0x00070007u
#endif
constexpr uint32_t kPolyMask8 = RCP_POLY_MASK;
#define kPolyMask kPolyMask8
#ifndef RCP_DBG_NO_EXP
#define RCP_DBG_NO_EXP 0
#endif

__global__ void __launch_bounds__(kThreads, 1) attn_fwd_qk8_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // 2 query tiles
  uint8_t* sKV = smem + 2 * kQTileBytes8;     // kSlots K/V blocks (K uses the first 8 KB of a slot)

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
        mbar_arrive_expect_tx(&bar_q, 2 * kQTileBytes8);
        for (int t = 0; t < 2; ++t)  // e4m3 Q: one 128-byte-row box per tile
          tma_load_2d(sQ + t * kQTileBytes8, &p.tm_q, &bar_q, head * kD, (2 * qblk + t) * kQRows, pol_q);
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
            if (kv == 0) {  // e4m3 K: one 8 KB box
              mbar_arrive_expect_tx(&bar_full[slot], kKBytes8);
              tma_load_2d(sKV + slot * kKVBytes, &p.tm_k, &bar_full[slot], kvh * kD, j * kKRows, pol_kv);
            } else {        // bf16 V: two 8 KB boxes
              mbar_arrive_expect_tx(&bar_full[slot], kKVBytes);
              for (int h = 0; h < 2; ++h)
                tma_load_2d(sKV + slot * kKVBytes + h * kKVBoxBytes, &p.tm_v, &bar_full[slot],
                            kvh * kD + h * 64, j * kKRows, pol_kv);
            }
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
      const uint32_t idesc_s = make_idesc_e4m3_f32(kQRows, kKRows);
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
        const uint32_t qa = q_lo + ((tt * kQTileBytes8) >> 4);
        const uint32_t ka = k_lo + (((ld % kSlots) * kKVBytes) >> 4);
        const uint32_t d = tmem + kTmemS + (2 * tt + buf) * kKRows;
#pragma unroll
        for (int kk = 0; kk < kD / 32; ++kk)  // e4m3: K = 32 per MMA, 32 bytes along the 128-byte row
          mma_ss_f8_lo(d, qa + ((kk * 32) >> 4), ka + ((kk * 32) >> 4), idesc_s, kk > 0);
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
    // fp8 Q / K: the per-head dequantisation scales fold into the softmax scale
    const float sl2 = p.scale_log2 * __ldg(p.q_scale + head) * __ldg(p.k_scale + kvh);
    const uint64_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    const int n = __ldg(p.act_n + qblk);
    const uint32_t* act = p.act + static_cast<int64_t>(qblk) * p.n_kblocks;
    uint32_t e_next = n > 0 ? __ldg(act) : 0u;
    int it = 0;
    for (; it < n; ++it) {
      const int buf = it & 1;
      const uint32_t s_addr = lane_base + kTmemS + (2 * w + buf) * kKRows;
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

#undef kPolyMask

int attn_qk8_launch(const AttnParams& prm, int64_t grid, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    RCP_CUDA(cudaFuncSetAttribute(attn_fwd_qk8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBytesQK8));
    attr_set = true;
  }
  attn_fwd_qk8_kernel<<<static_cast<unsigned>(grid), kThreads, kSmemBytesQK8, st>>>(prm);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

}  // namespace rcp
