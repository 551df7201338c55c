// K1: causal-by-position GQA flash-attention forward for sm_100a with LSE.
//
// Replaces ringcp.attention.gqa_attention (attention.py:230-282) on the ring
// hot path.  One CTA = two 128-row query tiles of one query head; the tiles
// share every K/V tile the TMA producer streams through a 2-stage ring.
//
// Warp roles (384 threads):
//   warp 0      TMA producer (one elected lane): Q once, then K_j / V_j
//   warp 1      MMA issuer (one elected lane):   S_t = Q_t K_j^T  (SS, K-major)
//                                                O_t += P_t V_j   (TS, P in TMEM)
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1)
//   warps 4-7   softmax for query tile 0 (thread i owns TMEM lane / row i)
//   warps 8-11  softmax for query tile 1
// The MMA order S0(j) S1(j) | PV0(j) S0(j+1) PV1(j) S1(j+1) | ... lets softmax of
// one tile overlap the tensor-core work of the other ("ping-pong").  P_t is
// written as packed bf16 into the first 64 columns of S_t's TMEM region and
// consumed from TMEM by the TS MMA.  tcgen05 ops complete in issue order, so
// the commit that publishes S_t(j) also proves PV_t(j-1) finished — the softmax
// may then rescale O_t in place without another barrier.
//
// Masking: per-tile summaries (min/max position and sequence over valid rows)
// classify every (query tile, key tile) pair as EMPTY (skipped: no TMA, no MMA),
// FULL (no per-element mask) or PARTIAL (per-element seq/pos test), which keeps
// the general position-based mask of the reference off the dense path.
// Softmax runs in the exp2 domain with a lazily raised running max (rescale O
// only when the max grows by more than 2^8); LSE = (m + log2 l) * ln 2 (natural
// log, as attention.py:274-277) and rows that admit nothing give 0 / -inf.
#include <climits>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace rcp {

constexpr int kD = 128;
constexpr int kTileRows = 128;
constexpr int kStages = 2;
constexpr int kThreads = 384;
constexpr uint32_t kTileBytes = kTileRows * kD * 2;  // 32 KB: two 16 KB SW128 boxes
constexpr uint32_t kBoxBytes = kTileBytes / 2;
constexpr uint32_t kSmemBytes = (2 + 2 * kStages) * kTileBytes + 1024;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct AttnParams {
  CUtensorMap tm_q, tm_k, tm_v;
  const int32_t* q_pos;
  const int32_t* q_seq;
  const int32_t* k_pos;
  const int32_t* k_seq;
  const TileSum* q_sum;
  const TileSum* k_sum;
  float* o;
  float* lse;
  int tq, tk, hq, hkv, group;
  int n_qtiles, n_qblk, n_ktiles;
  int mode;
  float scale_log2;
};

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

// Next key tile after j that is non-empty for either query tile (-1: done).
__device__ __forceinline__ int next_active(const AttnParams& p, int j, const TileSum& q0,
                                           const TileSum& q1) {
  for (++j; j < p.n_ktiles; ++j) {
    const TileSum k = load_sum(p.k_sum, j, p.n_ktiles);
    if (classify_tile(q0, k) != kTileEmpty || classify_tile(q1, k) != kTileEmpty) return j;
  }
  return -1;
}

__device__ __forceinline__ uint64_t kmajor_desc(uint32_t tile_addr, int kk) {
  // K-major SW128: 8-row groups 1024 B apart; k-step kk (16 elements) selects
  // box kk/4 and a 32-byte column offset inside the 128-byte swizzle row.
  return make_sw128_desc(tile_addr + (kk >> 2) * kBoxBytes + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t tile_addr, int kk) {
  // MN-major SW128 (V as B operand, N = head dim contiguous): the two 64-column
  // boxes are LBO = 16 KB apart, 8-key groups SBO = 1 KB; k-step = 16 keys.
  return make_sw128_desc(tile_addr + kk * 2048, kBoxBytes, 1024);
}

__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                        // 2 tiles
  uint8_t* sK = smem + 2 * kTileBytes;       // kStages tiles
  uint8_t* sV = sK + kStages * kTileBytes;   // kStages tiles

  __shared__ uint64_t bar_q, bar_kf[kStages], bar_ke[kStages], bar_vf[kStages], bar_ve[kStages];
  __shared__ uint64_t bar_s[2], bar_p[2], bar_o[2];
  __shared__ uint32_t tmem_slot;

  const int warp = static_cast<int>(warp_id());
  const int head = blockIdx.x % p.hq;
  const int qblk = p.n_qblk - 1 - static_cast<int>(blockIdx.x / p.hq);  // late (heavy) blocks first
  const int kvh = head / p.group;
  const TileSum qs0 = load_sum(p.q_sum, 2 * qblk, p.n_qtiles);
  const TileSum qs1 = load_sum(p.q_sum, 2 * qblk + 1, p.n_qtiles);

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar_kf[s], 1);
      mbar_init(&bar_ke[s], 1);
      mbar_init(&bar_vf[s], 1);
      mbar_init(&bar_ve[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t], 1);
      mbar_init(&bar_p[t], 128);
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
    if (elect_one()) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      int j = next_active(p, -1, qs0, qs1);
      if (j >= 0) {
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        mbar_arrive_expect_tx(&bar_q, 2 * kTileBytes);
        for (int t = 0; t < 2; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sQ + t * kTileBytes + h * kBoxBytes, &p.tm_q, &bar_q, head * kD + h * 64,
                        (2 * qblk + t) * kTileRows, pol_q);
        for (int it = 0; j >= 0; j = next_active(p, j, qs0, qs1), ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&bar_ke[s], ph ^ 1);
          mbar_arrive_expect_tx(&bar_kf[s], kTileBytes);
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sK + s * kTileBytes + h * kBoxBytes, &p.tm_k, &bar_kf[s],
                        kvh * kD + h * 64, j * kTileRows, pol_kv);
          mbar_wait(&bar_ve[s], ph ^ 1);
          mbar_arrive_expect_tx(&bar_vf[s], kTileBytes);
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sV + s * kTileBytes + h * kBoxBytes, &p.tm_v, &bar_vf[s],
                        kvh * kD + h * 64, j * kTileRows, pol_kv);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc_s = make_idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16_f32(128, 128, 0, 1);
      const uint32_t q_addr = smem_u32(sQ), k_addr = smem_u32(sK), v_addr = smem_u32(sV);
      auto issue_s = [&](int t, int stage) {
        const uint32_t qa = q_addr + t * kTileBytes, ka = k_addr + stage * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          mma_ss(tmem + t * 128, kmajor_desc(qa, kk), kmajor_desc(ka, kk), idesc_s, kk > 0);
      };
      auto issue_pv = [&](int t, int stage, bool acc) {
        const uint32_t va = v_addr + stage * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kTileRows / 16; ++kk)
          mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmajor_desc(va, kk), idesc_o,
                 (acc || kk > 0) ? 1u : 0u);
      };
      int j = next_active(p, -1, qs0, qs1);
      if (j >= 0) {
        mbar_wait(&bar_q, 0);
        mbar_wait(&bar_kf[0], 0);
        tc_fence_after();
        issue_s(0, 0);
        mma_commit(&bar_s[0]);
        issue_s(1, 0);
        mma_commit(&bar_s[1]);
        mma_commit(&bar_ke[0]);
        for (int it = 0;; ++it) {
          const int jn = next_active(p, j, qs0, qs1);
          const int s = it % kStages;
          const int s1 = (it + 1) % kStages;
          const uint32_t ph1 = ((it + 1) / kStages) & 1;
          mbar_wait(&bar_vf[s], (it / kStages) & 1);
          mbar_wait(&bar_p[0], it & 1);
          tc_fence_after();
          issue_pv(0, s, it > 0);
          if (jn >= 0) {
            mbar_wait(&bar_kf[s1], ph1);
            tc_fence_after();
            issue_s(0, s1);
            mma_commit(&bar_s[0]);
          } else {
            mma_commit(&bar_o[0]);
          }
          mbar_wait(&bar_p[1], it & 1);
          tc_fence_after();
          issue_pv(1, s, it > 0);
          mma_commit(&bar_ve[s]);
          if (jn >= 0) {
            issue_s(1, s1);
            mma_commit(&bar_s[1]);
            mma_commit(&bar_ke[s1]);
          } else {
            mma_commit(&bar_o[1]);
            break;
          }
          j = jn;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int w = (warp - 4) >> 2;                  // query tile 0 / 1
    const int t = static_cast<int>(threadIdx.x) - 128 - 128 * w;  // row inside the tile
    const int row = (2 * qblk + w) * kTileRows + t;
    const TileSum& qs = w ? qs1 : qs0;
    const bool row_ok = row < p.tq;
    const int my_pos = row_ok ? __ldg(p.q_pos + row) : -1;
    const int my_seq = row_ok ? __ldg(p.q_seq + row) : RCP_SEQ_PAD_Q;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t s_addr = lane_base + w * 128;
    const uint32_t o_addr = lane_base + 256 + w * 128;
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    int it = 0;
    for (int j = next_active(p, -1, qs0, qs1); j >= 0; j = next_active(p, j, qs0, qs1), ++it) {
      const TileSum ks = load_sum(p.k_sum, j, p.n_ktiles);
      const int cls = classify_tile(qs, ks);
      mbar_wait(&bar_s[w], it & 1);
      tc_fence_after();
      uint32_t pk[64];
      if (cls != kTileEmpty) {
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 128; c += 32) tmem_ld32(s_addr + c, sr + c);
        tmem_ld_wait();
        float s[128];
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = __uint_as_float(sr[c]);
        if (cls == kTilePartial) {
          const int base = j * kTileRows;
          if (base + kTileRows <= p.tk) {
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
        float mx = s[0];
#pragma unroll
        for (int c = 1; c < 128; ++c) mx = fmaxf(mx, s[c]);
        const float m_old = m;
        const float m_new = fmaxf(m, mx * sl2);
        const bool need = m_new > m + kRescaleThreshold;  // also true for -inf -> finite
        if (need) m = m_new;
        // Rows that have admitted nothing yet keep m = -inf: their scores are all
        // -inf, so exp2(s - 0) = 0.  Everything below is warp-uniform (the
        // tcgen05.ld/st are .sync.aligned).
        const float m_use = (m == -INFINITY) ? 0.f : m;
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < 128; c += 2) {
          const float p0 = ex2_approx(fmaf(s[c], sl2, -m_use));
          const float p1 = ex2_approx(fmaf(s[c + 1], sl2, -m_use));
          sum += p0 + p1;
          pk[c >> 1] = pack_bf16x2(p0, p1);
        }
        const float f = (need && m_old != -INFINITY) ? ex2_approx(m_old - m) : 1.0f;
        l = (m_old == -INFINITY ? 0.f : l * f) + sum;
        tmem_st32(s_addr, pk);
        tmem_st32(s_addr + 32, pk + 32);
        if (__any_sync(0xffffffffu, f != 1.0f && it > 0)) {
          // Rescale O_t rows in place (TMEM); PV_t(it-1) is complete (see header).
#pragma unroll
          for (int c = 0; c < 128; c += 32) {
            uint32_t r[32];
            tmem_ld32(o_addr + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st32(o_addr + c, r);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) pk[i] = 0u;
        tmem_st32(s_addr, pk);
        tmem_st32(s_addr + 32, pk + 32);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bar_p[w]);
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
      if (merge && row_ok) mw = merge_weights(__ldg(lrow), lse_new);
#pragma unroll
      for (int c = 0; c < 128; c += 32) {
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

// 2-D map over a token-major [rows, heads*128] bf16 array; box = 128 rows x 64 cols, SW128.
static int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols,
                    int64_t row_stride_elems) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return RCP_ERR_CUDA;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_elems) * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
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

extern "C" size_t rcp_attn_workspace_bytes(int64_t tq, int64_t tk) {
  return static_cast<size_t>(((tq + 127) / 128 + (tk + 127) / 128) * sizeof(TileSum));
}

extern "C" int rcp_attn_fwd(const void* q, int64_t q_row_stride, const void* k,
                            int64_t k_row_stride, const void* v, int64_t v_row_stride,
                            const int32_t* q_pos, const int32_t* q_seq, const int32_t* k_pos,
                            const int32_t* k_seq, int64_t tq, int64_t tk, int32_t hq,
                            int32_t hkv, int32_t head_dim, float scale, float* o, float* lse,
                            int32_t mode, void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
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
  RCP_CHECK_ARG(q_row_stride % 8 == 0 && k_row_stride % 8 == 0 && v_row_stride % 8 == 0,
                "row strides must be multiples of 8 elements");
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

  AttnParams prm;
  memset(&prm, 0, sizeof(prm));
  int rc;
  if ((rc = make_map(&prm.tm_q, q, tq, static_cast<int64_t>(hq) * kD, q_row_stride)) != RCP_OK) return rc;
  if ((rc = make_map(&prm.tm_k, k, tk, static_cast<int64_t>(hkv) * kD, k_row_stride)) != RCP_OK) return rc;
  if ((rc = make_map(&prm.tm_v, v, tk, static_cast<int64_t>(hkv) * kD, v_row_stride)) != RCP_OK) return rc;
  TileSum* qsum = static_cast<TileSum*>(workspace);
  const int n_qtiles = static_cast<int>((tq + 127) / 128);
  const int n_ktiles = static_cast<int>((tk + 127) / 128);
  TileSum* ksum = qsum + n_qtiles;
  if ((rc = launch_tile_summary(q_pos, q_seq, tq, RCP_SEQ_PAD_Q, qsum, st)) != RCP_OK) return rc;
  if ((rc = launch_tile_summary(k_pos, k_seq, tk, RCP_SEQ_PAD_K, ksum, st)) != RCP_OK) return rc;
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
  prm.n_ktiles = n_ktiles;
  prm.mode = mode;
  prm.scale_log2 = static_cast<float>(static_cast<double>(scale) * 1.4426950408889634);

  static bool attr_set = false;
  if (!attr_set) {
    RCP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBytes));
    attr_set = true;
  }
  const int64_t grid = static_cast<int64_t>(prm.n_qblk) * hq;
  RCP_CHECK_ARG(grid < (1ll << 31), "grid too large");
  attn_fwd_kernel<<<static_cast<unsigned>(grid), kThreads, kSmemBytes, st>>>(prm);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}
