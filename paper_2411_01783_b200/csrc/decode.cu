// K4: split-KV decode attention for ring pass-Q decode (Alg. 4).
//
// One query token per sequence against that sequence's cached KV shard on this
// rank.  HBM-bound: every cached K/V byte is read once.  Grid = (splits, kv
// heads, batch); a CTA owns kSplit keys of one KV head and all hq/hkv query
// heads that read it (GQA packing, so K/V are not re-read per query head).
// Pass 1 scores the split into shared memory, pass 2 forms the split's
// normalised partial (O_s, LSE_s); a combine kernel folds the splits in
// ascending order with the same fp32 merge as merge_attention.
#include <climits>

#include <cuda_bf16.h>

#include "common.cuh"

namespace rcp {

constexpr int kSplit = 256;       // keys per CTA
constexpr int kDecThreads = 256;  // 8 warps
constexpr int kMaxGroup = 16;     // query heads per KV head handled by one CTA

__global__ void __launch_bounds__(kDecThreads) decode_split_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
    const __nv_bfloat16* __restrict__ v, int64_t kv_row_stride, const int64_t* __restrict__ kv_start,
    const int64_t* __restrict__ kv_len, int hq, int hkv, int n_split, float scale_log2,
    float* __restrict__ part_o, float* __restrict__ part_lse) {
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int g = hq / hkv;
  const int64_t len = kv_len[b];
  const int64_t k0 = static_cast<int64_t>(split) * kSplit;
  const int64_t rem = len - k0;
  const int n = rem <= 0 ? 0 : (rem >= kSplit ? kSplit : static_cast<int>(rem));
  const int64_t out_row = (static_cast<int64_t>(b) * hq + kvh * g);  // first query head row
  if (n <= 0) {
    // empty split: partial is (0, -inf) for each head of the group
    for (int i = threadIdx.x; i < g * 128; i += blockDim.x) {
      const int h = i / 128, d = i % 128;
      part_o[((out_row + h) * n_split + split) * 128 + d] = 0.f;
      if (d == 0) part_lse[(out_row + h) * n_split + split] = -INFINITY;
    }
    return;
  }
  __shared__ float sq[kMaxGroup][128];
  __shared__ float ss[kMaxGroup][kSplit];
  __shared__ float smax[kMaxGroup], ssum[kMaxGroup];
  for (int i = threadIdx.x; i < g * 128; i += blockDim.x) {
    const int h = i / 128, d = i % 128;
    sq[h][d] = __bfloat162float(q[(out_row + h) * 128 + d]);
  }
  __syncthreads();
  const int64_t base = kv_start[b] + k0;
  // pass 1: scores, one key per thread (row of 128 bf16 via 16-byte vectors)
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const uint4* kr = reinterpret_cast<const uint4*>(k + (base + j) * kv_row_stride + kvh * 128);
    float acc[kMaxGroup];
#pragma unroll
    for (int h = 0; h < kMaxGroup; ++h) acc[h] = 0.f;
#pragma unroll 4
    for (int c = 0; c < 16; ++c) {
      const uint4 u = __ldg(kr + c);
      const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&u);
      float kf[8];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = __bfloat1622float2(e[t]);
        kf[2 * t] = f.x;
        kf[2 * t + 1] = f.y;
      }
#pragma unroll
      for (int h = 0; h < kMaxGroup; ++h) {
        if (h < g) {
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[h] = fmaf(sq[h][c * 8 + t], kf[t], acc[h]);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < kMaxGroup; ++h)
      if (h < g) ss[h][j] = acc[h] * scale_log2;
  }
  __syncthreads();
  // per-head max and sum (one warp per head, warps loop over heads)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int h = warp; h < g; h += kDecThreads / 32) {
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) mx = fmaxf(mx, ss[h][j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float e = exp2f(ss[h][j] - mx);
      ss[h][j] = e;
      sum += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      smax[h] = mx;
      ssum[h] = sum;
    }
  }
  __syncthreads();
  // pass 2: O[h][d] = sum_j p[h][j] v[j][d] / l ; thread -> (d pair), loop heads
  for (int i = threadIdx.x; i < g * 64; i += blockDim.x) {
    const int h = i / 64, d2 = i % 64;
    float a0 = 0.f, a1 = 0.f;
    for (int j = 0; j < n; ++j) {
      const __nv_bfloat162 vv = *reinterpret_cast<const __nv_bfloat162*>(
          v + (base + j) * kv_row_stride + kvh * 128 + 2 * d2);
      const float2 f = __bfloat1622float2(vv);
      const float pj = ss[h][j];
      a0 = fmaf(pj, f.x, a0);
      a1 = fmaf(pj, f.y, a1);
    }
    const float inv = 1.f / ssum[h];
    float* dst = part_o + ((out_row + h) * n_split + split) * 128 + 2 * d2;
    dst[0] = a0 * inv;
    dst[1] = a1 * inv;
    if (d2 == 0)
      part_lse[(out_row + h) * n_split + split] =
          (smax[h] + log2f(ssum[h])) * 0.69314718055994530942f;
  }
}

// Fold the splits of each (sequence, query head) row in ascending order.
__global__ void decode_combine_kernel(const float* __restrict__ part_o,
                                      const float* __restrict__ part_lse, int64_t rows,
                                      int n_split, float* __restrict__ o, float* __restrict__ lse) {
  const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float4* po = reinterpret_cast<const float4*>(part_o + row * n_split * 128);
  float4 acc = po[lane];
  float la = part_lse[row * n_split];
  for (int s = 1; s < n_split; ++s) {
    const float lb = part_lse[row * n_split + s];
    const float4 bv = po[s * 32 + lane];
    const MergeW w = merge_weights(la, lb);
    acc.x = merge_val(acc.x, bv.x, w);
    acc.y = merge_val(acc.y, bv.y, w);
    acc.z = merge_val(acc.z, bv.z, w);
    acc.w = merge_val(acc.w, bv.w, w);
    la = w.lse;
  }
  reinterpret_cast<float4*>(o + row * 128)[lane] = acc;
  if (lane == 0) lse[row] = la;
}

}  // namespace rcp

using namespace rcp;

extern "C" size_t rcp_decode_workspace_bytes(int64_t batch, int32_t hq, int64_t max_kv_len) {
  const int64_t ns = (max_kv_len + kSplit - 1) / kSplit;
  const int64_t n_split = ns < 1 ? 1 : ns;
  return static_cast<size_t>(batch * hq * n_split * (128 + 1) * sizeof(float));
}

extern "C" int rcp_decode_attn(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                               const int64_t* kv_start, const int64_t* kv_len, int64_t batch,
                               int64_t max_kv_len, int32_t hq, int32_t hkv, int32_t head_dim,
                               float scale, float* o, float* lse, void* workspace,
                               size_t workspace_bytes, void* stream) {
  RCP_CHECK_ARG(head_dim == 128, "head_dim must be 128, got %d", head_dim);
  RCP_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0,
                "n_query_heads=%d not divisible by n_kv_heads=%d", hq, hkv);
  RCP_CHECK_ARG(hq / hkv <= kMaxGroup, "at most %d query heads per kv head", kMaxGroup);
  RCP_CHECK_ARG(batch >= 0 && max_kv_len >= 0, "bad sizes");
  if (batch == 0) return RCP_OK;
  RCP_CHECK_ARG(q && o && lse && kv_start && kv_len, "null pointer");
  RCP_CHECK_ARG(kv_row_stride % 8 == 0, "kv row stride must be a multiple of 8");
  const size_t need = rcp_decode_workspace_bytes(batch, hq, max_kv_len);
  RCP_CHECK_ARG(workspace && workspace_bytes >= need, "workspace too small: need %zu", need);
  const int64_t ns = (max_kv_len + kSplit - 1) / kSplit;
  const int n_split = static_cast<int>(ns < 1 ? 1 : ns);
  float* part_o = static_cast<float*>(workspace);
  float* part_lse = part_o + batch * hq * n_split * 128;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float sl2 = static_cast<float>(static_cast<double>(scale) * 1.4426950408889634);
  dim3 grid(n_split, hkv, static_cast<unsigned>(batch));
  decode_split_kernel<<<grid, kDecThreads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
      static_cast<const __nv_bfloat16*>(v), kv_row_stride, kv_start, kv_len, hq, hkv, n_split, sl2,
      part_o, part_lse);
  RCP_CUDA(cudaGetLastError());
  const int64_t rows = batch * hq;
  decode_combine_kernel<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(
      part_o, part_lse, rows, n_split, o, lse);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}
