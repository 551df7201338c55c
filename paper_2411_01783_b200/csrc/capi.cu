// C-ABI plumbing and the HBM-bound helper kernels of ringcp-b200:
// error state, tile summaries, metadata folding, the N-way LSE merge (K2),
// the empty-result fill, the row gathers behind materialize_rank_block (K0)
// and its inverse scatter (rank slots -> token order).
#include <climits>
#include <cstring>
#include <string>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace rcp {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

// ------------------------------------------------------------------ tile summary
// One CTA of `rows` (64 or 128) threads per tile.
__global__ void __launch_bounds__(128) tile_summary_kernel(const int32_t* __restrict__ pos,
                                                           const int32_t* __restrict__ seq,
                                                           int64_t n, int32_t pad_seq,
                                                           TileSum* __restrict__ out) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int p = 0, s = 0;
  bool valid = false;
  if (row < n) {
    s = seq[row];
    p = pos[row];
    valid = (s != pad_seq);
  }
  int pmin = valid ? p : INT_MAX, pmax = valid ? p : INT_MIN;
  int smin = valid ? s : INT_MAX, smax = valid ? s : INT_MIN;
  int cnt = valid ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pmin = min(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
    pmax = max(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, o));
    smax = max(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  __shared__ int red[4][5];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[w][0] = pmin;
    red[w][1] = pmax;
    red[w][2] = smin;
    red[w][3] = smax;
    red[w][4] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    TileSum t = {INT_MAX, INT_MIN, INT_MAX, INT_MIN, 0, 0, 0, 0};
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
      t.pmin = min(t.pmin, red[i][0]);
      t.pmax = max(t.pmax, red[i][1]);
      t.smin = min(t.smin, red[i][2]);
      t.smax = max(t.smax, red[i][3]);
      t.nvalid += red[i][4];
    }
    t.uniform = (t.nvalid == static_cast<int>(blockDim.x) && t.smin == t.smax) ? 1 : 0;
    t.pad0 = t.pad1 = 0;
    out[blockIdx.x] = t;
  }
}

int launch_tile_summary(const int32_t* pos, const int32_t* seq, int64_t n, int32_t pad_seq,
                        int rows, TileSum* out, cudaStream_t stream) {
  const int64_t tiles = (n + rows - 1) / rows;
  if (tiles == 0) return RCP_OK;
  tile_summary_kernel<<<static_cast<unsigned>(tiles), rows, 0, stream>>>(pos, seq, n, pad_seq,
                                                                          out);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

// ------------------------------------------------------------------ metadata fold
__global__ void fold_meta_kernel(const int64_t* __restrict__ pos, const int64_t* __restrict__ seq,
                                 const uint8_t* __restrict__ valid, int64_t n, int32_t is_key,
                                 int32_t* __restrict__ pos_out, int32_t* __restrict__ seq_out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool ok = valid[i] != 0;
    if (ok) {
      pos_out[i] = static_cast<int32_t>(pos[i]);
      seq_out[i] = static_cast<int32_t>(seq[i]);
    } else {
      pos_out[i] = is_key ? RCP_POS_PAD_K : -1;
      seq_out[i] = is_key ? RCP_SEQ_PAD_K : RCP_SEQ_PAD_Q;
    }
  }
}

// ------------------------------------------------------------------ fill / merge
__global__ void fill_empty_kernel(float4* __restrict__ o, float* __restrict__ lse, int64_t rows) {
  const int64_t n4 = rows * 32;  // 128 floats per row
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    o[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((i & 31) == 0) lse[i >> 5] = -INFINITY;
  }
}

constexpr int kMaxMergeParts = 64;
struct MergeArgs {
  const float* o[kMaxMergeParts];
  const float* lse[kMaxMergeParts];
};

// One warp per (token, head) row of D values (D % 4 == 0), float4 per lane.
// Left fold over parts in list order — merge_attention (attention.py:319-334).
__global__ void __launch_bounds__(256) merge_kernel(const __grid_constant__ MergeArgs a,
                                                    int32_t n, int64_t rows, int32_t d4,
                                                    float* __restrict__ o_out,
                                                    float* __restrict__ lse_out) {
  const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float la_final = 0.f;
  for (int c = lane; c < d4; c += 32) {
    float4 acc = __ldg(reinterpret_cast<const float4*>(a.o[0] + row * d4 * 4) + c);
    float la = __ldg(a.lse[0] + row);
    for (int s = 1; s < n; ++s) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(a.o[s] + row * d4 * 4) + c);
      const float lb = __ldg(a.lse[s] + row);
      const MergeW w = merge_weights(la, lb);
      acc.x = merge_val(acc.x, b.x, w);
      acc.y = merge_val(acc.y, b.y, w);
      acc.z = merge_val(acc.z, b.z, w);
      acc.w = merge_val(acc.w, b.w, w);
      la = w.lse;
    }
    reinterpret_cast<float4*>(o_out + row * d4 * 4)[c] = acc;
    la_final = la;
  }
  if (lane == 0) lse_out[row] = la_final;
}

// Fixed-N form of the merge (N = 2..8, the ring sizes): one warp per 32 rows.
// Lane i first computes row i's whole chain of pairwise merge weights (the
// same merge_weights calls, in the same order, as merge_kernel and the fused
// attention epilogue, so the result is bitwise identical), keeping the
// (wa, wb) of every step in registers; then the warp streams the 32 rows with
// one float4 per lane, all N partial loads of a row issued before the fold
// and the step weights broadcast by shuffles.  The weight chain (4 expf + 1
// logf per step) is computed once per row instead of once per lane.
template <int N>
__global__ void __launch_bounds__(256) merge_rows32_kernel(const __grid_constant__ MergeArgs a, int64_t rows,
                                                           float* __restrict__ o_out,
                                                           float* __restrict__ lse_out) {
  const int lane = threadIdx.x & 31;
  const int64_t row0 = ((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5) * 32;
  if (row0 >= rows) return;
  float wa[N], wb[N];
  {
    const int64_t r = row0 + lane;
    float la = r < rows ? __ldg(a.lse[0] + r) : -INFINITY;
    wa[0] = wb[0] = 0.f;
#pragma unroll
    for (int s = 1; s < N; ++s) {
      const float lb = r < rows ? __ldg(a.lse[s] + r) : -INFINITY;
      const MergeW w = merge_weights(la, lb);
      wa[s] = w.wa;
      wb[s] = w.wb;
      la = w.lse;
    }
    if (r < rows) lse_out[r] = la;
  }
  const int64_t nr = rows - row0 < 32 ? rows - row0 : 32;
  for (int rr = 0; rr < nr; ++rr) {
    const int64_t row = row0 + rr;
    float4 v[N];
#pragma unroll
    for (int s = 0; s < N; ++s) v[s] = __ldg(reinterpret_cast<const float4*>(a.o[s] + row * 128) + lane);
    float4 acc = v[0];
#pragma unroll
    for (int s = 1; s < N; ++s) {
      MergeW w;
      w.wa = __shfl_sync(0xffffffffu, wa[s], rr);
      w.wb = __shfl_sync(0xffffffffu, wb[s], rr);
      acc.x = merge_val(acc.x, v[s].x, w);
      acc.y = merge_val(acc.y, v[s].y, w);
      acc.z = merge_val(acc.z, v[s].z, w);
      acc.w = merge_val(acc.w, v[s].w, w);
    }
    reinterpret_cast<float4*>(o_out + row * 128)[lane] = acc;
  }
}

// ------------------------------------------------------------------ gathers
// Generic row gather, one warp per row, 16-byte vectors:
// dst[i] = idx[i] >= 0 ? src[idx[i]] : 0.
__global__ void gather_rows_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                   const int64_t* __restrict__ idx, int64_t n_rows,
                                   int64_t vec_per_row) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
       r < n_rows; r += warps) {
    const int64_t s = idx[r];
    uint4* d = dst + r * vec_per_row;
    if (s >= 0) {
      const uint4* sp = src + s * vec_per_row;
      for (int64_t c = lane; c < vec_per_row; c += 32) d[c] = __ldg(sp + c);
    } else {
      for (int64_t c = lane; c < vec_per_row; c += 32) d[c] = make_uint4(0, 0, 0, 0);
    }
  }
}

constexpr int kMaxShardSeqs = 64;
struct ShardArgs {
  const uint4* src[kMaxShardSeqs];
  int64_t slot_begin[kMaxShardSeqs + 1];  // first dst slot of each sequence
  int64_t chunk[kMaxShardSeqs];           // chunk_len = ceil(T / 2N)
  int64_t new_len[kMaxShardSeqs];
  int64_t cached[kMaxShardSeqs];
  int64_t seq_id[kMaxShardSeqs];
};

// materialize_rank_block on device (sharding.py:105-115, 211-240): slot s of
// sequence i holds local token lo*c + s (s < c) or hi*c + (s - c), where
// (lo, hi) = (rank, 2N-1-rank); local indices >= new_len are padding.
// One warp per destination slot; lanes stream the row in 16-byte vectors.
__global__ void shard_gather_kernel(const __grid_constant__ ShardArgs a, int32_t n_seqs,
                                    int32_t n_ranks, int32_t rank, int64_t vec_per_row,
                                    uint4* __restrict__ dst, int32_t* __restrict__ pos_out,
                                    int32_t* __restrict__ seq_out, int32_t is_key) {
  const int lane = threadIdx.x & 31;
  const int64_t total_slots = a.slot_begin[n_seqs];
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t slot = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
       slot < total_slots; slot += warps) {
    int sq = 0;
    while (sq + 1 < n_seqs && a.slot_begin[sq + 1] <= slot) ++sq;
    const int64_t s = slot - a.slot_begin[sq];
    const int64_t ch = a.chunk[sq];
    const int64_t chunk_id = s < ch ? rank : 2 * n_ranks - 1 - rank;
    const int64_t local = chunk_id * ch + (s < ch ? s : s - ch);
    const bool valid = local < a.new_len[sq];
    uint4* d = dst + slot * vec_per_row;
    if (valid) {
      const uint4* sp = a.src[sq] + local * vec_per_row;
      for (int64_t c = lane; c < vec_per_row; c += 32) d[c] = __ldg(sp + c);
    } else {
      for (int64_t c = lane; c < vec_per_row; c += 32) d[c] = make_uint4(0, 0, 0, 0);
    }
    if (lane == 0 && pos_out != nullptr) {
      pos_out[slot] = valid ? static_cast<int32_t>(a.cached[sq] + local)
                            : (is_key ? RCP_POS_PAD_K : -1);
      seq_out[slot] = valid ? static_cast<int32_t>(a.seq_id[sq])
                            : (is_key ? RCP_SEQ_PAD_K : RCP_SEQ_PAD_Q);
    }
  }
}

// Inverse of shard_gather_kernel (the scatter half of materialize_rank_block,
// sharding.py:105-115, 211-240): every VALID slot of this rank's block goes
// back to row `local` of its sequence's token-ordered array; padding slots are
// dropped.  Each destination row is written by exactly one (rank, slot), so
// the N ranks' scatters tile the sequence.
// (ShardArgs.src carries the per-sequence DESTINATION rows here.)
__global__ void shard_scatter_kernel(const __grid_constant__ ShardArgs a, int32_t n_seqs, int32_t n_ranks,
                                     int32_t rank, int64_t vec_per_row, const uint4* __restrict__ src) {
  const int lane = threadIdx.x & 31;
  const int64_t total_slots = a.slot_begin[n_seqs];
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t slot = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
       slot < total_slots; slot += warps) {
    int sq = 0;
    while (sq + 1 < n_seqs && a.slot_begin[sq + 1] <= slot) ++sq;
    const int64_t s = slot - a.slot_begin[sq];
    const int64_t ch = a.chunk[sq];
    const int64_t chunk_id = s < ch ? rank : 2 * n_ranks - 1 - rank;
    const int64_t local = chunk_id * ch + (s < ch ? s : s - ch);
    if (local >= a.new_len[sq]) continue;  // warp-uniform
    const uint4* sp = src + slot * vec_per_row;
    uint4* d = const_cast<uint4*>(a.src[sq]) + local * vec_per_row;
    for (int64_t c = lane; c < vec_per_row; c += 32) d[c] = __ldg(sp + c);
  }
}

// Row `*counter` of a [n_rows, row_elems] int64 table -> dst, then ++*counter
// (clamped at n_rows - 1).  One CTA; lets a replayed CUDA graph step through
// metadata precomputed for all of its future steps without a host upload.
__global__ void __launch_bounds__(256) step_select_kernel(int64_t* __restrict__ dst,
                                                          const int64_t* __restrict__ table, int64_t row_elems,
                                                          int64_t* __restrict__ counter, int64_t n_rows) {
  __shared__ int64_t c;
  if (threadIdx.x == 0) c = *counter;
  __syncthreads();
  const int64_t r = c < n_rows ? c : n_rows - 1;
  for (int64_t i = threadIdx.x; i < row_elems; i += blockDim.x) dst[i] = table[r * row_elems + i];
  __syncthreads();
  if (threadIdx.x == 0) *counter = c + 1;
}

// fp32 -> bf16 (round to nearest even), 4 values per thread: the final
// attention output in the model dtype for a host copy of half the bytes.
__global__ void cast_f32_bf16_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = __ldg(src + i);
    uint32_t lo, hi;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(v.y), "f"(v.x));
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(v.w), "f"(v.z));
    dst[i] = make_uint2(lo, hi);
  }
}

static unsigned grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

// ------------------------------------------------- P2P (NVLink peer memory) transport
// The decode step's Q all-gather and partial All2All as plain kernels over
// CUDA-IPC-mapped buffers (rcp_ipc_*), graph-capturable: a put kernel stores
// into every peer's buffer, a signal kernel publishes the step's epoch into
// each peer's flag slot for this rank (release, system scope), and a wait
// kernel spins until every peer's flag in this rank's buffer reached the
// epoch (acquire).  The epoch is a device counter advanced once per step.
__global__ void p2p_epoch_kernel(unsigned long long* epoch) { *epoch += 1ull; }

__global__ void __launch_bounds__(256) p2p_put_kernel(void* const* __restrict__ dst, int n,
                                                      const uint4* __restrict__ src, int64_t n16,
                                                      unsigned long long* const* flag_dst,
                                                      unsigned long long* epoch, unsigned* counter) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(src + i);
    for (int p = 0; p < n; ++p) reinterpret_cast<uint4*>(dst[p])[i] = v;
  }
  if (flag_dst) {
    p2p_last_block_signal(counter, flag_dst, n, epoch, true);  // advance the epoch, then signal
  } else {
    __threadfence_system();
  }
}

__global__ void p2p_signal_kernel(unsigned long long* const* __restrict__ flag_dst, int n,
                                  const unsigned long long* __restrict__ epoch) {
  __threadfence_system();
  const unsigned long long e = *epoch;
  for (int p = threadIdx.x; p < n; p += blockDim.x)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag_dst[p]), "l"(e) : "memory");
}

__global__ void p2p_wait_kernel(const unsigned long long* __restrict__ flags, int n,
                                const unsigned long long* __restrict__ epoch, int* __restrict__ timed_out) {
  const unsigned long long e = *epoch;
  const long long t0 = clock64();
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    unsigned long long v;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + p) : "memory");
      if (v >= e) break;
      if (clock64() - t0 > (1ll << 34)) {  // ~9 s: a peer is gone — record it and fail loudly
        atomicExch(timed_out, 1);          // (the trap surfaces as a CUDA error at the next sync)
        __threadfence_system();
        __trap();
      }
      __nanosleep(64);
    }
  }
}

// Debug timeline stamp: slots[*counter % n_slots] = %globaltimer (ns), counter++.
__global__ void debug_stamp_kernel(unsigned long long* slots, unsigned long long* counter, int n_slots) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned long long i = (*counter)++;
  slots[i % static_cast<unsigned long long>(n_slots)] = t;
}

}  // namespace rcp

using namespace rcp;

extern "C" {

const char* rcp_last_error(void) { return g_last_error.c_str(); }

const char* rcp_version(void) { return "ringcp_b200 0.1.0 sm_100a"; }

int rcp_fold_meta(const int64_t* pos, const int64_t* seq, const uint8_t* valid, int64_t n,
                  int32_t is_key, int32_t* pos_out, int32_t* seq_out, void* stream) {
  RCP_CHECK_ARG(n >= 0, "n must be >= 0");
  if (n == 0) return RCP_OK;
  RCP_CHECK_ARG(pos && seq && valid && pos_out && seq_out, "null pointer");
  fold_meta_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      pos, seq, valid, n, is_key, pos_out, seq_out);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_fill_empty(float* o, float* lse, int64_t rows, int32_t head_dim, void* stream) {
  RCP_CHECK_ARG(head_dim == 128, "head_dim must be 128, got %d", head_dim);
  RCP_CHECK_ARG(rows >= 0, "rows must be >= 0");
  if (rows == 0) return RCP_OK;
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(o) & 15) == 0, "o must be 16-byte aligned");
  fill_empty_kernel<<<grid_for(rows * 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float4*>(o), lse, rows);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_merge_attn(const float* const* o_parts, const float* const* lse_parts, int32_t n,
                   int64_t rows, int32_t head_dim, float* o_out, float* lse_out, void* stream) {
  RCP_CHECK_ARG(n >= 1, "cannot merge an empty list of partials");
  RCP_CHECK_ARG(n <= kMaxMergeParts, "at most %d partials per merge call", kMaxMergeParts);
  RCP_CHECK_ARG(head_dim >= 4 && head_dim % 4 == 0, "head_dim must be a positive multiple of 4");
  RCP_CHECK_ARG(rows >= 0, "rows must be >= 0");
  if (rows == 0) return RCP_OK;
  MergeArgs a;
  memset(&a, 0, sizeof(a));
  const bool reverse = (rcp_fault_flags() & kFaultReverseMerge) != 0;  // negative control only
  for (int i = 0; i < n; ++i) {
    RCP_CHECK_ARG(o_parts[i] && lse_parts[i], "null partial %d", i);
    RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(o_parts[i]) & 15) == 0,
                  "partial %d output must be 16-byte aligned", i);
    const int k = reverse ? n - 1 - i : i;
    a.o[k] = o_parts[i];
    a.lse[k] = lse_parts[i];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // The 32-rows-per-warp form needs enough rows to fill the GPU; a small merge
  // (the decode step's: slots x heads rows) takes one warp per row instead —
  // bitwise the same fold (128 rows: ~10 us -> ~3 us).
  if (head_dim == 128 && n >= 2 && n <= 8 && rows >= 148 * 8 * 32) {
    const int64_t warps = (rows + 31) / 32;
    const unsigned blocks = static_cast<unsigned>((warps + 7) / 8);
    switch (n) {
      case 2: merge_rows32_kernel<2><<<blocks, 256, 0, st>>>(a, rows, o_out, lse_out); break;
      case 3: merge_rows32_kernel<3><<<blocks, 256, 0, st>>>(a, rows, o_out, lse_out); break;
      case 4: merge_rows32_kernel<4><<<blocks, 256, 0, st>>>(a, rows, o_out, lse_out); break;
      case 5: merge_rows32_kernel<5><<<blocks, 256, 0, st>>>(a, rows, o_out, lse_out); break;
      case 6: merge_rows32_kernel<6><<<blocks, 256, 0, st>>>(a, rows, o_out, lse_out); break;
      case 7: merge_rows32_kernel<7><<<blocks, 256, 0, st>>>(a, rows, o_out, lse_out); break;
      default: merge_rows32_kernel<8><<<blocks, 256, 0, st>>>(a, rows, o_out, lse_out); break;
    }
  } else {
    const int64_t threads = rows * 32;
    const unsigned blocks = static_cast<unsigned>((threads + 255) / 256);
    merge_kernel<<<blocks, 256, 0, st>>>(a, n, rows, head_dim / 4, o_out, lse_out);
  }
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_gather_rows(void* dst, const void* src, const int64_t* idx, int64_t n_rows,
                    int64_t row_bytes, void* stream) {
  RCP_CHECK_ARG(n_rows >= 0 && row_bytes > 0, "bad sizes");
  RCP_CHECK_ARG(row_bytes % 16 == 0, "row_bytes must be a multiple of 16");
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(dst) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(src) & 15) == 0,
                "dst/src must be 16-byte aligned");
  if (n_rows == 0) return RCP_OK;
  const int64_t vpr = row_bytes / 16;
  gather_rows_kernel<<<grid_for(n_rows * 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint4*>(dst), static_cast<const uint4*>(src), idx, n_rows, vpr);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_shard_gather(void* dst, const void* const* src_rows, const int64_t* new_len,
                     const int64_t* cached_len, const int64_t* seq_id, int32_t n_seqs,
                     int32_t n_ranks, int32_t rank, int64_t row_bytes, int32_t* pos_out,
                     int32_t* seq_out, int32_t is_key, void* stream) {
  RCP_CHECK_ARG(n_ranks >= 1, "n_ranks must be >= 1");
  RCP_CHECK_ARG(rank >= 0 && rank < n_ranks, "rank %d out of range for %d ranks", rank, n_ranks);
  RCP_CHECK_ARG(n_seqs >= 1, "cannot plan an empty sequence list");
  RCP_CHECK_ARG(n_seqs <= kMaxShardSeqs, "at most %d sequences per gather", kMaxShardSeqs);
  RCP_CHECK_ARG(row_bytes > 0 && row_bytes % 16 == 0, "row_bytes must be a positive multiple of 16");
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(dst) & 15) == 0, "dst must be 16-byte aligned");
  ShardArgs a;
  memset(&a, 0, sizeof(a));
  int64_t slot = 0;
  for (int i = 0; i < n_seqs; ++i) {
    RCP_CHECK_ARG(new_len[i] >= 1, "sequence %lld has no new tokens", (long long)seq_id[i]);
    RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(src_rows[i]) & 15) == 0,
                  "source of sequence %d must be 16-byte aligned", i);
    RCP_CHECK_ARG(cached_len[i] + new_len[i] <= INT32_MAX, "positions exceed int32");
    a.src[i] = static_cast<const uint4*>(src_rows[i]);
    a.chunk[i] = (new_len[i] + 2 * n_ranks - 1) / (2 * n_ranks);
    a.new_len[i] = new_len[i];
    a.cached[i] = cached_len[i];
    a.seq_id[i] = seq_id[i];
    a.slot_begin[i] = slot;
    slot += 2 * a.chunk[i];
  }
  a.slot_begin[n_seqs] = slot;
  const int64_t vpr = row_bytes / 16;
  shard_gather_kernel<<<grid_for(slot * 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      a, n_seqs, n_ranks, rank, vpr, static_cast<uint4*>(dst), pos_out, seq_out, is_key);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_shard_scatter(void* const* dst_rows, const void* src, const int64_t* new_len, int32_t n_seqs,
                      int32_t n_ranks, int32_t rank, int64_t row_bytes, void* stream) {
  RCP_CHECK_ARG(n_ranks >= 1, "n_ranks must be >= 1");
  RCP_CHECK_ARG(rank >= 0 && rank < n_ranks, "rank %d out of range for %d ranks", rank, n_ranks);
  RCP_CHECK_ARG(n_seqs >= 1, "cannot plan an empty sequence list");
  RCP_CHECK_ARG(n_seqs <= kMaxShardSeqs, "at most %d sequences per scatter", kMaxShardSeqs);
  RCP_CHECK_ARG(row_bytes > 0 && row_bytes % 16 == 0, "row_bytes must be a positive multiple of 16");
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(src) & 15) == 0, "src must be 16-byte aligned");
  ShardArgs a;
  memset(&a, 0, sizeof(a));
  int64_t slot = 0;
  for (int i = 0; i < n_seqs; ++i) {
    RCP_CHECK_ARG(new_len[i] >= 1, "sequence %d has no new tokens", i);
    RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(dst_rows[i]) & 15) == 0,
                  "destination of sequence %d must be 16-byte aligned", i);
    a.src[i] = static_cast<const uint4*>(dst_rows[i]);
    a.chunk[i] = (new_len[i] + 2 * n_ranks - 1) / (2 * n_ranks);
    a.new_len[i] = new_len[i];
    a.slot_begin[i] = slot;
    slot += 2 * a.chunk[i];
  }
  a.slot_begin[n_seqs] = slot;
  const int64_t vpr = row_bytes / 16;
  shard_scatter_kernel<<<grid_for(slot * 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      a, n_seqs, n_ranks, rank, vpr, static_cast<const uint4*>(src));
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_cast_f32_bf16(void* dst, const float* src, int64_t n, void* stream) {
  RCP_CHECK_ARG(n >= 0 && n % 4 == 0, "n must be a non-negative multiple of 4");
  if (n == 0) return RCP_OK;
  RCP_CHECK_ARG(dst && src, "null pointer");
  RCP_CHECK_ARG(((reinterpret_cast<uintptr_t>(src) & 15) | (reinterpret_cast<uintptr_t>(dst) & 7)) == 0,
                "src must be 16-byte and dst 8-byte aligned");
  cast_f32_bf16_kernel<<<grid_for(n / 4, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(src), static_cast<uint2*>(dst), n / 4);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_p2p_epoch_advance(uint64_t* epoch, void* stream) {
  RCP_CHECK_ARG(epoch, "null epoch");
  p2p_epoch_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<unsigned long long*>(epoch));
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_p2p_put(void* const* dst, int32_t n, const void* src, size_t bytes, uint64_t* const* flag_dst,
                uint64_t* epoch, uint32_t* counter, void* stream) {
  RCP_CHECK_ARG(dst && src && n >= 1 && bytes % 16 == 0, "bad p2p put (bytes %% 16 == 0, n >= 1)");
  RCP_CHECK_ARG((reinterpret_cast<uintptr_t>(src) & 15) == 0, "src must be 16-byte aligned");
  RCP_CHECK_ARG(!flag_dst || (epoch && counter), "a signalling put needs the epoch and a counter");
  const int64_t n16 = static_cast<int64_t>(bytes / 16);
  RCP_CHECK_ARG(n16 > 0 || !flag_dst, "a signalling put needs data");
  if (n16 == 0) return RCP_OK;
  const int64_t blocks = (n16 + 255) / 256;
  p2p_put_kernel<<<static_cast<unsigned>(blocks < 296 ? blocks : 296), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dst, n, static_cast<const uint4*>(src), n16, reinterpret_cast<unsigned long long* const*>(flag_dst),
      reinterpret_cast<unsigned long long*>(epoch), counter);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_p2p_signal(uint64_t* const* flag_dst, int32_t n, const uint64_t* epoch, void* stream) {
  RCP_CHECK_ARG(flag_dst && epoch && n >= 1, "bad p2p signal");
  p2p_signal_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long* const*>(flag_dst), n, reinterpret_cast<const unsigned long long*>(epoch));
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_p2p_wait(const uint64_t* flags, int32_t n, const uint64_t* epoch, int32_t* timed_out, void* stream) {
  RCP_CHECK_ARG(flags && epoch && timed_out && n >= 1, "bad p2p wait");
  p2p_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const unsigned long long*>(flags), n, reinterpret_cast<const unsigned long long*>(epoch),
      timed_out);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_debug_stamp(uint64_t* slots, uint64_t* counter, int32_t n_slots, void* stream) {
  RCP_CHECK_ARG(slots && counter && n_slots >= 1, "bad stamp buffer");
  debug_stamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long*>(slots), reinterpret_cast<unsigned long long*>(counter), n_slots);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

int rcp_step_select(int64_t* dst, const int64_t* table, int64_t row_elems, int64_t* counter, int64_t n_rows,
                    void* stream) {
  RCP_CHECK_ARG(dst && table && counter, "null pointer");
  RCP_CHECK_ARG(row_elems >= 1 && n_rows >= 1, "bad sizes");
  step_select_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, table, row_elems, counter, n_rows);
  RCP_CUDA(cudaGetLastError());
  return RCP_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ peer memory (CUDA IPC)
extern "C" int rcp_ipc_alloc(size_t bytes, void** dev_ptr_out, void* handle_out) {
  RCP_CHECK_ARG(bytes > 0 && dev_ptr_out != nullptr && handle_out != nullptr, "bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == RCP_IPC_HANDLE_BYTES, "IPC handle size");
  RCP_CUDA(cudaMalloc(dev_ptr_out, bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, *dev_ptr_out);
  if (e != cudaSuccess) {
    cudaFree(*dev_ptr_out);
    *dev_ptr_out = nullptr;
    set_error("cudaIpcGetMemHandle failed: %s", cudaGetErrorString(e));
    return RCP_ERR_CUDA;
  }
  memcpy(handle_out, &h, sizeof(h));
  return RCP_OK;
}

extern "C" int rcp_ipc_free(void* dev_ptr) {
  RCP_CHECK_ARG(dev_ptr != nullptr, "null pointer");
  RCP_CUDA(cudaFree(dev_ptr));
  return RCP_OK;
}

extern "C" int rcp_ipc_open(const void* handle, void** dev_ptr_out) {
  RCP_CHECK_ARG(handle != nullptr && dev_ptr_out != nullptr, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  RCP_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return RCP_OK;
}

extern "C" int rcp_ipc_close(void* dev_ptr) {
  RCP_CHECK_ARG(dev_ptr != nullptr, "null pointer");
  RCP_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return RCP_OK;
}


// ------------------------------------------------------------------ growable device arenas (CUDA VMM)
// A KV-cache arena reserves one large virtual address range and maps physical
// memory into it in granularity-sized chunks as it grows: growth never copies
// the cached rows and never needs old + new arenas at once, and the arena's
// base pointer (baked into CUDA graphs and tensor maps) never changes.
namespace {
template <typename F>
F driver_fn(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(f);
}
CUmemAllocationProp vmm_prop(int device) {
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  return prop;
}
}  // namespace

#define RCP_CU(call)                                                        \
  do {                                                                      \
    CUresult r_ = (call);                                                   \
    if (r_ != CUDA_SUCCESS) {                                               \
      ::rcp::set_error("%s failed: CUresult %d", #call, static_cast<int>(r_)); \
      return RCP_ERR_CUDA;                                                  \
    }                                                                       \
  } while (0)

extern "C" int rcp_vmm_granularity(int device, size_t* bytes_out) {
  RCP_CHECK_ARG(bytes_out != nullptr, "null pointer");
  auto gran = driver_fn<PFN_cuMemGetAllocationGranularity_v10020>("cuMemGetAllocationGranularity");
  RCP_CHECK_ARG(gran != nullptr, "CUDA VMM entry points unavailable");
  CUmemAllocationProp prop = vmm_prop(device);
  RCP_CU(gran(bytes_out, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  return RCP_OK;
}

extern "C" int rcp_vmm_reserve(size_t bytes, void** base_out) {
  RCP_CHECK_ARG(base_out != nullptr && bytes > 0, "bad arguments");
  auto reserve = driver_fn<PFN_cuMemAddressReserve_v10020>("cuMemAddressReserve");
  RCP_CHECK_ARG(reserve != nullptr, "CUDA VMM entry points unavailable");
  CUdeviceptr p = 0;
  RCP_CU(reserve(&p, bytes, 0, 0, 0));
  *base_out = reinterpret_cast<void*>(p);
  return RCP_OK;
}

// Map `bytes` (a multiple of the granularity) of new physical memory at base + offset.
extern "C" int rcp_vmm_map(void* base, size_t offset, size_t bytes, int device, uint64_t* handle_out) {
  RCP_CHECK_ARG(base != nullptr && bytes > 0 && handle_out != nullptr, "bad arguments");
  auto create = driver_fn<PFN_cuMemCreate_v10020>("cuMemCreate");
  auto map = driver_fn<PFN_cuMemMap_v10020>("cuMemMap");
  auto access = driver_fn<PFN_cuMemSetAccess_v10020>("cuMemSetAccess");
  auto release = driver_fn<PFN_cuMemRelease_v10020>("cuMemRelease");
  auto unmap = driver_fn<PFN_cuMemUnmap_v10020>("cuMemUnmap");
  RCP_CHECK_ARG(create && map && access && release && unmap, "CUDA VMM entry points unavailable");
  CUmemAllocationProp prop = vmm_prop(device);
  CUmemGenericAllocationHandle h;
  RCP_CU(create(&h, bytes, &prop, 0));
  const CUdeviceptr at = reinterpret_cast<CUdeviceptr>(base) + offset;
  CUresult r = map(at, bytes, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    release(h);
    set_error("cuMemMap failed: CUresult %d", static_cast<int>(r));
    return RCP_ERR_CUDA;
  }
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = access(at, bytes, &acc, 1);
  if (r != CUDA_SUCCESS) {
    unmap(at, bytes);
    release(h);
    set_error("cuMemSetAccess failed: CUresult %d", static_cast<int>(r));
    return RCP_ERR_CUDA;
  }
  *handle_out = static_cast<uint64_t>(h);
  return RCP_OK;
}

extern "C" int rcp_vmm_unmap(void* base, size_t offset, size_t bytes, uint64_t handle) {
  auto unmap = driver_fn<PFN_cuMemUnmap_v10020>("cuMemUnmap");
  auto release = driver_fn<PFN_cuMemRelease_v10020>("cuMemRelease");
  RCP_CHECK_ARG(unmap && release, "CUDA VMM entry points unavailable");
  RCP_CU(unmap(reinterpret_cast<CUdeviceptr>(base) + offset, bytes));
  RCP_CU(release(static_cast<CUmemGenericAllocationHandle>(handle)));
  return RCP_OK;
}

extern "C" int rcp_vmm_free(void* base, size_t bytes) {
  auto free_fn = driver_fn<PFN_cuMemAddressFree_v10020>("cuMemAddressFree");
  RCP_CHECK_ARG(free_fn != nullptr, "CUDA VMM entry points unavailable");
  RCP_CU(free_fn(reinterpret_cast<CUdeviceptr>(base), bytes));
  return RCP_OK;
}
