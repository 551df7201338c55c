// Shared host/device pieces of the ringcp-b200 C ABI: error reporting, the
// fp32 LSE merge used by both the fused attention epilogue and the merge
// kernel (so pass-KV and pass-Q fold bit-identically), and tile summaries.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ringcp_b200.h"

namespace rcp {

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);

#define RCP_CHECK_ARG(cond, ...)      \
  do {                                \
    if (!(cond)) {                    \
      ::rcp::set_error(__VA_ARGS__);  \
      return RCP_ERR_INVALID;         \
    }                                 \
  } while (0)

#define RCP_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ::rcp::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                       __LINE__);                                                   \
      return RCP_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

// Negative-control hooks for the parity harness (tests/test_gpu_negative_controls.py):
// RCP_FAULT=drop_block | mask_diag | reverse_merge makes the library WRONG on
// purpose (read once per process; never set in production).
enum : int { kFaultNone = 0, kFaultDropBlock = 1, kFaultMaskDiag = 2, kFaultReverseMerge = 4 };
int rcp_fault_flags();

// ------------------------------------------------------------------ merge math
// One pairwise LSE merge step, the fp32 restatement of
// ringcp.attention._merge_pair (attention.py:299-316).  Written with explicit
// round-to-nearest intrinsics so every kernel that folds partials produces the
// same bits regardless of FMA contraction.
struct MergeW {
  float lse, wa, wb;
};
__device__ __forceinline__ MergeW merge_weights(float la, float lb) {
  const float m = fmaxf(la, lb);
  MergeW r;
  if (m == -INFINITY) {
    r.lse = -INFINITY;
    r.wa = 0.f;
    r.wb = 0.f;
    return r;
  }
  const float tot = __fadd_rn(expf(__fsub_rn(la, m)), expf(__fsub_rn(lb, m)));
  r.lse = __fadd_rn(m, logf(tot));
  r.wa = (la == -INFINITY) ? 0.f : expf(__fsub_rn(la, r.lse));
  r.wb = (lb == -INFINITY) ? 0.f : expf(__fsub_rn(lb, r.lse));
  return r;
}
__device__ __forceinline__ float merge_val(float a, float b, const MergeW& w) {
  return __fadd_rn(__fmul_rn(a, w.wa), __fmul_rn(b, w.wb));
}

// ------------------------------------------------------------------ P2P completion signal
// Called by EVERY thread of every block of a grid after the block's peer
// stores: the last block to arrive (device counter, re-armed here) publishes
// the step epoch — first advanced by one if `advance` — into each of the n
// peers' flag slots (release, system scope).  Fuses the separate signal kernel
// of the decode step's p2p transport into the kernel that did the stores.
__device__ __forceinline__ void p2p_last_block_signal(unsigned* counter, unsigned long long* const* flag_dst,
                                                      int n, unsigned long long* epoch, bool advance) {
  __shared__ int s_last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y * gridDim.z - 1 ? 1 : 0;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    *counter = 0u;
    unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(epoch);
    if (advance) {
      e += 1ull;
      *reinterpret_cast<volatile unsigned long long*>(epoch) = e;
    }
    __threadfence_system();
    for (int p = 0; p < n; ++p)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag_dst[p]), "l"(e) : "memory");
  }
}

// ------------------------------------------------------------------ tile summaries
// Per 64- or 128-token tile of a block: min/max position and sequence id over the
// VALID rows, number of valid rows, and whether all rows are valid and of
// one sequence.  Used to classify (query tile, key tile) pairs as empty / full
// / partial so masked work is skipped and unmasked tiles skip the mask.
struct __align__(32) TileSum {
  int pmin, pmax, smin, smax, nvalid, uniform, pad0, pad1;
};

enum : int { kTileEmpty = 0, kTilePartial = 1, kTileFull = 2 };

__host__ __device__ __forceinline__ int classify_tile(const TileSum& q, const TileSum& k) {
  if (q.nvalid == 0 || k.nvalid == 0) return kTileEmpty;
  if (k.pmin > q.pmax) return kTileEmpty;
  if (k.smax < q.smin || k.smin > q.smax) return kTileEmpty;
  if (q.uniform && k.uniform && q.smin == k.smin && k.pmax <= q.pmin) return kTileFull;
  return kTilePartial;
}

// Launch the summary kernel for one metadata array (n rows, `rows`-row tiles, rows in {64, 128}).
int launch_tile_summary(const int32_t* pos, const int32_t* seq, int64_t n, int32_t pad_seq,
                        int rows, TileSum* out, cudaStream_t stream);

}  // namespace rcp
