/* ringcp_b200 — C ABI of the B200-native context-parallel attention engine.
 *
 * Drop-in boundary for the reference package `ringcp` (arXiv 2411.01783,
 * /root/reference/pkg/src/ringcp).  The reference is a Python API; every entry
 * point below is what that API's hot path calls on a B200, one call per
 * reference operation (file:line of the operation it replaces is given).
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless stated; nothing here allocates or
 *     frees caller memory.  Every call is asynchronous on `stream`
 *     (a cudaStream_t passed as void*), stream-ordered, and returns
 *     RCP_OK (0) or a negative error class; rcp_last_error() returns the
 *     thread-local message of the last failure.
 *   - Token-major layouts, bf16 inputs:  Q [Tq, Hq, 128], K/V [Tk, Hkv, 128]
 *     with an explicit row stride (elements between consecutive tokens,
 *     multiple of 8).  Outputs are fp32: O [Tq, Hq, 128] (contiguous) and
 *     LSE [Tq, Hq] (natural log, -inf for rows that admitted no key).
 *   - Per-token metadata is int32 and already FOLDED with the validity bit:
 *       valid query  : pos >= 0,  seq = its sequence id
 *       padding query: pos = -1,  seq = RCP_SEQ_PAD_Q   (INT32_MIN)
 *       valid key    : pos >= 0,  seq = its sequence id
 *       padding key  : pos = INT32_MAX, seq = RCP_SEQ_PAD_K (INT32_MIN + 1)
 *     so key j is admitted for query i iff seq_k[j] == seq_q[i] and
 *     pos_k[j] <= pos_q[i]  (ringcp.attention._admissible, attention.py:199-206).
 */
#ifndef RINGCP_B200_H
#define RINGCP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCP_OK 0
#define RCP_ERR_INVALID (-1)   /* bad argument: shape/alignment/geometry      */
#define RCP_ERR_CUDA (-2)      /* CUDA runtime/driver failure                 */
#define RCP_ERR_UNSUPPORTED (-3)

#define RCP_SEQ_PAD_Q (-2147483647 - 1)
#define RCP_SEQ_PAD_K (-2147483647)
#define RCP_POS_PAD_K 2147483647

#define RCP_MODE_OVERWRITE 0  /* O, LSE <- attention of this KV block                 */
#define RCP_MODE_MERGE 1      /* (O, LSE) <- merge((O, LSE), attention of this block) */

const char* rcp_last_error(void);
const char* rcp_version(void);
/* The attention kernel form this library runs: 4 (the product kernel); the
 * A/B build (_ringcp_b200_ab.so) also carries the measured alternatives
 * 12-17, selected by the RCP_ATTN_VERSION environment variable. */
int rcp_attn_version(void);

/* Workspace bytes rcp_attn_fwd needs for a (Tq, Tk) call (tile summaries). */
size_t rcp_attn_workspace_bytes(int64_t tq, int64_t tk);

/* Causal-by-position GQA attention of one query block against one KV block,
 * with per-row LSE.  Replaces ringcp.attention.gqa_attention
 * (attention.py:230-282).  head_dim must be 128; hq % hkv == 0; query head h
 * reads kv head h / (hq / hkv) (GqaConfig.query_to_kv_head, attention.py:64-66).
 * mode RCP_MODE_MERGE folds the result into (o, lse) with the pairwise merge of
 * ringcp.attention._merge_pair (attention.py:299-316) — the running merge of
 * the pass-KV ring (Alg. 2).  Padding key rows must hold
 * finite data (the Python layer zeroes them). */
int rcp_attn_fwd(const void* q, int64_t q_row_stride, const void* k, int64_t k_row_stride,
                 const void* v, int64_t v_row_stride, const int32_t* q_pos,
                 const int32_t* q_seq, const int32_t* k_pos, const int32_t* k_seq, int64_t tq,
                 int64_t tk, int32_t hq, int32_t hkv, int32_t head_dim, float scale, float* o,
                 float* lse, int32_t mode, void* workspace, size_t workspace_bytes,
                 void* stream);

/* rcp_attn_fwd with Q and K in e4m3 (OCP; value = scale * e4m3, one fp32
 * scale per query head in q_scale[hq] and per KV head in k_scale[hkv], device
 * arrays) and S = Q K^T on the tensor cores' 8-bit path (tcgen05 kind::f8f6f4);
 * V bf16, P bf16, outputs as rcp_attn_fwd.  Row strides in elements (= bytes
 * for q8 / k8, multiples of 16).  Opt-in FP8 mode: the
 * result is rcp_attn_fwd's on the dequantised Q / K. */
int rcp_attn_fwd_qk8(const void* q8, int64_t q_row_stride, const void* k8, int64_t k_row_stride, const void* v,
                     int64_t v_row_stride, const int32_t* q_pos, const int32_t* q_seq, const int32_t* k_pos,
                     const int32_t* k_seq, int64_t tq, int64_t tk, int32_t hq, int32_t hkv, int32_t head_dim,
                     float scale, const float* q_scale, const float* k_scale, float* o, float* lse, int32_t mode,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Left-fold merge of n partials (ascending list order), replacing
 * ringcp.attention.merge_attention (attention.py:319-334).  o_parts / lse_parts
 * are HOST arrays of n DEVICE pointers, each O [rows, head_dim] fp32 and LSE
 * [rows] fp32 (rows = Tq * Hq, head_dim % 4 == 0).  Output may alias part 0. */
int rcp_merge_attn(const float* const* o_parts, const float* const* lse_parts, int32_t n,
                   int64_t rows, int32_t head_dim, float* o_out, float* lse_out, void* stream);

/* Fill O = 0 and LSE = -inf (the result of attending to no key). */
int rcp_fill_empty(float* o, float* lse, int64_t rows, int32_t head_dim, void* stream);

/* Load-balanced shard gather: the device half of
 * ringcp.sharding.materialize_rank_block (sharding.py:211-240).
 * For each of n_seqs sequences (HOST arrays, one entry per sequence):
 *   src_rows[i]   device pointer to sequence i's dense new-token rows
 *   new_len[i], cached_len[i], seq_id[i]
 * writes dst (n_seqs * 2 * chunk_len_i slots, row_bytes each) with rank
 * `rank`'s chunks (C_rank, C_{2N-1-rank}), zero padding, and (optionally, if
 * non-null) the folded metadata pos/seq (query or key sentinels per
 * `is_key`) — positions = cached_len + local index (sharding.py:235). */
int rcp_shard_gather(void* dst, const void* const* src_rows, const int64_t* new_len,
                     const int64_t* cached_len, const int64_t* seq_id, int32_t n_seqs,
                     int32_t n_ranks, int32_t rank, int64_t row_bytes, int32_t* pos_out,
                     int32_t* seq_out, int32_t is_key, void* stream);

/* Inverse of rcp_shard_gather (the device scatter of the load-balanced
 * sharding, sharding.py:105-115, 211-240 read backwards): every VALID slot of
 * rank `rank`'s block `src` (slot order, row_bytes per slot) is written to row
 * `local` of sequence i's token-ordered array dst_rows[i] (HOST array of n_seqs
 * device pointers); padding slots are dropped.  Run for every rank, the
 * scatters tile each sequence exactly once. */
int rcp_shard_scatter(void* const* dst_rows, const void* src, const int64_t* new_len, int32_t n_seqs,
                      int32_t n_ranks, int32_t rank, int64_t row_bytes, void* stream);

/* Row gather dst[i] = src[idx[i]] (idx < 0 -> zero row), idx int64 on device. */
int rcp_gather_rows(void* dst, const void* src, const int64_t* idx, int64_t n_rows,
                    int64_t row_bytes, void* stream);

/* Fold int64 positions / seq ids / bool valid into the int32 kernel metadata
 * described above.  is_key selects the key sentinels. */
int rcp_fold_meta(const int64_t* pos, const int64_t* seq, const uint8_t* valid, int64_t n,
                  int32_t is_key, int32_t* pos_out, int32_t* seq_out, void* stream);

/* Split-KV decode attention: one query token per sequence against the rank's
 * cached KV shard of that sequence (ring pass-Q decode, Alg. 4,
 * PAPER.md:353-370).  q [B, hq, 128] bf16; for sequence b the keys are rows
 * [kv_start[b], kv_start[b] + kv_len[b]) of the KV arena k/v ([kv_rows, hkv,
 * 128] bf16, row stride kv_row_stride), all causally visible (the cache holds
 * only the past and the token itself) and of the same sequence.  kv_start /
 * kv_len are device int64 arrays; max_kv_len bounds kv_len.  Any hq / hkv (16
 * query heads per CTA; larger groups take several CTAs per KV head).
 * Writes o [B, hq, 128] fp32, lse [B, hq] fp32 (-inf when kv_len == 0).
 * workspace: rcp_decode_workspace_bytes(B, hq, max_kv_len). */
size_t rcp_decode_workspace_bytes(int64_t batch, int32_t hq, int64_t max_kv_len);
int rcp_decode_attn(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                    int64_t kv_rows, const int64_t* kv_start, const int64_t* kv_len, int64_t batch,
                    int64_t max_kv_len, int32_t hq, int32_t hkv, int32_t head_dim, float scale,
                    float* o, float* lse, void* workspace, size_t workspace_bytes, void* stream);

/* FP8 KV cache (PAPER.md:393 — beyond the SPEC's bf16
 * contract, an opt-in RankKvCache(kv_dtype="e4m3") mode).  The arena holds
 * K/V as OCP e4m3 bytes ([kv_rows, hkv, 128], row stride in elements = bytes)
 * with one fp32 scale per KV head: value = scale[h] * e4m3.  Same contract as
 * rcp_decode_attn otherwise (q bf16; o / lse fp32; same workspace size); the
 * kernel reads half the bytes per key.  Parity: against the decode oracle on
 * the dequantised K/V, at the bf16 decode tolerance. */
int rcp_decode_attn_fp8(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                        int64_t kv_rows, const int64_t* kv_start, const int64_t* kv_len, int64_t batch,
                        int64_t max_kv_len, int32_t hq, int32_t hkv, int32_t head_dim, float scale,
                        const float* k_scale, const float* v_scale, float* o, float* lse, void* workspace,
                        size_t workspace_bytes, void* stream);

/* rcp_decode_attn / rcp_decode_attn_fp8 with the combined rows ROUTED: row
 * block d of the batch (batch / n_dst queries each) goes to o_dst[d] / lse_dst[d]
 * (DEVICE arrays of n_dst base pointers, e.g. the owners' CUDA-IPC receive
 * buffers) at query row dst_row_offset + (b % (batch / n_dst)) — the All2All
 * of Alg. 4 done by the combine kernel's own stores over NVLink.  k_scale /
 * v_scale NULL selects bf16 K/V, non-NULL e4m3.  flag_dst non-NULL (DEVICE
 * array of n_dst flag slots): the combine's last CTA also publishes *epoch
 * there once every row is stored (as rcp_p2p_signal; counter: a device u32,
 * zero before the first call, re-armed by the kernel). */
int rcp_decode_attn_routed(const void* q, const void* k, const void* v, int64_t kv_row_stride,
                           int64_t kv_rows, const int64_t* kv_start, const int64_t* kv_len, int64_t batch,
                           int64_t max_kv_len, int32_t hq, int32_t hkv, int32_t head_dim, float scale,
                           const float* k_scale, const float* v_scale, float* const* o_dst,
                           float* const* lse_dst, int32_t n_dst, int64_t dst_row_offset,
                           uint64_t* const* flag_dst, uint64_t* epoch, uint32_t* counter, void* workspace,
                           size_t workspace_bytes, void* stream);

/* bf16 rows -> e4m3 rows: row j of src ([n_rows, hkv * head_dim], row stride
 * in elements) is written to dst row dst_rows[j] (device int64; NULL = row j),
 * each element satfinite_rn(x * (1 / scale[head])) in IEEE fp32 (the
 * reciprocal once per head; bit-exact with
 * oracle/ringcp_oracle.py::quantize_e4m3). */
int rcp_kv_quantize_e4m3(void* dst, int64_t dst_row_stride, const int64_t* dst_rows, const void* src,
                         int64_t src_row_stride, int64_t n_rows, int32_t hkv, int32_t head_dim,
                         const float* scale, void* stream);
/* e4m3 rows -> bf16 rows (x = scale[head] * e4m3 in fp32, rounded to bf16):
 * snapshots and prefill messages built from an e4m3 cache. */
int rcp_kv_dequantize_e4m3(void* dst, int64_t dst_row_stride, const void* src, int64_t src_row_stride,
                           int64_t n_rows, int32_t hkv, int32_t head_dim, const float* scale, void* stream);
/* One decode step's cache appends (GraphedDecode): slot j < slots of the
 * step's new tokens k_in / v_in ([slots, hkv, head_dim] bf16) goes to arena row
 * meta[j] of the DEVICE step metadata (int64); its position / sequence id
 * meta[pos_off + j] / meta[seq_off + j] go to pos_arena / seq_arena (int32).
 * K/V rows are copied (bf16 arenas, k_scale = v_scale = NULL) or quantised as
 * rcp_kv_quantize_e4m3 (e4m3 arenas).  kv_row_stride in elements. */
int rcp_decode_append(const int64_t* meta, int32_t slots, int64_t pos_off, int64_t seq_off, const void* k_in,
                      const void* v_in, void* k_arena, void* v_arena, int64_t kv_row_stride, int32_t hkv,
                      int32_t head_dim, int32_t* pos_arena, int32_t* seq_arena, const float* k_scale,
                      const float* v_scale, void* stream);

/* Per-KV-head scale from bf16 rows: scale[h] = max(absmax_h, 2^-24) / 448
 * (fp32 IEEE division) rounded up to a power of two (then e4m3 * scale is
 * exact in bf16: prefill and decode read the same values).  workspace: hkv * 4 bytes of device memory. */
int rcp_kv_calibrate_e4m3(const void* src, int64_t src_row_stride, int64_t n_rows, int32_t hkv,
                          int32_t head_dim, float* scale, void* workspace, void* stream);

/* fp32 -> bf16 (round to nearest even) of n values (n % 4 == 0): the final
 * attention output in the model dtype, so the host-buffer path copies half the
 * bytes back (RingAttention.pass_kv_prefill_host with bf16 host outputs). */
int rcp_cast_f32_bf16(void* dst, const float* src, int64_t n, void* stream);

/* Device-side transport over CUDA-IPC peer memory (the decode step's Q
 * all-gather and partial All2All without NCCL, graph-capturable):
 *   rcp_p2p_epoch_advance: *epoch += 1 (once per step, every rank);
 *   rcp_p2p_put:    copy `bytes` (multiple of 16) of src to each of the n
 *                   destinations dst[0..n) (DEVICE array of pointers); with
 *                   flag_dst non-NULL its last block also advances *epoch
 *                   and publishes it to flag_dst[0..n) (counter: device u32,
 *                   zero initially, re-armed by the kernel);
 *   rcp_p2p_signal: publish *epoch to each flag_dst[p] (DEVICE array; this
 *                   rank's flag slot in peer p's buffer), release, system scope;
 *   rcp_p2p_wait:   wait until flags[0..n) (this rank's own slots) all reach
 *                   *epoch, acquire; after ~9 s sets *timed_out = 1 and traps
 *                   (a CUDA error at the caller's next sync) instead of hanging
 *                   or returning a wrong step. */
int rcp_p2p_epoch_advance(uint64_t* epoch, void* stream);
int rcp_p2p_put(void* const* dst, int32_t n, const void* src, size_t bytes, uint64_t* const* flag_dst,
                uint64_t* epoch, uint32_t* counter, void* stream);
int rcp_p2p_signal(uint64_t* const* flag_dst, int32_t n, const uint64_t* epoch, void* stream);
int rcp_p2p_wait(const uint64_t* flags, int32_t n, const uint64_t* epoch, int32_t* timed_out, void* stream);

/* Debug timeline: one 1-thread launch writing %globaltimer (ns) to
 * slots[*counter % n_slots] and advancing the device counter (stream-ordered
 * stamps between launches, e.g. inside a captured decode step). */
int rcp_debug_stamp(uint64_t* slots, uint64_t* counter, int32_t n_slots, void* stream);

/* Decode-graph helper: copy row *counter of the device int64 table
 * [n_rows, row_elems] to dst, then increment *counter (device int64, clamped
 * at n_rows - 1).  GraphedDecode precomputes the per-step metadata of all of
 * a graph's future steps (cache rows to append to, per-query KV segments,
 * positions) and replays without any host->device upload per step. */
int rcp_step_select(int64_t* dst, const int64_t* table, int64_t row_elems, int64_t* counter, int64_t n_rows,
                    void* stream);

/* Growable device arenas for the per-rank KV cache (RankKvCache):
 * reserve a virtual address range once, then map physical memory into it in
 * granularity-sized chunks as the cache grows — no copy of the cached rows and
 * no old + new arena at once; the base pointer never moves (CUDA graphs and
 * tensor maps stay valid).  rcp_vmm_map returns an opaque handle for
 * rcp_vmm_unmap; rcp_vmm_free releases the (fully unmapped) range. */
int rcp_vmm_granularity(int device, size_t* bytes_out);
int rcp_vmm_reserve(size_t bytes, void** base_out);
int rcp_vmm_map(void* base, size_t offset, size_t bytes, int device, uint64_t* handle_out);
int rcp_vmm_unmap(void* base, size_t offset, size_t bytes, uint64_t handle);
int rcp_vmm_free(void* base, size_t bytes);

/* Peer memory for the fused pass-Q All2All (Alg. 3's partial return,
 * SPEC.md:249-257): instead of an All2All after the ring, each ring step's
 * attention writes its partial O / LSE straight into the owning rank's
 * receive buffer over NVLink.  rcp_ipc_alloc makes a device allocation of
 * its own (cudaMalloc, so the exported handle covers exactly it) and returns
 * its RCP_IPC_HANDLE_BYTES opaque handle, exchanged by the host transport;
 * rcp_ipc_open maps a peer's allocation into the CURRENT device's address
 * space (peer access enabled lazily; no extra CUDA context on the peer);
 * rcp_ipc_close unmaps it and rcp_ipc_free releases an own allocation. */
#define RCP_IPC_HANDLE_BYTES 64
int rcp_ipc_alloc(size_t bytes, void** dev_ptr_out, void* handle_out);
int rcp_ipc_free(void* dev_ptr);
int rcp_ipc_open(const void* handle, void** dev_ptr_out);
int rcp_ipc_close(void* dev_ptr);

#ifdef __cplusplus
}
#endif
#endif /* RINGCP_B200_H */
