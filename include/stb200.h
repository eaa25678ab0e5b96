/*
 * stb200.h — C ABI of the B200-native tool-resident engine (libstb200.so).
 *
 * The reference (`/root/reference/pkg/src/spectool`) is a pure-Python
 * discrete-event engine with no FFI: every phase is a virtual-time charge
 * `sim.schedule(rate * tokens, continuation)`. Each entry point below is the
 * device work that replaces one of those charges; the comment on each names
 * the reference call site it stands in for. Plain pointers and sizes only:
 * device pointers are raw CUDA addresses (torch tensors' data_ptr()),
 * `stream` is a cudaStream_t passed as void*. All calls are stream-ordered,
 * allocate nothing on the hot path, and return 0 or a negative STB_E* code;
 * `stb_last_error()` holds the message for the calling thread.
 *
 * Layout: the KV pool owns, per layer, K and V pages
 * `[num_blocks][n_kv][block_size=16][d_head]` bf16; the block table is
 * `int32 [max_slots][max_blocks_per_slot]` on the device, mirrored on the host
 * where the deterministic LIFO allocator runs.
 */
#ifndef STB200_H
#define STB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STB_OK 0
#define STB_EINVAL (-1)
#define STB_ENOMEM (-2)
#define STB_ECUDA (-3)
#define STB_ECAPACITY (-4)

typedef struct stb_kv_pool stb_kv_pool;

/* ---- diagnostics ------------------------------------------------------- */
const char* stb_last_error(void);
int stb_version(void);
/* number of kernel launches issued through this library since load */
int64_t stb_launch_count(void);

/* ---- K1: paged KV pool, block allocator, block table --------------------
 * Replaces the reference's integer KV accounting: `seq.kv_tokens = ...`
 * (engine.py:259,285,313,335,366), the evict/reset (engine.py:382-384) and
 * the slot release (engine.py:385,397). The reference pool is unbounded
 * (SPEC.md:521); this one is sized in blocks and reports STB_ECAPACITY.   */
int stb_kv_pool_create(int device, int layers, int n_kv, int d_head, int block_size, int num_blocks,
                       int max_slots, int max_blocks_per_slot, stb_kv_pool** out);
int stb_kv_pool_destroy(stb_kv_pool* pool);
/* grow slot's block list to ceil(new_len / block_size) blocks (LIFO pops) */
int stb_kv_reserve(stb_kv_pool* pool, int slot, int new_len);
/* free blocks beyond ceil(new_len / block_size) (rollback / evict-to-prefix) */
int stb_kv_truncate(stb_kv_pool* pool, int slot, int new_len);
/* free every block of the slot (request finished / vanilla evict) */
int stb_kv_release(stb_kv_pool* pool, int slot);
int stb_kv_free_blocks(const stb_kv_pool* pool);
int stb_kv_slot_len(const stb_kv_pool* pool, int slot);
/* host copy of a slot's block ids; returns the count (or error) */
int stb_kv_slot_blocks(const stb_kv_pool* pool, int slot, int32_t* out, int cap);
/* upload block-table rows changed since the last sync (async on stream) */
int stb_kv_sync(stb_kv_pool* pool, void* stream);
/* device addresses: K/V base of a layer, the device block table and its row stride */
int stb_kv_layer_ptrs(const stb_kv_pool* pool, int layer, void** k_pages, void** v_pages);
int stb_kv_block_table(const stb_kv_pool* pool, int32_t** dev_table, int* row_stride);
/* K1 commit: scatter bf16 rows k,v [n][n_kv*d_head] (row stride ld elements)
 * into the pages of (slot_of[i], pos_of[i]); 16-byte vector stores. */
int stb_kv_commit(stb_kv_pool* pool, int layer, const void* k, const void* v, int64_t ld, const int32_t* slot_of,
                  const int32_t* pos_of, int n, void* stream);
/* K1 copy: duplicate whole blocks src[i] -> dst[i] in every layer (fork / COW) */
int stb_kv_copy_blocks(stb_kv_pool* pool, const int32_t* src, const int32_t* dst, int n, void* stream);

/* ---- fused QKV epilogue: RoPE on q/k + K1 commit of k/v -----------------
 * qkv fp32 [n][(n_q + 2 n_kv) d_head] from the QKV GEMM; writes q bf16
 * [n][n_q d_head] (rotated) and commits rotated k and v into the pool.
 * Rows < clear_rows of qkv are zeroed after they are read (so the next
 * stream-K GEMM into qkv can accumulate without a memset).               */
int stb_qkv_rope_commit(stb_kv_pool* pool, int layer, float* qkv, void* q_out, const int32_t* slot_of,
                        const int32_t* pos_of, int n, int n_q, float rope_theta, int clear_rows, void* stream);
/* Same, with Qwen3 qk-norm (config C3): each q and k head row is RMS-normalised over
 * d_head and scaled by q_norm / k_norm (bf16 [d_head]) before RoPE. The reference
 * has no decoder; this is part of the self-defined model of the
 * charges at engine.py:251,270,296,358. NULL norms = stb_qkv_rope_commit.       */
int stb_qkv_norm_rope_commit(stb_kv_pool* pool, int layer, float* qkv, void* q_out, const int32_t* slot_of,
                             const int32_t* pos_of, int n, int n_q, float rope_theta, const void* q_norm,
                             const void* k_norm, float eps, int clear_rows, void* stream);

/* Same, gpt-oss attention inputs (config C4): `bias` (fp32 [(n_q + 2 n_kv) d_head], or NULL) is
 * added to every q / k / v row before RoPE; `inv_freq` (device fp32 [d_head / 2], or NULL for
 * theta^(-2i/d)) are the rotary frequencies — the YaRN table for gpt-oss — and `rope_scale`
 * multiplies cos and sin (YaRN's attention factor; 1 = plain RoPE).                  */
int stb_qkv_rope_commit_ex(stb_kv_pool* pool, int layer, float* qkv, void* q_out, const int32_t* slot_of,
                           const int32_t* pos_of, int n, int n_q, float rope_theta, const float* inv_freq,
                           float rope_scale, const float* bias, int clear_rows, void* stream);

/* ---- K3: paged decode attention (one query per sequence) ----------------
 * Replaces the decode charges engine.py:270,276,302,317. q/out bf16
 * [B][n_q][d_head]; slots/ctx_lens int32 [B]; split-K over the context with
 * an in-kernel merge. `work` is a caller-owned scratch of at least
 * stb_attn_decode_workspace(B, n_q, n_kv, d_head) bytes for the calling device,
 * ZEROED ONCE by the caller (its tail holds the split-merge tickets, which every
 * launch leaves zero again); the call allocates nothing, so a CUDA graph captured
 * for any B stays valid as long as `work` does. The grid depends on B alone.
 * max_ctx (0 = unchecked) is validated against the block-table capacity.    */
int64_t stb_attn_decode_workspace(int B, int n_q, int n_kv, int d_head);
int stb_attn_decode(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                    const int32_t* ctx_lens, int B, int n_q, float scale, int max_ctx, void* work, void* stream);
/* Same, gpt-oss attention (config C4): `window` > 0 restricts each query to its last `window`
 * keys (sliding-window layers: key j is visible from query position p iff p - window < j <= p);
 * `sinks` (device fp32 [n_q], or NULL) adds exp(sink_h) to head h's softmax denominator (a
 * learned logit with no value row). window = 0 and sinks = NULL is stb_attn_decode.        */
int stb_attn_decode_ex(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                       const int32_t* ctx_lens, int B, int n_q, float scale, int max_ctx, int window,
                       const float* sinks, void* work, void* stream);
/* Same with multi-query entries (the verify pass of engine.py:296 riding in the decode launch):
 * entry b holds n_qs[b] (1 .. 16 / group) consecutive query rows of q / out starting at packed row
 * q_rows[b]; they are the last n_qs[b] positions of the entry's ctx_lens[b] keys and attend
 * causally (query i of the entry sees keys < ctx_lens[b] - (n_qs[b] - 1 - i)). A short run of n
 * queries is ceil(n * group / 16) entries with the same slot; a decode row is an entry with
 * n_qs = 1. Plain attention only (no window, no sinks).                                     */
int stb_attn_decode_mq(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                       const int32_t* ctx_lens, const int32_t* q_rows, const int32_t* n_qs, int B, int n_q,
                       float scale, int max_ctx, void* work, void* stream);
/* Same (q_rows / n_qs may both be NULL: one query per entry), with the work partition shared
 * across a step's layers: plan_mode 0 computes it in the launch, 1 also stores it in the
 * workspace, 2 loads the one stored by an earlier launch on the same stream with the same
 * (B, slots, ctx_lens, q_rows, n_qs) — every layer of a decode step after the first.      */
int stb_attn_decode_planned(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                            const int32_t* ctx_lens, const int32_t* q_rows, const int32_t* n_qs, int B, int n_q,
                            float scale, int max_ctx, int plan_mode, void* work, void* stream);

/* ---- K2: append-prefill attention (n new queries against resident pages)
 * Replaces prefill engine.py:251, verify engine.py:296 and ingest
 * engine.py:358. Sequence s owns query rows [q_start[s], q_start[s+1]) of
 * q/out bf16 [T][n_q][d_head]; its keys are the first ctx_lens[s] pages
 * rows (the new tokens already committed); query i sits at absolute
 * position ctx_lens[s] - n_s + i and attends causally.                    */
int stb_attn_prefill(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                     const int32_t* q_start, const int32_t* ctx_lens, int S, int T, int n_q, float scale,
                     int max_q, void* stream);
/* Same, told how many (query-tile pair, kv head, run) work units hold queries
 * (0 = unknown; a query-tile pair is 2*128/G query tokens): a launch with fewer
 * units than half the SMs (e.g. one 33-token verify pass = 8 units) splits each
 * unit's KV range over up to 18 CTAs, and a second small kernel merges the
 * partial rows by log-sum-exp.                                               */
int stb_attn_prefill_split(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                           const int32_t* q_start, const int32_t* ctx_lens, int S, int T, int n_q, float scale,
                           int max_q, int active_units, void* stream);

/* Same, with the sliding window and sinks of stb_attn_decode_ex (tensor-core path only). */
int stb_attn_prefill_ex(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                        const int32_t* q_start, const int32_t* ctx_lens, int S, int T, int n_q, float scale,
                        int max_q, int active_units, int window, const float* sinks, void* stream);

/* ---- K4: speculation validation (greedy LCP, bit-exact int32) -----------
 * Replaces validate_draft (engine.py:96-111) + the consume rule (engine.py:291).
 * For sequence s: draft ids [d_off[s], d_off[s+1]); the model's ids at the
 * draft positions are model_first[s] (if >= 0: a token sampled by an earlier
 * step) followed by the verify pass's samples model[m_off[s] .. m_off[s+1]);
 * span_len[s]. accepted = LCP(draft, model ids) clamped to span_len;
 * consume = span_len if accepted == span_len else accepted + 1;
 * new_len[s] = kv_len[s] + accepted + base_extra[s] (KV rows that survive
 * rollback). model_first may be NULL. */
int stb_spec_validate(const int32_t* draft, const int32_t* d_off, const int32_t* model, const int32_t* m_off,
                      const int32_t* model_first, const int32_t* span_len, const int32_t* kv_len,
                      const int32_t* base_extra, int S, int32_t* accepted, int32_t* consume, int32_t* new_len,
                      void* stream);

/* K4b: canonical tool-call key digests (the `_span_end` key lookup, engine.py:339-355, and the
 * store's key index, engine.py:63-65): probe / keys hold 128-bit digests as two uint64 each (the
 * host hashes the canonical key bytes, domain.py:123-158); out[i] = the lowest j with
 * key_rid[j] == probe_rid[i] and keys[j] == probe[i] (bit-exact), else -1. */
int stb_key_match(const void* probe, const int32_t* probe_rid, int n, const void* keys, const int32_t* key_rid, int m,
                  int32_t* out, void* stream);

/* ---- K5: bf16 tensor-core GEMM (tcgen05 + TMA + TMEM) --------------------
 * C[M][N] (fp32, row stride ldc) = A[M][K] (bf16, lda) * W[N][K]^T (bf16, ldw).
 * Persistent, one CTA per SM. split_k: 0 = automatic schedule; 1 = whole
 * tiles per CTA (plain stores); >= 2 = stream-K over min(split_k, SMs) CTAs,
 * partial tiles reduced with fp32 red.add into C. C is zeroed by the call
 * unless flags has STB_GEMM_C_ZEROED (the caller guarantees C == 0, e.g.
 * because the consumer of the previous product cleared the rows it read). */
#define STB_GEMM_C_ZEROED 1
/* fused SiLU-gate epilogue (tile schedule only, else STB_EINVAL): W rows hold (gate,
 * up) pairs interleaved (row 2i = gate_i, row 2i+1 = up_i); C is then bf16
 * act[M][N/2] (row stride ldc elements) = silu(gate) * up, computed in fp32 exactly
 * as stb_silu_mul does */
#define STB_GEMM_SILU_MUL 2
/* W is in the tiled HBM layout written by stb_weight_tile (ldw ignored): every
 * 128-row x 64-column weight tile is one contiguous 16 KiB block, already in the
 * 128-byte-swizzled order the tensor core reads, so each pipeline stage is one
 * linear bulk copy (whole DRAM pages) instead of 128 strided 128-byte rows */
#define STB_GEMM_W_TILED 4
/* ---- K5 with fused epilogues (the row ops that used to follow each GEMM) ----
 * C = A * W^T is accumulated in `work` (fp32 [M][N], row stride ldwork), which
 * must be zero on entry and is left zero on exit: stream-K partial tiles are
 * reduced into it with fp32 red.add, the last CTA of each tile (ticket counter)
 * reads the finished tile back and runs the epilogue, then clears it. Whole
 * tiles run the epilogue straight from TMEM. `ss_in` (optional) applies the
 * RMSNorm of the GEMM's input row after the reduction (the norm weight is
 * folded into W): v *= rsqrt(sum_p ss_in[t][p] * inv_dim + eps).
 *   STB_EPI_SILU   out bf16 [M][N/2] (ldo) = silu(gate) * up (W rows interleaved
 *                  as for STB_GEMM_SILU_MUL)
 *   STB_EPI_RESID  x[t][f] += v (fp32, ldx); out bf16 [M][N] (ldo) = x;
 *                  ss_out[t][f / 128] = sum of x^2 over the tile's 128 features
 *                  (the next norm's statistics, written
 *                  with plain stores — deterministic, no atomics)
 *   STB_EPI_QKV    [qk-norm] + RoPE on the q and k heads, q -> out bf16
 *                  [M][n_q*d_head] (ldo), k and v committed into the pool pages
 *                  of `layer` at (slot_of[t], pos_of[t]) — stb_qkv_norm_rope_commit
 *                  fused into the QKV projection (engine.py:251,270,296,358)   */
#define STB_EPI_SILU 1
#define STB_EPI_QKV 2
#define STB_EPI_RESID 3
typedef struct stb_gemm_epi {
  int kind;
  const float* ss_in;   /* [M][ss_parts] partial sums of squares (summed here) */
  int ss_parts;         /* row stride of ss_in / ss_out: >= ceil(d/128), a multiple of 4,
                           unused slots zero (stb_embed_prep zeroes them) */
  float inv_dim, eps;
  void* out;
  int64_t ldo;
  float* x;
  int64_t ldx;
  float* ss_out;
  stb_kv_pool* pool;
  int layer, n_q;
  const int32_t* slot_of;
  const int32_t* pos_of;
  float rope_theta;
  const void* q_norm;
  const void* k_norm;
  float qk_eps;
} stb_gemm_epi;
int stb_gemm_bf16_fused(const void* A, int64_t lda, const void* W, int64_t ldw, float* work, int64_t ldwork, int M,
                        int N, int K, int flags, const stb_gemm_epi* epi, void* stream);
/* x[t] = embed[ids[t]] (fp32), xb = bf16(x), ss[t][0] = sum x^2, ss[t][p] = 0 for
 * 1 <= p < ss_parts: the first layer's fused-norm inputs */
int stb_embed_prep(const int32_t* ids, const void* table, float* x, void* xb, float* ss, int ss_parts, int n, int d,
                   void* stream);

/* elements of the tiled copy of an N x K weight (N padded to 128, K to 64) */
int64_t stb_weight_tiled_elems(int N, int K);
/* out (bf16, stb_weight_tiled_elems(N, K)) = W[N][K] (row stride ldw) in the tiled
 * layout: tile (n, k) at ((n * ceil(K/64)) + k) * 8192 elements, row r of the tile
 * at r * 64, 16-byte chunk c of the row stored at chunk c ^ (r & 7); padding = 0 */
int stb_weight_tile(const void* W, int64_t ldw, int N, int K, void* out, void* stream);
/* 1 if the automatic schedule runs this shape stream-K (C accumulated with reductions) */
int stb_gemm_is_stream(int M, int N, int K);
int stb_gemm_bf16(const void* A, int64_t lda, const void* W, int64_t ldw, float* C, int64_t ldc, int M, int N, int K,
                  int split_k, int flags, void* stream);

/* ---- K5 decode block: a chain of decode-shaped GEMMs and the row ops between them in
 * ONE persistent launch (one CTA per SM, grid-wide barriers between phases). Each
 * GEMM is stream-K over every SM with fp32 red.add into c; its weight tiles stream
 * into the shared-memory ring while the previous phase's reductions and row ops are
 * still finishing, so HBM stays busy across the chain. A decode step then runs
 * [O, norm, gate-up, SiLU, down, norm, QKV(next layer), RoPE+commit] as one launch per
 * layer between the attention launches (replaces the per-token decode charges
 * `engine.py:270,276,302,317` — the same math as the stb_gemm_bf16 /
 * stb_add_rmsnorm / stb_silu_mul / stb_qkv_norm_rope_commit sequence).
 *   STB_OP_GEMM  c[M][n] += x[M][k] (bf16, row stride ldx) * w^T; w in the
 *                stb_weight_tile layout; c fp32 (row stride ldc), zero on entry
 *   STB_OP_NORM  x_res[M][n] += c (when c != NULL; c cleared to 0);
 *                y = bf16(x_res * rsqrt(mean(x_res^2) + eps) * w) when y != NULL
 *                (stb_add_rmsnorm with clear_rows = M)
 *   STB_OP_SILU  y[M][n] = silu(c[t][2i]) * c[t][2i+1] (c cleared; stb_silu_mul)
 *   STB_OP_ROPE  stb_qkv_norm_rope_commit on c = qkv[M][(n_q + 2 n_kv) d_head]
 *                (cleared), q -> y, k / v into layer `layer` of `pool`
 * M <= 64; at most 4 GEMMs and 5 row ops; a row op that opens the chain reads the
 * output of the previous launch on the stream. */
#define STB_OP_GEMM 1
#define STB_OP_NORM 2
#define STB_OP_SILU 3
#define STB_OP_ROPE 4
typedef struct stb_block_op {
  int kind;
  const void* x;       /* GEMM: activations */
  int64_t ldx;
  const void* w;       /* GEMM: tiled weights; NORM: norm weight (bf16 [n]) */
  float* c;            /* GEMM: accumulator; NORM: delta; SILU: gate/up; ROPE: qkv */
  int64_t ldc;
  int n, k;            /* GEMM: N, K; NORM: d; SILU: d_ff */
  float* x_res;        /* NORM: fp32 residual stream [M][n] */
  void* y;             /* NORM / SILU / ROPE: bf16 output */
  float eps;           /* NORM; ROPE (qk-norm) */
  stb_kv_pool* pool;   /* ROPE */
  int layer, n_q;
  const int32_t* slot_of;
  const int32_t* pos_of;
  float rope_theta;
  const void* q_norm;  /* ROPE: Qwen3 qk-norm weights (both or neither) */
  const void* k_norm;
} stb_block_op;
int stb_gemm_block(const stb_block_op* ops, int n_ops, int M, void* stream);

/* ---- small fused ops (HBM-bound elementwise / row ops) ------------------ */
/* x fp32 [n][d] <- table bf16 [ids[i]][d] */
int stb_embed(const int32_t* ids, const void* table, float* x, int n, int d, void* stream);
/* x += delta (if delta != NULL); y bf16 = rmsnorm(x) * w; delta rows < clear_rows
 * are zeroed after reading (see stb_qkv_rope_commit) */
int stb_add_rmsnorm(float* x, float* delta, const void* w, void* y, int n, int d, float eps, int clear_rows,
                    void* stream);
/* y bf16 [n][f] = silu(gate) * up with gu fp32 [n][2f] holding (gate_i, up_i) pairs
 * interleaved (gu[t][2i], gu[t][2i+1]); gu rows < clear_rows zeroed after reading */
int stb_silu_mul(float* gu, void* y, int n, int f, int clear_rows, void* stream);
/* stb_add_rmsnorm with a bias row (fp32 [d], or NULL) added to every delta row: the O
 * projection's bias of the gpt-oss family (config C4) */
int stb_add_bias_rmsnorm(float* x, float* delta, const float* bias, const void* w, void* y, int n, int d, float eps,
                         int clear_rows, void* stream);
/* rows[i] = x[idx[i]] as bf16 after rmsnorm: final norm fused with row gather */
int stb_gather_rmsnorm(const float* x, const int32_t* idx, const void* w, void* y, int n, int d, float eps,
                       void* stream);
/* script-forced greedy sampling: out[r] = argmax(logits[r] + bias * onehot(target[r]))
 * (target < 0: plain argmax); raw_argmax[r] / raw_max[r] = unbiased argmax / max;
 * clear != 0 zeroes the logits rows after reading */
int stb_sample_forced(float* logits, int64_t ld, const int32_t* target, int R, int V, float bias, int32_t* out,
                      int32_t* raw_argmax, float* raw_max, int clear, void* stream);

/* ---- MoE MLP of the gpt-oss family (config C4; moe.cu) --------------------
 * Replaces the MLP share of the phase charges engine.py:251,270,296,358 for routed-expert
 * models. Per layer: router logits [T][E] (K5, bf16) -> stb_moe_route -> stb_moe_gather ->
 * stb_moe_gemm_mxfp4 (gate-up) -> stb_moe_gemm_mxfp4 (down) -> stb_moe_combine.
 * route: + bias, top-k per token (ties -> lower id), softmax over the k logits; expert[t*k+r],
 *   weight[t*k+r], rank[t*k+r] = arrival order within the expert (counts[E] must be zero on
 *   entry and hold the per-expert totals on exit; stb_moe_combine zeroes them again).
 * gather: offsets[E+1] = exclusive prefix of counts; perm[t*k+r] = offsets[e] + rank; xperm
 *   fp16 [T*k][d] = the token rows, expert-contiguous.
 * gemm: per expert e, out rows [offsets[e], offsets[e+1]) = xperm rows x W_e^T (+ bias[e]); W_e
 *   MXFP4 tiles (runtime/weights.py pack_mxfp4_tiles: [E][ceil(N/128)][K/64][4352] bytes);
 *   STB_MOE_GATE_UP: out fp16 [rows][N/2] (ldo) = (clamp(up,-l,l) + 1) * g * sigmoid(1.702 g),
 *   g = min(gate, l), gate / up = even / odd rows of W_e; STB_MOE_DOWN: out fp32 [rows][N].
 *   `rows` = T*k (the host's only view of the routing: it sizes the token tile); rows_cap =
 *   rows allocated in xperm.
 * combine: x[t] += sum_r weight[t*k+r] * y[perm[t*k+r]] (r ascending); h_out bf16 = RMSNorm(x) *
 *   norm_w (skipped if h_out is NULL).                                                    */
#define STB_MOE_GATE_UP 1
#define STB_MOE_DOWN 2
int stb_moe_route(const float* logits, int64_t ld, const float* bias, int T, int E, int k, int32_t* counts,
                  int32_t* expert, int32_t* rank, float* weight, void* stream);
int stb_moe_gather(const void* h, int64_t ldh, int T, int d, int k, int E, const int32_t* counts,
                   const int32_t* expert, const int32_t* rank, int32_t* offsets, int32_t* perm, void* xperm,
                   void* stream);
int stb_moe_gemm_mxfp4(const void* xperm, int rows_cap, const void* wtiles, const float* bias, const int32_t* counts,
                       int E, int N, int K, int kind, float limit, void* out, int64_t ldo, int rows, void* stream);
int stb_moe_combine(float* x, const float* y, int T, int d, int k, const int32_t* perm, const float* weight,
                    const void* norm_w, void* h_out, float eps, int32_t* counts, int E, void* stream);

/* Block-scaled path (the default for the MoE GEMMs): the same product on tcgen05.mma
 * kind::mxf8f6f4.block_scale, with the tensor core applying the weights' own ue8m0 scales, so no
 * thread dequantises the MXFP4 codes. The token rows are split first (stb_moe_quant) into two e4m3
 * halves with one ue8m0 scale per 32 along K (x = hi 2^s_hi + lo 2^s_lo, exact power-of-two
 * scaling; the pair keeps ~2^-8 of each 32-block's maximum, the precision of the bf16 activation):
 *   xq  [2][rows_cap][K] bytes (hi rows, then lo rows)   stb_moe_quant_bytes(rows_cap, K)
 *   xsf [ceil(K/128)][2][pitch = rows_cap rounded up to 4] words of four scale bytes (+ 72 words of overhang)   stb_moe_quant_scale_words(rows_cap, K)
 * stb_moe_gemm_mx takes them in place of the fp16 xperm, and the experts in the MX stage format
 * (runtime/weights.py pack_mx_stages: [E][ceil(N/128)][ceil(K/128)][8704] bytes, per 128-row x
 * 128-wide stage 8192 B of packed codes then 32 x 4 scale words, word (l, j) = the four K-slice
 * scales of row 32 j + l; 16-byte aligned); everything else as stb_moe_gemm_mxfp4. K <= 3072.
 * Replaces the same charges (engine.py:251,270,296,358).                                  */
int64_t stb_moe_quant_bytes(int rows_cap, int K);
int64_t stb_moe_quant_scale_words(int rows_cap, int K);
int stb_moe_quant(const void* x, int64_t ldx, int rows, int K, int rows_cap, void* xq, uint32_t* xsf, void* stream);
/* gather + quant in one pass for the gate-up input: offsets / perm exactly as stb_moe_gather, the
 * routed bf16 rows of h split into xq / xsf as stb_moe_quant would (no fp16 xperm). */
int stb_moe_gather_mx(const void* h, int64_t ldh, int T, int d, int k, int E, const int32_t* counts,
                      const int32_t* expert, const int32_t* rank, int32_t* offsets, int32_t* perm, int rows_cap,
                      void* xq, uint32_t* xsf, void* stream);
/* gate-up on the block-scaled path with the down projection's input split fused into its epilogue:
 * q_out / q_sf (sized by stb_moe_quant_bytes / _scale_words(q_cap, N/2)) receive what
 * stb_moe_quant would write from the SwiGLU rows (computed in fp32, not rounded to fp16 first);
 * `out` (the fp16 act) may then be NULL. Needs N/2 % 64 == 0. */
int stb_moe_gemm_mx_q(const void* xq, const uint32_t* xsf, int rows_cap, const void* wtiles, const float* bias,
                      const int32_t* counts, int E, int N, int K, int kind, float limit, void* out, int64_t ldo,
                      int rows, void* q_out, uint32_t* q_sf, int q_cap, void* stream);
int stb_moe_gemm_mx(const void* xq, const uint32_t* xsf, int rows_cap, const void* wtiles, const float* bias,
                    const int32_t* counts, int E, int N, int K, int kind, float limit, void* out, int64_t ldo, int rows,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STB200_H */
