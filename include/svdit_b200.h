/*
 * svdit_b200.h — C ABI of the B200-native Sparse-vDiT attention hot path.
 *
 * This is the drop-in boundary for the reference's operator layer
 * (svdit 0.1.0, /root/reference/pkg/src/svdit).  The reference has no FFI:
 * it is pure NumPy.  Each entry point below replaces one Python function of
 * the reference's hot path; the Python shim in paper_2506_03065_b200/ binds
 * them with ctypes and keeps the reference signatures.
 *
 *   reference (file:line)                              replaced by
 *   layout.py:135-158  block_grid(layout)              svd_grid_size / svd_grid_arrays
 *   patterns.py:176-181 frame_period(grid)             svd_frame_period
 *   patterns.py:219-259 build_mask(spec, grid)         svd_mask_build
 *   attention.py:164-183 group_heads(assignment, grid) svd_plan_create + svd_plan_group_* accessors
 *   attention.py:186-212 fused_layer_attention(...)    svd_attn_fwd
 *   attention.py:57-98  sparse_attention(q,k,v,mask)   svd_plan_create_from_masks + svd_attn_fwd
 *   attention.py:101-105 full_mask_attention(...)      svd_plan_create (FULL spec) + svd_attn_fwd
 *   attention.py:51-54  skip_attention(...)            svd_plan_create (SKIP spec) + svd_attn_fwd
 *   attention.py:108-146 block_key_mass(q, k, grid)    svd_block_key_mass
 *   model.py:352-355    _layernorm (layer_qkv / layer_finish)   svd_layernorm
 *   model.py:169-195    rope(q), rope(k) (layer_qkv)            svd_rope_table + svd_rope_apply
 *   model.py:357-359    _gelu (layer_finish MLP)                svd_gelu
 *
 * Conventions
 *  - Every function returns an svd_status; on failure a message is available
 *    from svd_last_error() (thread-local).  Status codes map 1:1 onto the
 *    reference's exception classes (errors.py:9-34).
 *  - Plans are immutable once created and may be shared across threads and
 *    CUDA streams.  Device-side plan tables are uploaded lazily, once per
 *    device, on the first svd_attn_fwd call on that device.
 *  - Q/K/V/O are caller-owned device buffers of bf16, addressed through
 *    element strides for the logical [B, H, N, d] view, so both [B,H,N,d]
 *    and [B,N,H,d] storage work without copies.
 *  - svd_attn_fwd is stream-ordered and never synchronises the host.
 */
#ifndef SVDIT_B200_H
#define SVDIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum svd_status {
  SVD_OK = 0,
  SVD_ERR_SHAPE = 1,            /* errors.py:13  ShapeError          */
  SVD_ERR_DEGENERATE_ROW = 2,   /* errors.py:17  DegenerateRowError  */
  SVD_ERR_DEGENERATE_MASK = 3,  /* errors.py:21  DegenerateMaskError */
  SVD_ERR_CONFIG = 4,           /* errors.py:25  ConfigError         */
  SVD_ERR_CUDA = 5,             /* CUDA runtime / driver failure      */
  SVD_ERR_UNSUPPORTED = 6,      /* shape outside the kernel's support */
  SVD_ERR_INTERNAL = 7
} svd_status;

typedef enum svd_mode {         /* patterns.py:31-36 Mode */
  SVD_FULL = 0,
  SVD_SKIP = 1,
  SVD_DIAGONAL = 2,
  SVD_MULTI_DIAGONAL = 3,
  SVD_VERTICAL_STRIPE = 4
} svd_mode;

/* layout.py:26-31 TokenLayout */
typedef struct svd_layout {
  int64_t text_tokens;
  int64_t frames;
  int64_t tokens_per_frame;
  int64_t block_size;
} svd_layout;

/* patterns.py:50-75 PatternSpec.  period <= 0 encodes None (frame period);
 * n_stripes < 0 encodes stripes=None (unresolved).  Stripes may be given in
 * any order with duplicates: they are normalised to sorted-unique exactly as
 * PatternSpec.__post_init__ does (patterns.py:74-75). */
typedef struct svd_spec {
  int32_t mode;
  int32_t halfwidth;
  int32_t period;
  int32_t md_halfwidth;
  int32_t stripe_count;
  int32_t include_diagonal;
  int32_t n_stripes;
  const int64_t* stripes;
} svd_spec;

typedef struct svd_plan svd_plan;

typedef struct svd_plan_info {
  int64_t n_tokens;            /* N                                            */
  int64_t n_blocks;            /* nb = ceil(N / block_size)                    */
  int64_t n_segments;          /* ceil(N / 64): the kernel's 64-token grain    */
  int32_t n_heads;
  int32_t n_groups;
  int32_t fine_mask;           /* 1 when block_size is not a multiple of 64    */
  int32_t sharded;             /* 1 for a svd_plan_shard() view                */
  int64_t n_work_items;        /* CTAs per batch entry                         */
  int64_t n_kv_entries;        /* 128-key tiles over all distinct KV lists     */
  int64_t computed_tiles;      /* 128x128 MMA tiles issued per batch entry     */
  double  active_pairs;        /* sum over heads, active (qb,kb): |qb|*|kb|;   */
                               /* active FLOPs = 4 * d * active_pairs          */
                               /* (costmodel.py:26-32 convention)              */
  double  dense_pairs;         /* N^2 * H                                      */
  int32_t n_split_groups;      /* split-KV items (shard views), else 0         */
  int32_t max_split_parts;     /* parts of the most-split item (1 if none)     */
} svd_plan_info;

/* Thread-local text of the last error (never NULL). */
const char* svd_last_error(void);
/* Library build string (arch, version). */
const char* svd_version(void);

/* ---- layout.py:135-158 block_grid ------------------------------------- */
int svd_grid_size(const svd_layout* layout, int64_t* n_tokens, int64_t* n_blocks);
/* bounds: nb+1 entries; has_text, mixed: nb bytes; frame_index: nb entries. */
int svd_grid_arrays(const svd_layout* layout, int64_t* bounds, uint8_t* has_text,
                    uint8_t* mixed, int64_t* frame_index);
/* patterns.py:176-181 frame_period (round-half-even, clamped to >= 1). */
int svd_frame_period(const svd_layout* layout, int64_t* period);

/* ---- patterns.py:219-259 build_mask ------------------------------------ */
/* active: nb*nb bytes (row-major, 1 = active).  For SKIP *is_skip = 1 and
 * active is left untouched (the reference returns active=None). */
int svd_mask_build(const svd_layout* layout, const svd_spec* spec, uint8_t* active,
                   int32_t* is_skip);

/* ---- attention.py:164-183 group_heads + the kernel schedule ------------ */
int svd_plan_create(const svd_layout* layout, const svd_spec* specs, int32_t n_heads,
                    svd_plan** plan);
/* An explicit-mask plan (sparse_attention on a caller-built BlockMask):
 * group_skip[g] != 0 marks a SKIP group (mask ignored); masks holds
 * n_groups*nb*nb bytes; head_group[h] in [0, n_groups). */
int svd_plan_create_from_masks(const svd_layout* layout, int32_t n_groups,
                               const int32_t* group_skip, const uint8_t* masks,
                               const int32_t* head_group, int32_t n_heads, svd_plan** plan);
void svd_plan_destroy(svd_plan* plan);
int svd_plan_get_info(const svd_plan* plan, svd_plan_info* info);
/* Group g of the reference grouping: first-occurrence order, ascending heads. */
int svd_plan_group_heads(const svd_plan* plan, int32_t g, int32_t* heads, int32_t* n_heads,
                         int32_t* is_skip);
/* Block mask of group g (nb*nb bytes); SKIP groups return SVD_ERR_CONFIG. */
int svd_plan_group_mask(const svd_plan* plan, int32_t g, uint8_t* active);
/* CSR of group g's active key blocks, ascending per row
 * (patterns.py:205-208 active_key_blocks).  row_ptr: nb+1; col_idx: nnz. */
int svd_plan_group_nnz(const svd_plan* plan, int32_t g, int64_t* nnz);
int svd_plan_group_csr(const svd_plan* plan, int32_t g, int64_t* row_ptr, int64_t* col_idx);
/* The plan restricted to the listed heads, in that order (head i of the
 * subset = plan head heads[i]): the parent's groups, masks, schedules and KV
 * lists are copied, not rebuilt (the host-buffer pipeline launches head
 * chunks this way).  Not for shard plans. */
int svd_plan_subset(const svd_plan* plan, const int32_t* heads, int32_t n_heads, svd_plan** out);
/* Restrict the plan's work items to one rank's share (LPT by tile cost) for
 * head/q-range sharding over world ranks.  The shard writes its rows into
 * a packed [rows, d] buffer; svd_plan_shard_rows() reports the row count and
 * the (head, token) of every packed row (for the all-gather unpack). */
int svd_plan_shard(const svd_plan* plan, int32_t world, int32_t rank, svd_plan** shard);
/* As svd_plan_shard, with the shard's long items split along their KV list
 * (split-KV, merged in the kernel) so no item exceeds max_item_tiles 128-key
 * tiles: 0 = an eighth of the shard's mean per-SM load on n_sms SMs (what
 * svd_plan_shard does with n_sms = 148), < 0 = never split. */
int svd_plan_shard_sm(const svd_plan* plan, int32_t world, int32_t rank, int32_t n_sms,
                      int32_t max_item_tiles, svd_plan** shard);
/* As svd_plan_shard_sm, choosing how items are dealt to ranks:
 * SVD_PARTITION_ITEMS — LPT over all items (any rank may touch any head);
 * SVD_PARTITION_HEADS — contiguous head ranges of equal cost (McNaughton's
 * wrap-around: at most the two boundary heads of a rank are split by query
 * range), so a rank reads only its own heads' Q/K/V. */
enum { SVD_PARTITION_ITEMS = 0, SVD_PARTITION_HEADS = 1 };
int svd_plan_shard_ex(const svd_plan* plan, int32_t world, int32_t rank, int32_t n_sms,
                      int32_t max_item_tiles, int32_t partition, svd_plan** shard);
int svd_plan_shard_rows(const svd_plan* shard, int64_t* n_rows, int32_t* row_head,
                        int32_t* row_token);
/* The work items of a shard plan that belong to the listed heads, as a shard
 * plan with the parent's packed row layout (one chunk of a rank's pipelined
 * end-to-end step: copy-in of a head chunk overlaps the previous chunk's
 * kernel).  No reference counterpart (multi-GPU is this repo's own). */
int svd_plan_shard_heads(const svd_plan* shard, const int32_t* heads, int32_t n_heads, svd_plan** out);

/* Kernel schedule dump (tests / tooling): items as 12 int32 each
 * {head, group, kv_begin, kv_count, qseg[4], out_base, 0, 0, 0} and KV
 * entries as 4 int32 each {kseg0, kseg1, flags, 0}. */
int svd_plan_schedule(const svd_plan* plan, int32_t* items, int32_t* kv);

/* ---- attention.py:186-212 fused_layer_attention (bf16, sm_100a) -------- */
/* strides: 4 element strides each for the logical [B, H, N, tensor_dim]
 * view.  head_dim is the true d (softmax scale 1/sqrt(d)); tensor_dim is the
 * stored width, 64 or 128 (head_dim <= tensor_dim, padded with zeros).
 * For a shard plan, o is the packed [rows, tensor_dim] buffer, o_strides[2]
 * its row stride.  dtype: 0 = bf16 (only). */
int svd_attn_fwd(const svd_plan* plan, const void* q, const void* k, const void* v, void* o,
                 const int64_t* q_strides, const int64_t* k_strides, const int64_t* v_strides,
                 const int64_t* o_strides, int32_t batch, int32_t head_dim, int32_t tensor_dim,
                 int32_t dtype, void* stream);

/* As svd_attn_fwd, with an optional output head permutation: plan head h
 * writes O head o_head_map[h] (device int32[n_heads]; NULL = identity).
 * Lets a head-subset plan write straight into a full-layer O — e.g. pinned
 * host memory, so the host-buffer pipeline needs no copy-out stage. */
int svd_attn_fwd_ex(const svd_plan* plan, const void* q, const void* k, const void* v, void* o,
                    const int64_t* q_strides, const int64_t* k_strides, const int64_t* v_strides,
                    const int64_t* o_strides, int32_t batch, int32_t head_dim, int32_t tensor_dim,
                    int32_t dtype, const int32_t* o_head_map, void* stream);

/* As svd_attn_fwd_ex, with attention.py:98 require_finite fused into the
 * epilogue: when any output row holds a non-finite value the kernel ORs 1
 * into *nonfinite (device int32 the caller zeroes; NULL = no check).  The
 * shim reads it back and raises ShapeError, as the reference does. */
int svd_attn_fwd_v2(const svd_plan* plan, const void* q, const void* k, const void* v, void* o,
                    const int64_t* q_strides, const int64_t* k_strides, const int64_t* v_strides,
                    const int64_t* o_strides, int32_t batch, int32_t head_dim, int32_t tensor_dim,
                    int32_t dtype, const int32_t* o_head_map, int32_t* nonfinite, void* stream);

/* The general form of the launch: every option of the operator in one
 * struct (zero-initialise, then set what you need).
 *   q, k, v, o, *_strides, batch, head_dim, tensor_dim, dtype: as svd_attn_fwd.
 *   in_heads     heads of the q/k/v tensors (0 = the plan's heads).
 *   in_head_map  device int32[plan heads]: plan head h reads q/k/v head
 *                in_head_map[h] (NULL = identity) — e.g. the search's
 *                candidate plan, whose heads are (candidate, head) pairs
 *                over one set of q/k/v (search.py:334-372).
 *   o_head_map   device int32[plan heads]: plan head h writes o head
 *                o_head_map[h] (NULL = identity).
 *   nonfinite    as svd_attn_fwd_v2 (NULL = no check).
 *   row_stats    device float [batch * stats_heads][ceil(N / 128)][2][128]:
 *                for every row of plan heads < stats_heads the softmax
 *                statistics (-m, 1/l) in the log2 domain (m the row max of
 *                s / sqrt(head_dim) * log2(e), l the sum of 2^(s' - m)), the
 *                row-statistics pass of block_key_mass (NULL = none).  Rows
 *                past N are written as (-inf, 0) where an item covers them. */
typedef struct svd_fwd_args {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  int64_t q_strides[4];
  int64_t k_strides[4];
  int64_t v_strides[4];
  int64_t o_strides[4];
  int32_t batch;
  int32_t head_dim;
  int32_t tensor_dim;
  int32_t dtype;
  int32_t in_heads;
  int32_t stats_heads;
  const int32_t* in_head_map;
  const int32_t* o_head_map;
  int32_t* nonfinite;
  float* row_stats;
} svd_fwd_args;
int svd_attn_fwd_args(const svd_plan* plan, const svd_fwd_args* args, void* stream);

/* Fused compute + reassembly for multi-GPU: as svd_attn_fwd, but every
 * output row the plan (typically a svd_plan_shard view) produces is stored
 * into all n_peers O buffers — this rank's and its peers' [B, H, N,
 * tensor_dim] outputs mapped into this process (CUDA IPC / NVLink P2P) —
 * straight from the kernel epilogue, so no separate all-gather or unpack
 * runs on the data path.  All peers share o_strides.  n_peers <= 8. */
int svd_attn_fwd_peers(const svd_plan* plan, const void* q, const void* k, const void* v,
                       void* const* o_peers, int32_t n_peers, const int64_t* q_strides,
                       const int64_t* k_strides, const int64_t* v_strides,
                       const int64_t* o_strides, int32_t batch, int32_t head_dim,
                       int32_t tensor_dim, int32_t dtype, void* stream);

/* CUDA IPC helpers for svd_attn_fwd_peers: export a device pointer as a
 * 64-byte handle + byte offset into its allocation; import a peer's handle
 * on the CURRENT device (peer access enabled lazily) and get the pointer;
 * close an imported mapping (pass the pointer svd_ipc_import returned). */
int svd_ipc_export(const void* ptr, uint8_t* handle64, int64_t* offset);
int svd_ipc_import(const uint8_t* handle64, int64_t offset, void** ptr);
int svd_ipc_close(void* ptr, int64_t offset);

/* Stream-ordered barrier between the ranks of svd_attn_fwd_peers, over peer
 * memory (no host synchronisation): flags[r] is rank r's int32[n_peers]
 * flag array mapped into this process (flags[rank] = this rank's own).  The
 * kernel stores `epoch` into slot `rank` of every rank's array (release,
 * system scope) and waits until every slot of its own array reaches `epoch`
 * (acquire).  Enqueued after the shard kernel, it completes once every
 * rank's rows of that step are in every O.  Epochs increase by one per step
 * (wrap-around safe).  A wait longer than timeout_s (<= 0: 30 s) stores 1 into
 * *timed_out (device int32, may be NULL) and returns, so a dead peer cannot
 * hang the GPU. */
int svd_peer_barrier(int32_t* const* flags, int32_t n_peers, int32_t rank, int32_t epoch,
                     int32_t* timed_out, double timeout_s, void* stream);

/* Per-head sum of squared differences in fp64 (numerics.py:114-121 mse, the
 * search's reconstruction error, search.py:65-79): out[h] += sum over
 * (b, n, c<d) of (a - b)^2 for bf16 [B, H, N, >=d] tensors given by element
 * strides; b == NULL means zeros (the SKIP candidate).  out is a device
 * double[H] the caller zeroes; divide by B*N*d for the MSE. */
int svd_head_sqdiff(const void* a, const void* b, const int64_t* a_strides,
                    const int64_t* b_strides, int32_t batch, int32_t heads, int64_t n_tokens,
                    int32_t head_dim, double* out, void* stream);

/* ---- block_key_mass (attention.py:108-146; the search's stripe calibration) --
 * mass[b, h, kb] (device double [B, H, nb], nb = ceil(N / block_size)) = the
 * softmax attention mass of all query rows on key block kb, / N: each (b, h)
 * row sums to 1.  q, k: bf16 [B, H, N, tensor_dim] via element strides,
 * scale 1/sqrt(head_dim).  Two tensor-core passes (row max / sum, then
 * per-key sums) and an fp64 per-block sum; deterministic.  workspace: device
 * scratch of svd_key_mass_workspace(batch, heads, N) bytes, 16-byte aligned. */
int64_t svd_key_mass_workspace(int32_t batch, int32_t heads, int64_t n_tokens);
int svd_block_key_mass(const void* q, const void* k, const int64_t* q_strides,
                       const int64_t* k_strides, int32_t batch, int32_t heads, int64_t n_tokens,
                       int32_t head_dim, int32_t tensor_dim, int32_t block_size, int32_t dtype,
                       void* workspace, int64_t workspace_bytes, double* mass, void* stream);

/* block_key_mass's key-sum pass alone, given the row statistics a forward
 * launch already produced (svd_fwd_args.row_stats of an all-FULL plan over
 * the same q, k): the search's first evaluation of a layer gets the FULL
 * candidate and the stripe calibration from one attention pass plus this
 * key-sum pass.  row_stats: [batch * heads][ceil(N / 128)][2][128];
 * workspace as svd_block_key_mass (its row-statistics part is unused). */
int svd_block_key_mass_from_stats(const void* q, const void* k, const int64_t* q_strides,
                                  const int64_t* k_strides, int32_t batch, int32_t heads,
                                  int64_t n_tokens, int32_t head_dim, int32_t tensor_dim,
                                  int32_t block_size, int32_t dtype, const float* row_stats,
                                  void* workspace, int64_t workspace_bytes, double* mass,
                                  void* stream);

/* Scatter a gathered [world * max_rows, d] buffer of packed shard rows back
 * into O [B=1, H, N, d] (the multi-GPU reassembly after the NCCL all-gather). */
int svd_unpack_rows(const int32_t* row_head_dev, const int32_t* row_token_dev, int64_t n_rows,
                    const void* packed, int64_t packed_row_stride, void* o,
                    const int64_t* o_strides, int32_t head_dim, void* stream);

/* ---- steps either side of the operator (model.py:372-402) ------------------
 * The projections are plain GEMMs (cuBLAS); these are the streaming passes
 * between them.  All pointers are device pointers, 16-byte aligned. */

/* C[M, N] = A[M, K] . B[K, N] on the tensor cores (tcgen05, fp32 accumulate)
 * with the block's element-wise step fused into the epilogue.  A, B: bf16
 * row-major with leading dimensions lda / ldb (elements; the weight B as
 * stored, [in, out]).  epilogue:
 *   0 = bf16 out
 *   1 = bf16 out, RoPE (model.py:169-195) on columns [0, rope_cols): column c
 *       belongs to head-local column c % head_dim, pair (2i, 2i+1) rotates by
 *       rope_table[row % n_tokens][i] = (cos, sin) (svd_rope_table)
 *   2 = bf16 out, exact GELU (model.py:357-359)
 *   3 = fp32 out + resid (fp32 [M, ldr])
 *   4 = fp32 out
 * N, K multiples of 8; out rows 16-byte aligned. */
int svd_gemm(const void* a, int64_t lda, const void* b, int64_t ldb, void* out, int64_t ldo, int64_t M,
             int64_t N, int64_t K, int32_t epilogue, const float* resid, int64_t ldr, const void* rope_table,
             int32_t rope_cols, int32_t head_dim, int64_t n_tokens, void* stream);

/* LayerNorm without affine over rows of `dim` fp32 values (model.py:352-355),
 * bf16 output y.  resid != NULL fuses the residual add first: x_out = x +
 * resid (fp32, may alias x) and y = LN(x_out).  dim % 4 == 0. */
int svd_layernorm(const float* x, const float* resid, float* x_out, void* y, int64_t rows,
                  int32_t dim, float eps, void* stream);

/* RoPE table (model.py:169-195): table[n][c] = (cos, sin)(n * base^(-2c/d)),
 * float2[n_tokens][head_dim / 2], computed in fp64. */
int svd_rope_table(void* table, int64_t n_tokens, int32_t head_dim, double base, void* stream);

/* RoPE in place on the q block (columns [0, H*d)) and the k block (columns
 * [k_off, k_off + H*d)) of a bf16 [rows = B*N, ld] projection output; row r
 * is token r % n_tokens.  head_dim % 8 == 0, ld and k_off multiples of 8. */
int svd_rope_apply(void* qkv, int64_t rows, int64_t ld, int64_t k_off, int64_t n_tokens,
                   int32_t heads, int32_t head_dim, const void* table, void* stream);

/* Exact GELU in place on `count` bf16 values (model.py:357-359); count % 8 == 0. */
int svd_gelu(void* u, int64_t count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SVDIT_B200_H */
