/* qspec_b200.h -- C ABI of the B200-native QSpec decode hot path.
 *
 * Plain pointers and sizes only: every buffer is caller-allocated device memory,
 * every call is asynchronous on the caller's cudaStream_t (passed as void*),
 * nothing allocates or synchronises, and errors come back as status codes
 * (QS_OK == 0) that the Python shim maps onto the reference exception classes
 * (pkg/src/qspec/errors.py:6-39).
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/qspec):
 *   qs_quantize_weight / qs_init_weight  <- quant.py:197-218 quantize_groupwise,
 *                                           storage.py:135-182 random_init (LCG draws)
 *   qs_lcg_fill                          <- storage.py:62-101 Lcg64.fill
 *   qs_repack_ref                        <- storage.py:352-422 load_checkpoint (codes+scales)
 *   qs_act_quant                         <- quant.py:179-194 _quantize_groups,
 *                                           quant.py:229-245 fake_quantize_activations
 *   qs_rmsnorm                           <- numerics.py:46-62 rmsnorm (numpy pairwise sum order)
 *   qs_w4a4_linear / qs_w4a16_linear     <- quant.py:248-261 qlinear_forward (LOW / HIGH)
 *   qs_forward                           <- model.py:255-348 forward
 *   qs_forward_tp                        <- model.py:255-348 forward, one tensor-parallel shard
 *   qs_draft_prep / qs_verify_prep /
 *   qs_accept / qs_ar_prep / qs_ar_commit <- specdec.py:103-176, 258-335 (+ model.py:211-229 kv_commit)
 */
#ifndef QSPEC_B200_H
#define QSPEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  QS_OK = 0,
  QS_ERR_SHAPE = 1,    /* -> ShapeError */
  QS_ERR_CONFIG = 2,   /* -> ConfigError */
  QS_ERR_OVERFLOW = 3, /* -> SequenceOverflowError */
  QS_ERR_TOKEN = 4,    /* -> TokenIdError */
  QS_ERR_CUDA = 5      /* CUDA launch / runtime failure */
};

enum { QS_MODE_HIGH = 0, QS_MODE_LOW = 1 }; /* quant.py:37-41 ExecutionMode */

/* One quantised weight store in the device chunk layout. */
typedef struct {
  const uint8_t* codes; /* [n_tiles][n_chunks][4][128][16] packed int4 */
  const float* scales;  /* [n_tiles][n_chunks][128], tile-major */
  int32_t n, k, g, n_pad, n_tiles, G, gp, cpg, n_chunks;
} qs_qweight_t;

typedef struct {
  const float* attn_norm;
  const float* ffn_norm;
  qs_qweight_t qkv;     /* rows: q | k | v */
  qs_qweight_t o;
  qs_qweight_t gate_up; /* rows interleaved: gate_i, up_i */
  qs_qweight_t down;
  float* k_cache;       /* [num_pages][n_kv_heads][page][head_dim] fp32 */
  float* v_cache;
} qs_layer_t;

typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, d_ff, vocab, group_size, rope_len;
  float norm_eps;
  const float* tok_emb;    /* [vocab][d_model] */
  const float* final_norm; /* [d_model] */
  const float* rope_cos;   /* [rope_len][head_dim/2] */
  const float* rope_sin;
  qs_qweight_t lm_head;
  const qs_layer_t* layers; /* HOST array [n_layers] */
  const int32_t* block_table; /* device [slots][bt_ld] page ids */
  int32_t bt_ld, page;
  int32_t hadamard; /* opt-in (default 0; the reference has no rotation): every linear operand
                       group is rotated by the orthonormal 128-point Walsh-Hadamard transform
                       before quantisation; the weights were rotated the same way when built
                       (qs_hadamard_rows), so x.W^T is unchanged up to rounding */
} qs_model_t;

/* One forward pass: T tokens; query blocks = runs of tokens of one slot. */
typedef struct {
  int32_t T;
  const int32_t* tokens;    /* device [T] */
  const int32_t* positions; /* device [T] absolute positions */
  const int32_t* slots;     /* device [T] KV slot (block-table row) */
  int32_t n_blk;
  const int32_t* blk_tok0;  /* device [n_blk]; NULL (with blk_ntok NULL): uniform blocks, block i =
                               tokens [i * blk_qmax, (i + 1) * blk_qmax) */
  const int32_t* blk_ntok;  /* device [n_blk] */
  int32_t blk_qmax;         /* max tokens per block (<= 64 / (n_heads/n_kv_heads)) */
  int32_t ctx_cap;          /* max context any query can see */
} qs_batch_t;

typedef struct {
  float* x;       /* [t_max][d_model] residual stream */
  float* h;       /* [t_max][d_ff] */
  float* attn;    /* [t_max][d_model] */
  float* q;       /* [t_max][n_heads*head_dim] */
  uint8_t* img;   /* activation operand image */
  float* ascale;  /* activation scales */
  float* part;    /* stream-K partials */
  int32_t* counters; /* zero-initialised once; kernels leave them zero */
  float* arg_val;
  int32_t* arg_idx;
  float* att_o;   /* split-KV attention partials [t_max][n_heads][chunks][head_dim] */
  float* att_ml;  /* [t_max][n_heads][chunks][2] chunk max / chunk sum */
} qs_workspace_t;

typedef struct {
  size_t x, h, attn, q, img, ascale, part, counters, arg_val, arg_idx, att_o, att_ml; /* bytes */
} qs_workspace_sizes_t;

/* Device sequence state for B slots (SoA), driven by the control kernels. */
typedef struct {
  int32_t *pending, *committed, *n_out, *done, *finish, *max_new, *g_eff, *drafted, *out_tokens;
  int32_t *n_drafted, *n_accepted, *n_cycles, *dropped, *trace, *trace_tok;
  int32_t out_cap, trace_cap;
  int32_t B, gamma, eos, max_seq;
  int32_t *tok, *pos, *slot;
  const int32_t* argmax;
} qs_seq_t;

/* ------------------------------------------------------------------ info */
const char* qs_version(void);
int qs_num_sms(int32_t* out);
int qs_linear_max_tokens(void); /* largest T one linear launch accepts (64) */
int qs_attention_chunk_len(void); /* key positions per split-KV chunk (the attention grid covers
                                     ceil(qs_batch_t.ctx_cap / this) chunks) */
int qs_workspace_size(const qs_model_t* m, int32_t t_max, qs_workspace_sizes_t* out);
int qs_qweight_geometry(int32_t n, int32_t k, int32_t g, qs_qweight_t* out); /* fills dims, not pointers */

/* --------------------------------------------------------------- weights */
int qs_init_weight(uint64_t seed, uint64_t draw_offset, float scale, int32_t rows, int32_t cols, int32_t g,
                   uint8_t* codes, float* scales, int32_t n_pad, int32_t row_off, int32_t row_stride,
                   uint8_t* ref_codes, float* ref_scales, void* stream);
int qs_quantize_weight(const float* w, int32_t rows, int32_t cols, int32_t g, uint8_t* codes, float* scales,
                       int32_t n_pad, int32_t row_off, int32_t row_stride, uint8_t* ref_codes, float* ref_scales,
                       void* stream);
int qs_lcg_fill(float* out, uint64_t seed, uint64_t draw_offset, int64_t count, float scale, void* stream);
int qs_repack_ref(const uint8_t* ref_codes, const float* ref_scales, int32_t rows, int32_t cols, int32_t g,
                  uint8_t* codes, float* scales, int32_t n_pad, int32_t row_off, int32_t row_stride, void* stream);

/* ------------------------------------------------------------- operators */
/* In-place orthonormal 128-point Walsh-Hadamard transform of every 128-block of every row
   of x [rows][cols] (cols % 128 == 0): the opt-in rotation (qs_model_t.hadamard) */
int qs_hadamard_rows(float* x, int64_t rows, int32_t cols, void* stream);
int qs_act_quant(const float* x, int32_t T, int32_t K, int32_t g, int8_t* codes, float* scales, float* fq,
                 void* stream);
/* numerics.py:46-62 rmsnorm: y = (x * (1/sqrt(mean(x^2) + eps))) * w per row, bit-exact
 * with numpy (pairwise float32 sum of squares); x, y [T, K] fp32 device, w [K]. */
int qs_rmsnorm(const float* x, const float* w, int32_t T, int32_t K, float eps, float* y, void* stream);
int qs_w4a4_linear(const qs_qweight_t* w, const float* x, int32_t T, float* y, const qs_workspace_t* ws,
                   void* stream);
int qs_w4a16_linear(const qs_qweight_t* w, const float* x, int32_t T, float* y, const qs_workspace_t* ws,
                    void* stream);
/* the tensor-core linear alone, on the operand image the previous qs_w4a*_linear call packed (microbench) */
int qs_linear_prepacked(const qs_qweight_t* w, int32_t T, int32_t mode, float* y, const qs_workspace_t* ws,
                        void* stream);
/* debug: device buffer [6][256] u64 that qs_linear_prepacked fills with a CTA-0 %globaltimer timeline (NULL: off) */
int qs_debug_timeline(uint64_t* buf);
/* debug: the launch_index-th linear launch enqueued by qs_forward after this call (from 1;
   0 = none) records that timeline (builds with -DQS_LIN_TIMELINE=1 only) */
int qs_debug_select(int32_t launch_index);
/* raw int32 per-(row, group, image-row) dots of the tensor-core integer core */
int qs_linear_group_dots(const qs_qweight_t* w, const float* x, int32_t T, int32_t mode, int32_t* dots,
                         const qs_workspace_t* ws, void* stream);

/* -------------------------------------------------------------- profiling */
/* Event ring around every linear launch of qs_forward (tag = mode*16 + kind,
 * kind: 0 qkv, 1 o, 2 gate_up, 3 down, 4 lm_head).  Host-side bookkeeping only;
 * records become event nodes when qs_forward is captured into a CUDA graph. */
int qs_profile_enable(int32_t max_launches); /* 0 disables */
int qs_profile_reset(void);
/* Device timeline of every forward-path launch enqueued while enabled: buf is a device
 * array of cap pairs (start, end) the caller fills with (UINT64_MAX, 0); each launch
 * takes the next pair and folds %globaltimer of every CTA's entry (min) and exit (max)
 * into it -- also when replayed from a CUDA graph captured while enabled.  Tags as for
 * qs_profile_read (mode*16 + kind, kind 5 = operand pack, 6 = attention).  buf NULL
 * disables; qs_ktrace_read returns the tags in launch order. */
int qs_ktrace_enable(uint64_t* buf, int32_t cap);
int qs_ktrace_read(int32_t* tags, int32_t max_out, int32_t* n_out);
int qs_profile_read(float* ms, int32_t* tags, int32_t max_out, int32_t* n_out);

/* ------------------------------------------------------------------ step */
int qs_forward(const qs_model_t* m, const qs_batch_t* b, int32_t mode, const qs_workspace_t* ws, float* logits,
               int32_t* argmax, void* stream);

/* Tensor-parallel forward (config 3, 13B TP 2/4/8): the model struct holds ONE
 * rank's shard -- q/k/v and gate/up column-split (n_heads, n_kv_heads, d_ff are
 * the rank's), o_proj and down_proj row-split along K (group-aligned), embedding,
 * norms and lm_head replicated.  After each row-split linear the partial [T, d]
 * sum is handed to `allreduce(ptr, count, stream, user)` (e.g. an NCCL all-reduce
 * enqueued on `stream`), then added into the residual stream: one all-reduce per
 * block half, 2 per layer.  Returns the hook's failure as QS_ERR_CUDA. */
typedef int (*qs_allreduce_fn)(float* ptr, int64_t count, void* stream, void* user);
/* all-gather of `bytes` per rank: recv[r * bytes ..] = send of rank r (hook mode) */
typedef int (*qs_allgather_fn)(const void* send, void* recv, int64_t bytes, void* stream, void* user);

/* Tensor-parallel QSpec step (config 4; reference loop specdec.py:258-317 over a TP
 * shard).  The model struct holds this rank's shard as for qs_forward_tp, except that
 * lm_head is VOCAB-SPLIT: rows [vocab_off, vocab_off + m->vocab) of the full head.  The
 * collectives run on `stream`: with nccl_comm set (qs_tp_nccl_init), ncclAllReduce of the
 * row-split partial sums (2 per layer) and ncclAllGather of each rank's (max, index) pair
 * per token, reduced in rank order with the lowest index winning ties (numerics.py:81-86)
 * -- no host callback, no synchronisation, so whole draft/verify cycles capture into one
 * CUDA graph.  With nccl_comm == NULL the two hooks are called instead (tests: gloo).
 * `logits` (optional) receives this rank's vocab shard [T][m->vocab]; `argmax` the global
 * token ids.  scratch: device buffer of qs_tp_scratch_bytes(world) bytes. */
typedef struct {
  int32_t world, rank;
  int32_t vocab_off;
  void* nccl_comm;
  qs_allreduce_fn allreduce;
  qs_allgather_fn allgather;
  void* user;
  void* scratch;
} qs_tp_t;
size_t qs_tp_scratch_bytes(int32_t world);
int qs_tp_nccl_unique_id(uint8_t* id128);
int qs_tp_nccl_init(int32_t world, int32_t rank, const uint8_t* id128, void** comm);
int qs_tp_nccl_destroy(void* comm);
int qs_forward_tp2(const qs_model_t* m, const qs_batch_t* b, int32_t mode, const qs_workspace_t* ws, float* logits,
                   int32_t* argmax, const qs_tp_t* tp, void* stream);
/* kernels the last qs_forward / qs_forward_tp call enqueued (host-side count) */
int qs_forward_launches(void);
/* fused next-operand emits, mask: 1 = gate_up's epilogue emits down_proj's operand, 2 = the
   residual epilogues (o_proj, down_proj) emit the RMSNorm'd operand of the next linear;
   0 = a separate act_pack before every linear.  Default: QS_EMIT env, else 3. */
int qs_set_emit(int32_t mask);

int qs_forward_tp(const qs_model_t* m, const qs_batch_t* b, int32_t mode, const qs_workspace_t* ws, float* logits,
                  int32_t* argmax, int32_t world, qs_allreduce_fn allreduce, void* user, void* stream);

/* --------------------------------------------------------------- control */
int qs_draft_prep(const qs_seq_t* s, int32_t step, void* stream);
int qs_verify_prep(const qs_seq_t* s, void* stream);
int qs_accept(const qs_seq_t* s, void* stream);
int qs_ar_prep(const qs_seq_t* s, void* stream);
int qs_ar_commit(const qs_seq_t* s, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QSPEC_B200_H */
