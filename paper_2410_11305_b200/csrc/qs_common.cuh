// Shared definitions: device layouts, argument blocks and helpers.
//
// Device weight layout ("chunk layout", produced once at load/quantize time):
//   codes  [n_tiles][n_chunks][4][128][16] bytes
//          tile  = 128 output rows, chunk = 128 (padded) K positions.
//          piece j (0..3) of row r holds packed bytes pb = 16j..16j+15 of the
//          row's 64-byte chunk; packed byte pb = nib(code[k=pb]) | nib(code[k=64+pb]) << 4
//          with OFFSET-BINARY nibbles nib(c) = c + 8 (k relative to the chunk): one mask
//          (and a shift) turns 4 nibbles into 4 unsigned bytes u = c + 8 for the tensor
//          core, and sum_k c*x = sum_k u*x - 8 * sum_k x (the "acorr" sums below).  Groups of g
//          codes are zero-padded to gp = roundup(g, 128) so every chunk belongs
//          to exactly one quantisation group (cpg = gp/128 chunks per group).
//   scales [n_tiles][n_chunks][128] fp32 (tile-major: one stage of a tile reads one
//          contiguous run; a group of gp > 128 repeats its scale in each of its chunks).
// Activation operand image (produced per step by act_pack):
//   img    [n_chunks][r_pad][128] int8, 128B-swizzled K-major (UMMA SW128),
//          row = token*L + limb.  L = 1 (W4A4 draft: int4 codes in int8),
//          L = 3 (W4A16 verify: 24-bit fixed point split in three int8 limbs).
//   ascale [n_chunks][a_ld] fp32 per (chunk, token): s_x (draft) or 2^-e (verify).
//   acorr  [n_chunks][a_ld][4] int32 per (chunk, token), right after ascale in the same
//          buffer: {8*S0, 8*S1, 8*S2, 8*(256*S1 + S0)}, S_l = sum over the chunk of the
//          token's limb-l image bytes (L = 1: S0 only) -- the offset-binary correction.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

namespace qs {

// Launch with programmatic stream serialisation (PDL): the kernel may start while
// its predecessor drains; every forward-path kernel calls pdl_wait() before it
// touches predecessor outputs.  QS_NO_PDL=1 in the environment disables it.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int kMaxDevices = 64;
constexpr int kLeafLd = 128;    // emit leaf-sum row stride (d_model tiles <= 128)
constexpr int kLeafRows = 64;   // emit leaf-sum rows (tokens) cleared per tile  // per-device caches of kernel attributes
constexpr int kTileN = 128;    // output rows per tile (UMMA M)
constexpr int kChunkK = 128;   // K positions per chunk (one SW128 row of int8)
constexpr int kChunkBytes = kTileN * kChunkK / 2;  // 8 KiB packed weights per (tile, chunk)

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int round_up(int a, int b) { return ceil_div(a, b) * b; }
// rows of the activation image for T tokens with L limbs (UMMA N: 8 or 16k)
__host__ __device__ inline int img_rows(int T, int L) {
  int r = T * L;
  return r <= 8 ? 8 : round_up(r, 16);
}

// Per-launch device timeline (qs_ktrace_enable): thread 0 of every CTA folds its
// %globaltimer at entry / exit into buf[2*slot] (min) / buf[2*slot+1] (max), so a
// replayed CUDA graph yields each kernel's [first CTA start, last CTA end] without
// breaking programmatic dependent launch.  buf == nullptr: off (one predicated branch).
struct KTrace {
  unsigned long long* buf;
  int slot;
};
__device__ __forceinline__ unsigned long long kt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ktrace_enter(const KTrace& k) {
  if (k.buf != nullptr && threadIdx.x == 0) atomicMin(&k.buf[2 * k.slot], kt_now());
}
__device__ __forceinline__ void ktrace_exit(const KTrace& k) {
  if (k.buf != nullptr && threadIdx.x == 0) atomicMax(&k.buf[2 * k.slot + 1], kt_now());
}
struct KTraceScope {
  const KTrace& k;
  __device__ __forceinline__ explicit KTraceScope(const KTrace& k_) : k(k_) { ktrace_enter(k); }
  __device__ __forceinline__ ~KTraceScope() { ktrace_exit(k); }
};

enum Emit : int { kEmitNone = 0, kEmitSilu = 1, kEmitRms = 2 };

enum PostOp : int {
  kOpStore = 0,     // out[t, n] = y
  kOpResidual = 1,  // out[t, n] += y          (o_proj / down_proj)
  kOpSiluMul = 2,   // out[t, n/2] = silu(y[2i]) * y[2i+1]   (interleaved gate/up)
  kOpQkvRope = 3,   // rope(q) -> out, rope(k) -> K cache, v -> V cache
  kOpLogits = 4,    // logits (optional store) + fused argmax
  kOpDump = 5,      // debug: raw int32 group dots
};

struct PackArgs {
  const float* x;
  int ldx;
  const int* gather_ids;
  const float* emb;
  float* x_out;
  const float* rms_w;
  float eps;
  int T, K, g, gp, G, n_chunks, r_pad, a_ld;
  uint8_t* img;
  float* ascale;
  int32_t* acorr;  // [n_chunks][a_ld][4] offset-binary correction sums (with img)
  int rotate;      // opt-in 128-point Hadamard rotation of every group before quantising
  int8_t* codes_out;
  float* scales_out;
  float* fq_out;
  float* y_out;
  // attention combine mode (o_proj operand): x[t, h*hd+d] = sum_c w_c o_c[d] / sum_c w_c l_c
  const float* att_o;   // [T][H][cmax][hd]
  const float* att_ml;  // [T][H][cmax][2]  (chunk max, chunk sum)
  const int* att_pos;   // [T] query positions (context = pos + 1)
  int att_hd, att_cmax, att_chunk;
  KTrace kt;
};

constexpr int kMaxPf = 6;  // prefetch ranges per linear launch

struct LinearArgs {
  const uint8_t* codes;
  const float* wscale;
  const uint8_t* act;
  const float* ascale;
  const int32_t* acorr;  // [n_chunks][a_ld][4], see the layout notes above
  int n, n_pad, n_tiles, G, cpg, n_chunks;
  int T, r_pad, a_ld;
  int n_cta;
  float* part;     // [(n_cta + n_tiles)][tmax][128]
  int* counters;   // [n_tiles + 1], zero on entry, left zero on exit
  int op;
  float* out;
  int ldo;
  // kOpQkvRope
  const int* pos;
  const int* slot;
  const float* rope_cos;
  const float* rope_sin;
  int hd, n_q, n_k, n_kv_heads;
  float* kcache;
  float* vcache;
  const int* block_table;
  int bt_ld, page, page_shift;  // page = 1 << page_shift
  // kOpLogits
  float* arg_val;
  int* arg_idx;
  int* argmax_out;
  int2* arg_rec;   // vocab-split TP: (max value bits, global index) per token instead of argmax_out
  int arg_off;     // this shard's first vocab row
  // kOpDump
  int32_t* dump;
  // operand producer of this linear (run by a preceding act_pack launch)
  PackArgs pk;
  // L2 prefetch.  Weights do not depend on activations, so HBM can stream ahead of the
  // dependency chain: this launch prefetches the byte ranges pf_ptr/pf_len (pieces of
  // LATER linears' codes and scales, a fixed window ahead in the forward's weight
  // stream), split evenly over its CTAs; pf_own also prefetches this CTA's own units
  // beyond what its shared-memory ring requests up front.
  const uint8_t* pf_ptr[kMaxPf];
  uint32_t pf_len[kMaxPf];
  int pf_n;
  int pf_own;
  KTrace kt;
  // Next-operand emit: the act pack of the NEXT linear fused into this epilogue.
  //   kEmitSilu (gate_up): the owner that completes a 128-wide group of silu outputs (a
  //     pair of interleaved gate/up tiles) quantises it into down_proj's operand chunk.
  //   kEmitRms (o_proj / down_proj residual): every tile owner publishes its numpy
  //     pairwise leaf sum of squares (leaf = tile = 128 elements), waits for all owners,
  //     forms 1/rms per token exactly as numerics.py:46-62 and quantises its own tile --
  //     one group -- of the RMSNorm'd row into the next linear's operand chunk.
  int emit;
  uint8_t* e_img;
  float* e_ascale;
  int32_t* e_acorr;
  const float* e_rms_w;
  float e_eps;
  int e_n;         // row width (the RMSNorm mean's n)
  // kEmitRms leaf sums, [t][kLeafLd] as ~bits(sum) (0 = not yet published): o_proj and
  // down_proj alternate between two buffers, each launch clearing the other one's entries
  // of its tiles (that buffer's last readers belong to a launch that has completed)
  unsigned* e_leaf;
  unsigned* e_leaf_clr;
  int* e_cnt;      // [8 + q] per group (kEmitSilu); zero on entry and exit
  int e_rotate;    // Hadamard-rotate the emitted groups (model option)
  // debug timeline (CTA 0): [role][i] globaltimer ns; roles: 0 producer issue, 1 unpack done,
  // 2 mma issued, 3 epilogue start (acc ready), 4 epilogue done
  unsigned long long* dbg;
};



struct AttnArgs {
  const float* q;
  int ldq;
  float* part_o;   // [T][H][cmax][hd] split-KV partials
  float* part_ml;  // [T][H][cmax][2]
  int cmax;        // chunks per query capacity
  const float* kcache;
  const float* vcache;
  const int* block_table;
  int bt_ld, page;
  const int* pos;
  const int* slot;
  const int* blk_tok0;
  const int* blk_ntok;
  int H, KV, hd, hpk;
  float inv_sqrt_hd;
  int qmax, ctx_cap;
  float* out;
  int ldo;
  KTrace kt;
};

struct QuantWArgs {
  // source: LCG (src == nullptr) or fp32 row-major [rows, cols]
  const float* src;
  unsigned long long seed, offset;  // offset = draw index of element (0, 0)
  float scale;                      // f32(1/sqrt(d_model)) applied to LCG draws
  int rows, cols, g;
  // destination chunk layout
  uint8_t* codes;
  float* scales;
  int n_pad, n_chunks, gp, G;
  int row_off, row_stride;  // dst_row = row_off + n * row_stride
  uint8_t* ref_codes;       // optional reference-layout packed codes (flat, even in low nibble)
  float* ref_scales;        // optional reference-layout scales [rows, G]
};

struct SeqState {
  int* pending;
  int* committed;
  int* n_out;
  int* done;
  int* finish;      // 0 running, 1 eos, 2 max_new_tokens
  int* max_new;
  int* g_eff;
  int* drafted;     // [B][gamma]
  int* out_tokens;  // [B][out_cap]
  int* n_drafted;
  int* n_accepted;
  int* n_cycles;
  int* dropped;
  int* trace;       // [B][trace_cap][4]: drafted_len, accept_len, kept_len, is_bonus
  int* trace_tok;   // [B][trace_cap][gamma]
  int out_cap, trace_cap;
  int B, gamma, eos, max_seq;
  int* tok;         // forward inputs
  int* pos;
  int* slot;
  const int* argmax;  // forward output
};

}  // namespace qs
