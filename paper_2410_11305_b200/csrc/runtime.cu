// C-ABI entry points and the native step runtime (qs_forward): the per-layer
// launch sequence of model.py:255-348 over device-resident weights and the
// shared paged KV cache.  No allocation, no synchronisation: everything is
// enqueued on the caller's stream, so the Python engine can capture whole
// draft/verify cycles into CUDA graphs.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include "../../include/qspec_b200.h"
#include "qs_common.cuh"

namespace qs {
cudaError_t launch_linear(int L, const LinearArgs& a, cudaStream_t st);
int linear_tmax_bucket(int T, int L);
cudaError_t launch_act_pack(int L, const PackArgs& a, cudaStream_t st);
cudaError_t launch_attention(const AttnArgs& a, int n_blk, cudaStream_t st);
size_t attention_smem_bytes(int qmax, int hpk, int hd, int ctx_cap);
int attention_chunks(int ctx_cap);
int attention_chunk_len();

cudaError_t launch_quantize_weight(const QuantWArgs& a, cudaStream_t st);
cudaError_t launch_lcg_fill(float* out, unsigned long long seed, unsigned long long offset, long long count,
                            float scale, cudaStream_t st);
cudaError_t launch_repack_ref(const uint8_t* ref_codes, const float* ref_scales, int rows, int cols, int g,
                              uint8_t* codes, float* scales, int n_pad, int n_chunks, int gp, int G, int row_off,
                              int row_stride, cudaStream_t st);

cudaError_t launch_control(int op, const SeqState& s, int j, cudaStream_t st);
int tp_allreduce_nccl(float* p, int64_t count, void* comm, cudaStream_t st);
int tp_argmax_reduce(const qs_tp_t* tp, int T, int32_t* argmax, cudaStream_t st);
cudaError_t launch_add_rows(float* x, const float* y, int n, cudaStream_t st);
cudaError_t launch_hadamard_rows(float* x, long long rows, int cols, cudaStream_t st);
}  // namespace qs

using namespace qs;

namespace qs {
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && e[0]) ? atoi(e) : dflt;
}
// L2 look-ahead window of the forward's weight stream, MB (QS_PF_WINDOW_MB; 0 = off)
int pf_window_mb() {
  static int w = env_int("QS_PF_WINDOW_MB", 0);  // measured: a 32-96 MB window slows the step
  return w;
}
int pf_own_enabled() {
  static int on = env_int("QS_PF_OWN", 0);
  return on;
}
bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("QS_NO_PDL");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}
}  // namespace qs

static unsigned long long* g_dbg = nullptr;
static int g_dbg_want = 0, g_dbg_seen = 0;
namespace {

// qs_ktrace_*: per-launch slots of the device timeline (KTrace in qs_common.cuh)
struct KTraceHost {
  unsigned long long* buf = nullptr;
  int cap = 0;
  std::vector<int32_t> tags;
} g_kt;

KTrace next_trace(int32_t tag) {
  if (g_kt.buf == nullptr || (int)g_kt.tags.size() >= g_kt.cap) return KTrace{nullptr, 0};
  g_kt.tags.push_back(tag);
  return KTrace{g_kt.buf, (int)g_kt.tags.size() - 1};
}

constexpr int kMaxT = 64;
static_assert(kMaxT <= kLeafRows, "emit leaf rows cover every token of a forward");
constexpr int kGbarOffset = 4096;  // emit counters live past every per-tile counter
constexpr int kEmitCnt = 8 + 1024;  // [0] arrive, [1] depart, [8 + q] per silu group

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// Optional per-linear event ring: when enabled, every linear launch issued by
// qs_forward is bracketed by two events (captured as event nodes inside a CUDA
// graph), so bench.py can attribute device time to the dominant kernel.
struct Prof {
  bool on = false;
  int cap = 0, n = 0;
  cudaEvent_t* ev = nullptr;
  int32_t* tag = nullptr;
} g_prof;

void prof_mark(cudaStream_t st, int32_t tag, bool begin) {
  if (!g_prof.on) return;
  const int i = g_prof.n;
  if (i >= g_prof.cap) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  cudaEventRecordWithFlags(g_prof.ev[i], st, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0);
  if (begin) g_prof.tag[i / 2] = tag;
  g_prof.n = i + 1;
}

}  // namespace
namespace {

// Launch a linear whose operand comes from a.pk: a separate act_pack launch
// overlapped via PDL, then the linear.
thread_local int g_launches = 0;  // kernels enqueued by the last qs_forward (qs_forward_launches)
thread_local int g_rotate = 0;    // qs_model_t.hadamard of the forward being enqueued (pack_args / set_emit)

cudaError_t launch_linear_packed(int L, LinearArgs& a, cudaStream_t st, int32_t tag = -1, bool pack = true) {
  const int32_t mode_bits = 16 * (L == 1 ? 1 : 0);
  cudaError_t e = cudaSuccess;
  if (pack) {  // else the operand was emitted by the previous linear's epilogue
    prof_mark(st, mode_bits + 5, true);  // kind 5: operand pack
    a.pk.kt = next_trace(mode_bits + 5);
    e = launch_act_pack(L, a.pk, st);
    prof_mark(st, 0, false);
    if (e != cudaSuccess) return e;
    ++g_launches;
  }
  ++g_launches;
  a.kt = next_trace(tag >= 0 ? tag : mode_bits + 15);
  // qs_debug_select(j): the j-th linear launch enqueued after the call records its CTA
  // timeline into the qs_debug_timeline buffer (QS_LIN_TIMELINE builds only)
  if (g_dbg_want > 0 && ++g_dbg_seen == g_dbg_want) a.dbg = g_dbg;
  if (tag >= 0) prof_mark(st, tag, true);
  e = launch_linear(L, a, st);
  if (tag >= 0) prof_mark(st, 0, false);
  return e;
}

int status(cudaError_t e) {
  if (e == cudaSuccess) return QS_OK;
  fprintf(stderr, "[qspec_b200] CUDA error: %s\n", cudaGetErrorString(e));
  return QS_ERR_CUDA;
}

void fill_geometry(int n, int k, int g, qs_qweight_t* w) {
  w->n = n;
  w->k = k;
  w->g = g;
  w->n_pad = round_up(n, kTileN);
  w->n_tiles = w->n_pad / kTileN;
  w->G = k / g;
  w->gp = round_up(g, kChunkK);
  w->cpg = w->gp / kChunkK;
  w->n_chunks = w->G * w->cpg;
}

PackArgs pack_args(const qs_qweight_t& w, const float* x, int ldx, int T, const qs_workspace_t* ws, int L) {
  PackArgs p{};
  p.rotate = g_rotate;
  p.x = x;
  p.ldx = ldx;
  p.T = T;
  p.K = w.k;
  p.g = w.g;
  p.gp = w.gp;
  p.G = w.G;
  p.n_chunks = w.n_chunks;
  p.r_pad = img_rows(linear_tmax_bucket(T, L), L);
  p.a_ld = round_up(T, 8);
  p.img = ws->img;
  p.ascale = ws->ascale;
  p.acorr = reinterpret_cast<int32_t*>(ws->ascale + (size_t)w.n_chunks * p.a_ld);
  return p;
}

// CTAs of one linear launch: every SM, unless that leaves fewer than QS_MIN_UNITS (tile,
// chunk) units per CTA -- a small linear (o_proj: 1024 units) spread over 148 CTAs splits
// each tile 4-5 ways and its stream-K fixups dominate.  Depends only on (N, K), never on
// T, so the reduction order stays batch-invariant.
int linear_ctas(int units, int n_tiles) {
  static int min_units = env_int("QS_MIN_UNITS", 0);
  int P = units < num_sms() ? units : num_sms();
  if (min_units > 0 && units / min_units < P) {
    P = units / min_units;
    if (P < n_tiles && n_tiles <= num_sms()) P = n_tiles;
    if (P < 1) P = 1;
  }
  return P;
}
LinearArgs linear_args(const qs_qweight_t& w, int T, int L, const qs_workspace_t* ws, int op, float* out,
                       int ldo) {
  LinearArgs a{};
  a.codes = w.codes;
  a.wscale = w.scales;
  a.act = ws->img;
  a.ascale = ws->ascale;
  a.acorr = reinterpret_cast<const int32_t*>(ws->ascale + (size_t)w.n_chunks * round_up(T, 8));
  a.n = w.n;
  a.n_pad = w.n_pad;
  a.n_tiles = w.n_tiles;
  a.G = w.G;
  a.cpg = w.cpg;
  a.n_chunks = w.n_chunks;
  a.T = T;
  a.r_pad = img_rows(linear_tmax_bucket(T, L), L);
  a.a_ld = round_up(T, 8);
  const int U = w.n_tiles * w.n_chunks;
  a.n_cta = linear_ctas(U, w.n_tiles);
  a.part = ws->part;
  a.counters = ws->counters;
  a.op = op;
  a.out = out;
  a.ldo = ldo;
  a.arg_val = ws->arg_val;
  a.arg_idx = ws->arg_idx;
  a.pf_n = 0;
  a.pf_own = pf_own_enabled();
  return a;
}

// The forward's weight stream in launch order (codes then scales of every linear).
// Linear j prefetches the stream bytes [E_{j-1} + W, E_j + W) (mod the stream length:
// the next forward of a decode loop streams the same weights), so every byte is
// requested once, W bytes before the linear that consumes it starts.
struct WeightStream {
  std::vector<const uint8_t*> ptr;
  std::vector<size_t> len;
  std::vector<size_t> lin_end;  // stream offset after each linear
  size_t total = 0;
  void add_linear(const qs_qweight_t& w) {
    const size_t cb = (size_t)w.n_tiles * w.n_chunks * kChunkBytes, sb = (size_t)w.n_tiles * w.n_chunks * kTileN * 4;
    ptr.push_back(w.codes);
    len.push_back(cb);
    ptr.push_back(reinterpret_cast<const uint8_t*>(w.scales));
    len.push_back(sb);
    total += cb + sb;
    lin_end.push_back(total);
  }
  // append the pieces of stream range [A, B) (A, B may exceed total: wrap) to a.pf_*
  void ranges(LinearArgs& a, size_t A, size_t B) const {
    a.pf_n = 0;
    if (total == 0 || B <= A) return;
    if (B - A > total) A = B - total;
    while (A < B && a.pf_n < kMaxPf) {
      const size_t a0 = A % total;
      size_t off = 0, i = 0;
      while (i < len.size() && off + len[i] <= a0) off += len[i++];
      const size_t take = std::min(B - A, off + len[i] - a0);
      a.pf_ptr[a.pf_n] = ptr[i] + (a0 - off);
      a.pf_len[a.pf_n] = (uint32_t)take;
      ++a.pf_n;
      A += take;
    }
  }
  void window(LinearArgs& a, int j) const {
    const size_t W = (size_t)pf_window_mb() << 20;
    if (W == 0) return;
    const size_t prev = j == 0 ? 0 : lin_end[j - 1];
    ranges(a, prev + W, lin_end[j] + W);
  }
};

int check_weight(const qs_qweight_t* w) {
  if (!w || !w->codes || !w->scales) return QS_ERR_SHAPE;
  if (w->g < 1 || w->k % w->g != 0) return QS_ERR_CONFIG;
  return QS_OK;
}

int run_linear(const qs_qweight_t* w, const float* x, int T, float* y, const qs_workspace_t* ws, int L, int op,
               int32_t* dump, cudaStream_t st) {
  int rc = check_weight(w);
  if (rc) return rc;
  if (T < 1 || T > kMaxT || !x || !ws) return QS_ERR_SHAPE;
  LinearArgs a = linear_args(*w, T, L, ws, op, y, w->n);
  a.pk = pack_args(*w, x, w->k, T, ws, L);
  a.dump = dump;
  return status(launch_linear_packed(L, a, st));
}

SeqState seq_state(const qs_seq_t* s) {
  SeqState q;
  q.pending = s->pending;
  q.committed = s->committed;
  q.n_out = s->n_out;
  q.done = s->done;
  q.finish = s->finish;
  q.max_new = s->max_new;
  q.g_eff = s->g_eff;
  q.drafted = s->drafted;
  q.out_tokens = s->out_tokens;
  q.n_drafted = s->n_drafted;
  q.n_accepted = s->n_accepted;
  q.n_cycles = s->n_cycles;
  q.dropped = s->dropped;
  q.trace = s->trace;
  q.trace_tok = s->trace_tok;
  q.out_cap = s->out_cap;
  q.trace_cap = s->trace_cap;
  q.B = s->B;
  q.gamma = s->gamma;
  q.eos = s->eos;
  q.max_seq = s->max_seq;
  q.tok = s->tok;
  q.pos = s->pos;
  q.slot = s->slot;
  q.argmax = s->argmax;
  return q;
}

}  // namespace

extern "C" {

int qs_profile_enable(int32_t max_launches) {
  // events are never destroyed: graphs captured while profiling keep referencing them
  g_prof.on = max_launches > 0;
  if (!g_prof.on) return QS_OK;  // keep the recorded ring readable
  g_prof.n = 0;
  if (2 * max_launches <= g_prof.cap) return QS_OK;
  g_prof.cap = 2 * max_launches;
  g_prof.ev = new cudaEvent_t[g_prof.cap];
  g_prof.tag = new int32_t[max_launches];
  for (int i = 0; i < g_prof.cap; ++i)
    if (cudaEventCreate(&g_prof.ev[i]) != cudaSuccess) return QS_ERR_CUDA;
  return QS_OK;
}

int qs_ktrace_enable(uint64_t* buf, int32_t cap) {
  g_kt.buf = reinterpret_cast<unsigned long long*>(buf);
  g_kt.cap = buf ? cap : 0;
  g_kt.tags.clear();
  return QS_OK;
}

int qs_ktrace_read(int32_t* tags, int32_t max_out, int32_t* n_out) {
  const int n = (int)g_kt.tags.size() < max_out ? (int)g_kt.tags.size() : max_out;
  for (int i = 0; i < n; ++i) tags[i] = g_kt.tags[i];
  *n_out = n;
  return QS_OK;
}

int qs_profile_reset(void) {
  g_prof.n = 0;
  return QS_OK;
}

int qs_profile_read(float* ms, int32_t* tags, int32_t max_out, int32_t* n_out) {
  const int n = g_prof.n / 2 < max_out ? g_prof.n / 2 : max_out;
  for (int i = 0; i < n; ++i) {
    if (cudaEventSynchronize(g_prof.ev[2 * i + 1]) != cudaSuccess) return QS_ERR_CUDA;
    if (cudaEventElapsedTime(&ms[i], g_prof.ev[2 * i], g_prof.ev[2 * i + 1]) != cudaSuccess) return QS_ERR_CUDA;
    tags[i] = g_prof.tag[i];
  }
  *n_out = n;
  return QS_OK;
}

const char* qs_version(void) { return "qspec_b200 0.1 (sm_100a tcgen05 kind::i8)"; }

int qs_num_sms(int32_t* out) {
  *out = num_sms();
  return QS_OK;
}

int qs_linear_max_tokens(void) { return kMaxT; }
int qs_attention_chunk_len(void) { return attention_chunk_len(); }

int qs_qweight_geometry(int32_t n, int32_t k, int32_t g, qs_qweight_t* out) {
  if (n < 1 || k < 1 || g < 1 || k % g != 0) return QS_ERR_CONFIG;
  fill_geometry(n, k, g, out);
  out->codes = nullptr;
  out->scales = nullptr;
  return QS_OK;
}

int qs_workspace_size(const qs_model_t* m, int32_t t_max, qs_workspace_sizes_t* out) {
  if (t_max < 1 || t_max > kMaxT) return QS_ERR_SHAPE;
  const int hd = m->d_model / m->n_heads;
  qs_qweight_t wd, wf, wl;
  fill_geometry(m->d_model, m->d_model, m->group_size, &wd);
  fill_geometry(m->d_model, m->d_ff, m->group_size, &wf);
  fill_geometry(m->vocab, m->d_model, m->group_size, &wl);
  const int chunks = wd.n_chunks > wf.n_chunks ? wd.n_chunks : wf.n_chunks;
  int tiles = wl.n_tiles;
  const int t_ff = round_up(2 * m->d_ff, kTileN) / kTileN;
  const int t_qkv = round_up((m->n_heads + 2 * m->n_kv_heads) * hd, kTileN) / kTileN;
  if (t_ff > tiles) tiles = t_ff;
  if (t_qkv > tiles) tiles = t_qkv;
  out->x = (size_t)t_max * m->d_model * 4;
  out->h = (size_t)t_max * m->d_ff * 4;
  out->attn = (size_t)t_max * m->d_model * 4;
  out->q = (size_t)t_max * m->n_heads * hd * 4;
  out->img = 2 * (size_t)chunks * img_rows(kMaxT, 3) * 128;  // two operand slots (emit double buffer)
  out->ascale = 2 * (size_t)chunks * kMaxT * 4 * 5;  // two slots of ascale + acorr [n_chunks][a_ld][4]
  out->part = (size_t)(num_sms() + tiles) * kMaxT * kTileN * 4;
  // per-tile counters | emit counters [kGbarOffset, +8 + 1024) | 2 x emit leaf sums [64][128]
  out->counters = (size_t)(kGbarOffset + kEmitCnt + 2 * kLeafRows * kLeafLd) * 4;
  if (tiles + 1 > kGbarOffset) return QS_ERR_SHAPE;
  out->arg_val = (size_t)wl.n_tiles * kMaxT * 4;
  out->arg_idx = (size_t)wl.n_tiles * kMaxT * 4;
  const int cmax = attention_chunks(m->rope_len > 0 ? m->rope_len : 4096);
  out->att_o = (size_t)t_max * m->n_heads * cmax * hd * 4;
  out->att_ml = (size_t)t_max * m->n_heads * cmax * 8;
  return QS_OK;
}

int qs_init_weight(uint64_t seed, uint64_t draw_offset, float scale, int32_t rows, int32_t cols, int32_t g,
                   uint8_t* codes, float* scales, int32_t n_pad, int32_t row_off, int32_t row_stride,
                   uint8_t* ref_codes, float* ref_scales, void* stream) {
  if (g < 1 || cols % g != 0) return QS_ERR_CONFIG;
  qs_qweight_t geo;
  fill_geometry(n_pad, cols, g, &geo);
  QuantWArgs a{};
  a.src = nullptr;
  a.seed = seed;
  a.offset = draw_offset;
  a.scale = scale;
  a.rows = rows;
  a.cols = cols;
  a.g = g;
  a.codes = codes;
  a.scales = scales;
  a.n_pad = n_pad;
  a.n_chunks = geo.n_chunks;
  a.gp = geo.gp;
  a.G = geo.G;
  a.row_off = row_off;
  a.row_stride = row_stride;
  a.ref_codes = ref_codes;
  a.ref_scales = ref_scales;
  return status(launch_quantize_weight(a, (cudaStream_t)stream));
}

int qs_quantize_weight(const float* w, int32_t rows, int32_t cols, int32_t g, uint8_t* codes, float* scales,
                       int32_t n_pad, int32_t row_off, int32_t row_stride, uint8_t* ref_codes, float* ref_scales,
                       void* stream) {
  if (g < 1 || cols % g != 0) return QS_ERR_CONFIG;
  if (!w) return QS_ERR_SHAPE;
  qs_qweight_t geo;
  fill_geometry(n_pad, cols, g, &geo);
  QuantWArgs a{};
  a.src = w;
  a.rows = rows;
  a.cols = cols;
  a.g = g;
  a.codes = codes;
  a.scales = scales;
  a.n_pad = n_pad;
  a.n_chunks = geo.n_chunks;
  a.gp = geo.gp;
  a.G = geo.G;
  a.row_off = row_off;
  a.row_stride = row_stride;
  a.ref_codes = ref_codes;
  a.ref_scales = ref_scales;
  return status(launch_quantize_weight(a, (cudaStream_t)stream));
}

int qs_lcg_fill(float* out, uint64_t seed, uint64_t draw_offset, int64_t count, float scale, void* stream) {
  if (count <= 0) return QS_OK;
  return status(launch_lcg_fill(out, seed, draw_offset, count, scale, (cudaStream_t)stream));
}

int qs_repack_ref(const uint8_t* ref_codes, const float* ref_scales, int32_t rows, int32_t cols, int32_t g,
                  uint8_t* codes, float* scales, int32_t n_pad, int32_t row_off, int32_t row_stride, void* stream) {
  if (g < 1 || cols % g != 0) return QS_ERR_CONFIG;
  qs_qweight_t geo;
  fill_geometry(n_pad, cols, g, &geo);
  return status(launch_repack_ref(ref_codes, ref_scales, rows, cols, g, codes, scales, n_pad, geo.n_chunks, geo.gp,
                                  geo.G, row_off, row_stride, (cudaStream_t)stream));
}

int qs_hadamard_rows(float* x, int64_t rows, int32_t cols, void* stream) {
  if (!x || rows < 0 || cols % 128 != 0) return QS_ERR_SHAPE;
  if (rows == 0) return QS_OK;
  return status(launch_hadamard_rows(x, rows, cols, (cudaStream_t)stream));
}

int qs_act_quant(const float* x, int32_t T, int32_t K, int32_t g, int8_t* codes, float* scales, float* fq,
                 void* stream) {
  if (g < 1 || K % g != 0) return QS_ERR_CONFIG;
  if (T < 1 || !x) return QS_ERR_SHAPE;
  PackArgs p{};
  p.x = x;
  p.ldx = K;
  p.T = T;
  p.K = K;
  p.g = g;
  p.gp = round_up(g, kChunkK);
  p.G = K / g;
  p.codes_out = codes;
  p.scales_out = scales;
  p.fq_out = fq;
  return status(launch_act_pack(1, p, (cudaStream_t)stream));
}

int qs_rmsnorm(const float* x, const float* w, int32_t T, int32_t K, float eps, float* y, void* stream) {
  if (T < 1 || K < 1 || !x || !w || !y) return QS_ERR_SHAPE;
  if (!(eps > 0.f)) return QS_ERR_SHAPE;
  int g = K < 128 ? K : 128;  // any group size works: only the normalised row is written
  while (K % g) --g;
  PackArgs p{};
  p.x = x;
  p.ldx = K;
  p.T = T;
  p.K = K;
  p.g = g;
  p.gp = round_up(g, kChunkK);
  p.G = K / g;
  p.rms_w = w;
  p.eps = eps;
  p.y_out = y;
  return status(launch_act_pack(1, p, (cudaStream_t)stream));
}

int qs_w4a4_linear(const qs_qweight_t* w, const float* x, int32_t T, float* y, const qs_workspace_t* ws,
                   void* stream) {
  return run_linear(w, x, T, y, ws, 1, kOpStore, nullptr, (cudaStream_t)stream);
}

int qs_w4a16_linear(const qs_qweight_t* w, const float* x, int32_t T, float* y, const qs_workspace_t* ws,
                    void* stream) {
  return run_linear(w, x, T, y, ws, 3, kOpStore, nullptr, (cudaStream_t)stream);
}

int qs_debug_timeline(uint64_t* buf) {
  g_dbg = reinterpret_cast<unsigned long long*>(buf);
  return QS_OK;
}

int qs_debug_select(int32_t launch_index) {
  g_dbg_want = launch_index;
  g_dbg_seen = 0;
  return QS_OK;
}

int qs_linear_prepacked(const qs_qweight_t* w, int32_t T, int32_t mode, float* y, const qs_workspace_t* ws,
                        void* stream) {
  int rc = check_weight(w);
  if (rc) return rc;
  if (T < 1 || T > kMaxT || !ws) return QS_ERR_SHAPE;
  const int L = mode == QS_MODE_LOW ? 1 : 3;
  LinearArgs a = linear_args(*w, T, L, ws, kOpStore, y, w->n);
  a.dbg = g_dbg;
  return status(launch_linear(L, a, (cudaStream_t)stream));
}

int qs_linear_group_dots(const qs_qweight_t* w, const float* x, int32_t T, int32_t mode, int32_t* dots,
                         const qs_workspace_t* ws, void* stream) {
  return run_linear(w, x, T, nullptr, ws, mode == QS_MODE_LOW ? 1 : 3, kOpDump, dots, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
struct TpHooks {
  int world;
  qs_allreduce_fn fn;
  void* user;
  const qs_tp_t* tp2;  // qs_forward_tp2: NCCL / gather hooks + vocab-split lm_head
};
// Operand slots: the image + scales a linear reads, and the one its epilogue emits for
// the NEXT linear, must differ (some CTAs still stream their operand while finished
// owners emit), so the workspace holds two and the forward alternates between them.
struct Slot {
  uint8_t* img;
  float* ascale;
};
void use_slot(LinearArgs& a, const qs_qweight_t& w, const Slot& sl) {
  a.act = sl.img;
  a.ascale = sl.ascale;
  a.acorr = reinterpret_cast<const int32_t*>(sl.ascale + (size_t)w.n_chunks * a.a_ld);
  a.pk.img = sl.img;
  a.pk.ascale = sl.ascale;
  a.pk.acorr = reinterpret_cast<int32_t*>(sl.ascale + (size_t)w.n_chunks * a.pk.a_ld);
}
void set_emit(LinearArgs& a, int kind, const qs_qweight_t& next, const Slot& sl, const float* rms_w, float eps,
              int n, const qs_workspace_t* ws, int leaf_buf = 0) {
  a.emit = kind;
  a.e_img = sl.img;
  a.e_ascale = sl.ascale;
  a.e_acorr = reinterpret_cast<int32_t*>(sl.ascale + (size_t)next.n_chunks * a.a_ld);
  a.e_rms_w = rms_w;
  a.e_eps = eps;
  a.e_n = n;
  a.e_cnt = ws->counters + kGbarOffset;
  a.e_rotate = g_rotate;
  unsigned* leaves = reinterpret_cast<unsigned*>(ws->counters + kGbarOffset + kEmitCnt);
  a.e_leaf = leaves + leaf_buf * kLeafRows * kLeafLd;
  a.e_leaf_clr = leaves + (leaf_buf ^ 1) * kLeafRows * kLeafLd;
}
int g_emit = -1;  // fused next-operand emits (mask: 1 silu, 2 rmsnorm): -1 = QS_EMIT env (default 3)
int emit_mask() {
  if (g_emit < 0) g_emit = env_int("QS_EMIT", 3) & 3;
  return g_emit;
}

int forward_impl(const qs_model_t* m, const qs_batch_t* b, int32_t mode, const qs_workspace_t* ws, float* logits,
                 int32_t* argmax, cudaStream_t st, const TpHooks* tp) {
  const int T = b->T;
  if (T < 1 || T > kMaxT) return QS_ERR_SHAPE;
  const int L = mode == QS_MODE_LOW ? 1 : 3;
  const int world = tp ? tp->world : 1;
  const int d = m->d_model, H = m->n_heads, KV = m->n_kv_heads, hd = d / (H * world), ff = m->d_ff;
  g_launches = 0;
  g_rotate = m->hadamard ? 1 : 0;
  struct RotReset {
    ~RotReset() { g_rotate = 0; }
  } rot_reset;  // the standalone linear API never rotates
  if (m->hadamard && m->group_size != 128) return QS_ERR_CONFIG;
  if (m->page < 1 || (m->page & (m->page - 1)) != 0) return QS_ERR_CONFIG;  // KV page: a power of two
  // tensor parallel: o_proj / down_proj are row-split, so their outputs are partial
  // sums -> store into ws->attn, all-reduce (caller's hook, e.g. NCCL on this
  // stream), then add into the residual stream
  const int res_op = tp ? kOpStore : kOpResidual;
  float* res_out = tp ? ws->attn : ws->x;
  auto reduce_into_x = [&]() -> int {
    int rc = (tp->tp2 && tp->tp2->nccl_comm) ? tp_allreduce_nccl(ws->attn, (int64_t)T * d, tp->tp2->nccl_comm, st)
                                            : tp->fn(ws->attn, (int64_t)T * d, st, tp->user);
    if (rc != 0) return QS_ERR_CUDA;
    ++g_launches;
    return status(launch_add_rows(ws->x, ws->attn, T * d, st));
  };
  const int hpk = H / KV;
  if (b->blk_qmax * hpk > 64 || hd % 4 != 0) return QS_ERR_SHAPE;
  if (b->ctx_cap > m->rope_len) return QS_ERR_OVERFLOW;
  const int att_cmax = attention_chunks(m->rope_len);
  if (attention_smem_bytes(b->blk_qmax, hpk, hd, b->ctx_cap) > 200 * 1024) return QS_ERR_SHAPE;
  // operand slots (qs_workspace_size allots two)
  Slot slot[2];
  {
    qs_qweight_t wd, wf;
    fill_geometry(d, d, m->group_size, &wd);
    fill_geometry(d, ff, m->group_size, &wf);
    const int chunks = wd.n_chunks > wf.n_chunks ? wd.n_chunks : wf.n_chunks;
    slot[0] = Slot{ws->img, ws->ascale};
    slot[1] = Slot{ws->img + (size_t)chunks * img_rows(kMaxT, 3) * 128, ws->ascale + (size_t)chunks * kMaxT * 5};
  }
  // fused next-operand emits (LinearArgs::emit): not under TP (the residual is added after
  // the all-reduce), g = 128 only (a tile is a group), d = 128 * 2^k (a tile is a numpy
  // pairwise leaf) and every CTA owning at most one residual tile
  // Measured (bench.py, B=1 / B=16): the emits win for small forwards (AR 2.38 -> 2.33 ms)
  // and lose at T=64 (the 32 o/down owners quantise 64 tokens each while the act_pack
  // kernel spreads them over 512 CTAs and overlaps the next linear's weight prefetch), so
  // they run for T <= QS_EMIT_TMAX (default 16) only.
  static const int emit_tmax = env_int("QS_EMIT_TMAX", 16);
  const bool emit_ok = !tp && T <= emit_tmax && m->group_size == 128 && d % 128 == 0;
  const int d_tiles = d / 128;
  // (o_proj / down_proj have d/128 tiles of >= d/128 chunks: n_cta = min(units, #SMs) >= n_tiles
  // iff n_tiles <= #SMs, and then no CTA's unit range holds two tile starts)
  const bool emit_rms =
      emit_ok && (emit_mask() & 2) && (d_tiles & (d_tiles - 1)) == 0 && d_tiles <= 128 && d_tiles <= num_sms();
  const bool emit_silu = emit_ok && (emit_mask() & 1) && ff % 128 == 0 && ff / 128 <= kEmitCnt - 8;
  cudaError_t e;
  WeightStream ws_stream;
  for (int li = 0; li < m->n_layers; ++li) {
    ws_stream.add_linear(m->layers[li].qkv);
    ws_stream.add_linear(m->layers[li].o);
    ws_stream.add_linear(m->layers[li].gate_up);
    ws_stream.add_linear(m->layers[li].down);
  }
  ws_stream.add_linear(m->lm_head);
  int lin_j = 0;
  const int s0 = 0;            // slot read by qkv / gate_up / lm_head
  bool qkv_ready = false;      // qkv's operand already emitted by the previous down_proj
  auto qkv_args = [&](int li) {
    const qs_layer_t& ly = m->layers[li];
    // q|k|v projection; operand = rmsnorm(x) (+ embedding gather on layer 0), fused
    // pre-phase; epilogue: RoPE + KV write (model.py:302-309, 339-340)
    LinearArgs a = linear_args(ly.qkv, T, L, ws, kOpQkvRope, ws->q, H * hd);
    a.pk = pack_args(ly.qkv, ws->x, d, T, ws, L);
    a.pk.rms_w = ly.attn_norm;
    a.pk.eps = m->norm_eps;
    if (li == 0) {
      a.pk.gather_ids = b->tokens;
      a.pk.emb = m->tok_emb;
      a.pk.x_out = ws->x;
    }
    use_slot(a, ly.qkv, slot[s0]);
    a.pos = b->positions;
    a.slot = b->slots;
    a.rope_cos = m->rope_cos;
    a.rope_sin = m->rope_sin;
    a.hd = hd;
    a.n_q = H * hd;
    a.n_k = KV * hd;
    a.n_kv_heads = KV;
    a.kcache = ly.k_cache;
    a.vcache = ly.v_cache;
    a.block_table = m->block_table;
    a.bt_ld = m->bt_ld;
    a.page = m->page;
    a.page_shift = __builtin_ctz((unsigned)m->page);
    return a;
  };
  const qs_tp_t* tp2 = tp ? tp->tp2 : nullptr;
  auto head_args = [&]() {
    // final norm + lm_head + argmax (model.py:342-344, numerics.py:81-86)
    LinearArgs a = linear_args(m->lm_head, T, L, ws, kOpLogits, logits, m->vocab);
    a.pk = pack_args(m->lm_head, ws->x, d, T, ws, L);
    a.pk.rms_w = m->final_norm;
    a.pk.eps = m->norm_eps;
    use_slot(a, m->lm_head, slot[s0]);
    a.argmax_out = argmax;
    if (tp2) {  // vocab-split head: per-rank (max, index) records, gathered and reduced below
      a.arg_rec = reinterpret_cast<int2*>(tp2->scratch);
      a.arg_off = tp2->vocab_off;
    }
    return a;
  };
  for (int li = 0; li < m->n_layers; ++li) {
    const qs_layer_t& ly = m->layers[li];
    {
      LinearArgs a = qkv_args(li);
      ws_stream.window(a, lin_j++);
      if ((e = launch_linear_packed(L, a, st, mode * 16 + 0, !qkv_ready)) != cudaSuccess) return status(e);
    }
    // attention (model.py:293-330), split-KV partials
    AttnArgs at{};
    at.q = ws->q;
    at.ldq = H * hd;
    at.kcache = ly.k_cache;
    at.vcache = ly.v_cache;
    at.block_table = m->block_table;
    at.bt_ld = m->bt_ld;
    at.page = m->page;
    at.pos = b->positions;
    at.slot = b->slots;
    at.blk_tok0 = b->blk_tok0;
    at.blk_ntok = b->blk_ntok;
    at.H = H;
    at.KV = KV;
    at.hd = hd;
    at.hpk = hpk;
    at.inv_sqrt_hd = 1.0f / sqrtf((float)hd);
    at.qmax = b->blk_qmax;
    at.ctx_cap = b->ctx_cap;
    at.out = ws->attn;
    at.ldo = d;
    at.part_o = ws->att_o;
    at.part_ml = ws->att_ml;
    at.cmax = att_cmax;
    prof_mark(st, mode * 16 + 6, true);  // kind 6: attention
    at.kt = next_trace(mode * 16 + 6);
    if ((e = launch_attention(at, b->n_blk, st)) != cudaSuccess) return status(e);
    ++g_launches;
    prof_mark(st, 0, false);
    // o_proj + residual (model.py:332); its operand pack merges the attention chunks;
    // its epilogue emits gate_up's operand rmsnorm(x) * ffn_norm (model.py:333)
    LinearArgs ao = linear_args(ly.o, T, L, ws, res_op, res_out, d);
    ao.pk = pack_args(ly.o, ws->attn, ly.o.k, T, ws, L);
    ao.pk.att_o = ws->att_o;
    ao.pk.att_ml = ws->att_ml;
    ao.pk.att_pos = b->positions;
    ao.pk.att_hd = hd;
    ao.pk.att_cmax = att_cmax;
    ao.pk.att_chunk = attention_chunk_len();
    use_slot(ao, ly.o, slot[s0 ^ 1]);
    if (emit_rms) set_emit(ao, kEmitRms, ly.gate_up, slot[s0], ly.ffn_norm, m->norm_eps, d, ws);
    ws_stream.window(ao, lin_j++);
    // gate|up on rmsnorm(x), epilogue silu(gate) * up (model.py:333-335), then down_proj's
    // operand groups
    LinearArgs agu = linear_args(ly.gate_up, T, L, ws, kOpSiluMul, ws->h, ff);
    agu.pk = pack_args(ly.gate_up, ws->x, d, T, ws, L);
    agu.pk.rms_w = ly.ffn_norm;
    agu.pk.eps = m->norm_eps;
    use_slot(agu, ly.gate_up, slot[s0]);
    if (emit_silu) set_emit(agu, kEmitSilu, ly.down, slot[s0 ^ 1], nullptr, 0.f, ff, ws);
    ws_stream.window(agu, lin_j++);
    // down_proj + residual (model.py:336); epilogue emits the next qkv's (or lm_head's)
    // operand rmsnorm(x) * attn_norm / final_norm (model.py:302, 342)
    LinearArgs adn = linear_args(ly.down, T, L, ws, res_op, res_out, d);
    adn.pk = pack_args(ly.down, ws->h, ff, T, ws, L);
    use_slot(adn, ly.down, slot[s0 ^ 1]);
    const bool last = li + 1 == m->n_layers;
    if (emit_rms)
      set_emit(adn, kEmitRms, last ? m->lm_head : m->layers[li + 1].qkv, slot[s0],
               last ? m->final_norm : m->layers[li + 1].attn_norm, m->norm_eps, d, ws, 1);
    ws_stream.window(adn, lin_j++);
    if ((e = launch_linear_packed(L, ao, st, mode * 16 + 1)) != cudaSuccess) return status(e);
    if (tp) {
      const int rc = reduce_into_x();
      if (rc) return rc;
    }
    if ((e = launch_linear_packed(L, agu, st, mode * 16 + 2, !emit_rms)) != cudaSuccess) return status(e);
    if ((e = launch_linear_packed(L, adn, st, mode * 16 + 3, !emit_silu)) != cudaSuccess) return status(e);
    if (tp) {
      const int rc = reduce_into_x();
      if (rc) return rc;
    }
    qkv_ready = emit_rms;
  }
  LinearArgs a = head_args();
  ws_stream.window(a, lin_j++);
  e = launch_linear_packed(L, a, st, mode * 16 + 4, !qkv_ready);
  if (e != cudaSuccess || !tp2) return status(e);
  return tp_argmax_reduce(tp2, T, argmax, st);
}
}  // namespace

extern "C" {
int qs_forward(const qs_model_t* m, const qs_batch_t* b, int32_t mode, const qs_workspace_t* ws, float* logits,
               int32_t* argmax, void* stream) {
  return forward_impl(m, b, mode, ws, logits, argmax, (cudaStream_t)stream, nullptr);
}

int qs_forward_launches(void) { return g_launches; }

int qs_forward_tp2(const qs_model_t* m, const qs_batch_t* b, int32_t mode, const qs_workspace_t* ws, float* logits,
                   int32_t* argmax, const qs_tp_t* tp, void* stream) {
  if (!tp || tp->world < 1 || tp->rank < 0 || tp->rank >= tp->world || !tp->scratch) return QS_ERR_CONFIG;
  if (!tp->nccl_comm && (!tp->allreduce || !tp->allgather)) return QS_ERR_CONFIG;
  if (m->n_heads % m->n_kv_heads != 0 || m->d_model % (m->n_heads * tp->world) != 0) return QS_ERR_CONFIG;
  TpHooks h{tp->world, tp->allreduce, tp->user, tp};
  return forward_impl(m, b, mode, ws, logits, argmax, (cudaStream_t)stream, &h);
}

int qs_set_emit(int32_t mask) {
  g_emit = mask & 3;
  return QS_OK;
}

int qs_forward_tp(const qs_model_t* m, const qs_batch_t* b, int32_t mode, const qs_workspace_t* ws, float* logits,
                  int32_t* argmax, int32_t world, qs_allreduce_fn allreduce, void* user, void* stream) {
  if (world < 1 || !allreduce || m->n_heads % m->n_kv_heads != 0) return QS_ERR_CONFIG;
  if (m->d_model % (m->n_heads * world) != 0) return QS_ERR_CONFIG;
  TpHooks tp{world, allreduce, user, nullptr};
  return forward_impl(m, b, mode, ws, logits, argmax, (cudaStream_t)stream, &tp);
}

}  // extern "C"

extern "C" {
int qs_draft_prep(const qs_seq_t* s, int32_t step, void* stream) {
  return status(launch_control(0, seq_state(s), step, (cudaStream_t)stream));
}
int qs_verify_prep(const qs_seq_t* s, void* stream) {
  return status(launch_control(1, seq_state(s), 0, (cudaStream_t)stream));
}
int qs_accept(const qs_seq_t* s, void* stream) {
  return status(launch_control(2, seq_state(s), 0, (cudaStream_t)stream));
}
int qs_ar_prep(const qs_seq_t* s, void* stream) {
  return status(launch_control(3, seq_state(s), 0, (cudaStream_t)stream));
}
int qs_ar_commit(const qs_seq_t* s, void* stream) {
  return status(launch_control(4, seq_state(s), 0, (cudaStream_t)stream));
}

}  // extern "C"
