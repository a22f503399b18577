// Persistent decode-forward kernel: one launch runs a whole forward
// (model.py:255-348) -- every decoder layer's operand packs, tensor-core
// linears, RoPE/KV writes and split-KV attention, then the final norm, lm_head
// and argmax -- on one CTA per SM.
//
// Why: a 7B decode forward is 290 small dependent steps over 3.5 GB of int4
// weights.  Launched one kernel at a time, every step pays a launch, a pipeline
// ramp (TMEM alloc, first-byte DRAM latency) and a drain, and the weight stream
// stops at every dependency.  Here the weight stream never waits on activations:
//
//   warp 0        weight producer: bulk copies of every linear's packed int4
//                 weights, in program order, into a deep smem ring.  It depends
//                 on nothing but ring slots, so HBM keeps streaming through every
//                 pack / attention / stream-K dependency of the forward.
//   unpack warps  int4 -> int8 into TMEM A slots (weights only: they run ahead
//                 too, and release the weight slot as soon as it is in registers)
//   warp 3        operand producer: waits for the linear's operand PACK phase
//                 to complete (device counter), then streams the activation
//                 image + scales
//   warp 1        MMA issuer: tcgen05.mma.kind::i8 (A = weights in TMEM,
//                 B = image in smem, D = int32 in TMEM)
//   worker warps  epilogue of every linear (TMEM drain, per-chunk fp32 scale
//                 accumulate, deterministic stream-K fixup, fused post-op) AND
//                 the non-GEMM phases: operand packs (RMSNorm / embedding gather
//                 / attention merge + per-group quantisation) and attention.
//
// Phase completion is counted in global memory (release add / acquire poll);
// consumers wait on the count of the phase they depend on.  The arithmetic of
// every output is the arithmetic of the per-kernel path (linear_tc.cu,
// act_pack.cu, attention.cu) -- same stream-K partition, same reduction order --
// so the two paths are bit-identical (tests/test_gpu_mk.py).
#include <cstdio>

#include "pack_dev.cuh"

#ifndef QS_POLL_NS
#define QS_POLL_NS 20
#endif

namespace qs {

template <int L, int TMAX>
struct MkCfg {
  static constexpr int kRowsMax = (L * TMAX) <= 8 ? 8 : ((L * TMAX + 15) / 16) * 16;
  static constexpr int kAccCols = kRowsMax;
  static constexpr int kCPS = (2 * 4 * kAccCols + 2 * 4 * 32 <= 512) ? 4
                              : (2 * 2 * kAccCols + 2 * 2 * 32 <= 512) ? 2 : 1;
  static constexpr int kFree0 = 512 - 2 * kCPS * kAccCols - 2 * kCPS * 32;
  static constexpr int kASlots = 2 + (kFree0 >= kCPS * 32 ? 1 : 0);
  static constexpr int kFree1 = kFree0 - (kASlots - 2) * kCPS * 32;
  static constexpr int kAccBufs = 2 + (kFree1 / (kCPS * kAccCols) > 2 ? 2 : kFree1 / (kCPS * kAccCols));
  static constexpr int kAColBase = kAccBufs * kCPS * kAccCols;
  static constexpr int kTmemCols = 512;
  static_assert(kAColBase + kASlots * kCPS * 32 <= kTmemCols, "TMEM budget");
  static constexpr int kActBytes = kRowsMax * 128;
  static constexpr int kWStageBytes = kCPS * kChunkBytes;
  static constexpr int kAStageBytes = kCPS * kActBytes;
  // operand (image) and scale rings deep enough that the operand producer can run a
  // whole linear's images ahead of the MMA once its dependency is met (~48 KB)
  static constexpr int kASt0 = (48 * 1024) / kAStageBytes;
  static constexpr int kASt = kASt0 < 2 ? 2 : (kASt0 > 8 ? 8 : kASt0);
  static constexpr int kSSt = 8;
  static constexpr int kSEntry = kCPS * (128 + (TMAX < 8 ? 8 : TMAX)) * 4;  // ascale rows are a_ld = roundup(T, 8)
  // worker scratch: [0, 2K) logits argmax reduction, [2K, 3K) phase args, [4K, ..) attention q / scores
  static constexpr int kWorkBytes = 4096 + (16 * 128 + 16 * 64 + 16 + 16) * 4;
  // 4 control warps + 4 unpack warps + 4 (T <= 8) or 8 worker warps: 384 threads
  // (168 registers each, no spills) for small T, 512 for the wide epilogues.
  static constexpr int kUnpackWarps = TMAX <= 8 ? 8 : 4;  // 2 (1) warps per TMEM lane quadrant
  static constexpr int kEpiWarps = TMAX <= 8 ? 4 : 8;
  static constexpr int kThreads = 32 * (4 + kUnpackWarps + kEpiWarps);
  static constexpr int kEpiHalves = kEpiWarps / 4;
  static constexpr int kUnpackHalves = kUnpackWarps / 4;  // warps sharing one lane quadrant's pieces
  static constexpr int kEpiThreads = kEpiWarps * 32;
  static constexpr int kTokChunk = TMAX < 8 ? TMAX : 8;  // tokens per epilogue token chunk
  static constexpr int kOwnChunks = ((TMAX < 8 ? 8 : TMAX) / 8 + kEpiHalves - 1) / kEpiHalves;
  static constexpr int kSmemCap = 227 * 1024 - 1024;  // minus alignment slack
  static constexpr int kFixed = kASt * kAStageBytes + kSSt * kSEntry + kWorkBytes + 1024;
  static constexpr int kWSt0 = (kSmemCap - kFixed) / kWStageBytes;
  static constexpr int kWSt = kWSt0 > 16 ? 16 : kWSt0;
  static_assert(kWSt >= 2, "weight ring depth");
  static constexpr int kAOff = kWSt * kWStageBytes;
  static constexpr int kSOff = kAOff + kASt * kAStageBytes;
  static constexpr int kWorkOff = kSOff + kSSt * kSEntry;
  static constexpr int kBarOff = kWorkOff + kWorkBytes;
  static constexpr int kNumBars = 2 * kWSt + 2 * kASt + 2 * kASlots + 2 * kAccBufs + 2 * kSSt;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 64 + 1024;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ uint32_t mk_sext_nib(uint32_t n) {
  return ((n ^ 0x88888888u) - 0x08080808u) ^ 0x80808080u;
}
__device__ __forceinline__ long long mk_umul_div(long long a, long long b, long long c) { return a * b / c; }
__device__ __forceinline__ int mk_unit_bound(int c, int U, int P) { return (int)mk_umul_div(c, U, P); }
__device__ __forceinline__ int mk_cta_of_unit(int u, int U, int P) {
  int c = (int)mk_umul_div(u, P, U);
  while (c + 1 < P && mk_unit_bound(c + 1, U, P) <= u) ++c;
  while (c > 0 && mk_unit_bound(c, U, P) > u) --c;
  return c;
}
__device__ __forceinline__ float mk_silu(float g) { return __fdiv_rn(g, __fadd_rn(1.0f, expf(-g))); }

// Hang guard: every spin in this kernel gives up after ~4 s and traps (a logic
// error surfaces as a launch failure instead of a wedged GPU).
constexpr unsigned long long kSpinLimitNs = 4000000000ull;
__device__ __forceinline__ void spin_check(unsigned long long& t0, uint32_t& n) {
  if ((++n & 255u) == 0) {
    const unsigned long long t = gtimer();
    if (t0 == 0) {
      t0 = t;
    } else if (t - t0 > kSpinLimitNs) {
      printf("[qspec_b200] forward kernel: wait timed out (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}
// try_wait with a suspend-time hint: the thread sleeps in hardware until the phase
// completes (or the hint expires), so waiting roles take no issue slots from the
// workers sharing their SM sub-partition.
__device__ __forceinline__ bool mbar_try_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// Waits back off exponentially (32 ns .. QS_WAIT_MAX_NS): a spinning waiter's
// try_wait traffic shares the SM's LSU/MIO path with the workers' global loads.
#ifndef QS_WAIT_MAX_NS
#define QS_WAIT_MAX_NS 256
#endif
__device__ __forceinline__ void mk_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  unsigned long long t0 = 0;
  uint32_t n = 0, ns = 32;
  while (!mbar_try(bar, parity)) {
    __nanosleep(ns);
    ns = ns < QS_WAIT_MAX_NS ? 2 * ns : ns;
    spin_check(t0, n);
  }
}
// Every lane waits on the barrier itself: the warp stays converged and sleeps in
// hardware (a lone waiting lane leaves 31 lanes spinning in WARPSYNC, stealing
// issue slots from the warps that share the sub-partition).
__device__ __forceinline__ void mk_wait_warp(uint64_t* bar, uint32_t parity) {
  mk_wait(bar, parity);
  __syncwarp();
}
// Poll with relaxed loads (no per-poll L1 invalidation), then one acquire fence.
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mk_wait_count(const int* p, int v) {
  unsigned long long t0 = 0;
  uint32_t n = 0;
  while (ld_relaxed_gpu(p) < v) {
    __nanosleep(QS_POLL_NS);
    spin_check(t0, n);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
template <typename T>
__device__ __forceinline__ T* ldg_ptr(T* const* p) {
  return reinterpret_cast<T*>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}

struct MkIt {  // runs of <= CPS chunks of one tile (same as linear_tc.cu StageIt)
  int u, u1, NC, cps;
  int tile, ch0, nq;
  __device__ __forceinline__ bool next() {
    if (u >= u1) return false;
    tile = u / NC;
    ch0 = u - tile * NC;
    int end = u + cps;
    const int tile_end = (tile + 1) * NC;
    if (end > tile_end) end = tile_end;
    if (end > u1) end = u1;
    nq = end - u;
    u = end;
    return true;
  }
};
__device__ __forceinline__ MkIt mk_units(const LinearArgs& a, int c, int cps) {
  const int U = a.n_tiles * a.n_chunks, P = a.n_cta;
  MkIt it{0, 0, a.n_chunks, cps, 0, 0, 0};
  if (c < P) {
    it.u = mk_unit_bound(c, U, P);
    it.u1 = mk_unit_bound(c + 1, U, P);
  }
  return it;
}
// same, reading the program (global, read-only for the whole launch) through the nc path
__device__ __forceinline__ MkIt mk_units_g(const LinearArgs* a, int c, int cps) {
  const int NC = __ldg(&a->n_chunks);
  const int U = __ldg(&a->n_tiles) * NC, P = __ldg(&a->n_cta);
  MkIt it{0, 0, NC, cps, 0, 0, 0};
  if (c < P) {
    it.u = mk_unit_bound(c, U, P);
    it.u1 = mk_unit_bound(c + 1, U, P);
  }
  return it;
}

// ------------------------------------------------------------------ worker phases
// 1/rms of token t with the association of token_inv_rms(nthreads = 128) computed
// by ONE warp: lane l plays threads l, l+32, l+64, l+96 (bit-identical result).
__device__ __forceinline__ float warp_inv_rms(const PackArgs& a, int t, int lane) {
  const float* src_row = a.gather_ids != nullptr ? a.emb + (size_t)a.gather_ids[t] * a.K : a.x + (size_t)t * a.ldx;
  const float4* row4 = reinterpret_cast<const float4*>(src_row);
  const int K4 = a.K >> 2;
  float part[4] = {0.f, 0.f, 0.f, 0.f};
  for (int base = 0; base < K4; base += 512) {
#pragma unroll
    for (int vh = 0; vh < 4; vh += 2) {  // 8 loads in flight (no spills)
      float4 v[2][4];
#pragma unroll
      for (int vw = 0; vw < 2; ++vw)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k4 = base + u * 128 + (vh + vw) * 32 + lane;
          v[vw][u] = k4 < K4 ? __ldcg(row4 + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int vw = 0; vw < 2; ++vw) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          part[vh + vw] = __fadd_rn(part[vh + vw], __fmul_rn(v[vw][u].x, v[vw][u].x));
          part[vh + vw] = __fadd_rn(part[vh + vw], __fmul_rn(v[vw][u].y, v[vw][u].y));
          part[vh + vw] = __fadd_rn(part[vh + vw], __fmul_rn(v[vw][u].z, v[vw][u].z));
          part[vh + vw] = __fadd_rn(part[vh + vw], __fmul_rn(v[vw][u].w, v[vw][u].w));
        }
      }
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int vw = 0; vw < 4; ++vw) {
    float p = part[vw];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) p = __fadd_rn(p, __shfl_xor_sync(0xffffffffu, p, off));
    ss = __fadd_rn(ss, p);
  }
  const float ms = __fdiv_rn(ss, (float)a.K);
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, a.eps)));
}

// One warp: split-KV attention partial of (block blk, kv head kvh, key chunk ch,
// query group qg of up to QG queries) -- the arithmetic of attn_partial_kernel
// (scores per key by a lane-split dot + xor tree, chunk max / sum by lane
// stride + tree, o_c[d] = sequential fma over keys), with K/V rows read straight
// from the (L2-resident) cache instead of staged in shared memory.  Rows are
// fetched page by page (one block-table lookup per kKB keys), kKB loads in
// flight per lane, and the live state is sized so nothing spills: a spilled load
// result serialises the loads behind it.
constexpr int kMkChunk = 64;
// Branch-free around every shuffle (selects and predicated loads only): a shuffle
// the compiler cannot prove converged gets a BRA.DIV + WARPSYNC.COLLECTIVE slow path.
template <int QG>
__device__ __forceinline__ void attn_warp_item(const AttnArgs& a, int blk, int kvh, int ch, int qg, int lane,
                                           unsigned long long* td) {
  constexpr int kKB = 8;  // keys per load batch
  if (td && lane == 0) td[0] = gtimer();
  const int ntok = a.blk_ntok[blk];
  if (ntok <= 0) return;
  const int tok0 = a.blk_tok0[blk];
  const int j0 = ch * kMkChunk;
  int cmax = 0;
  for (int i = 0; i < ntok; ++i) cmax = max(cmax, a.pos[tok0 + i] + 1);
  if (j0 >= cmax) return;
  const int nk = min(kMkChunk, cmax - j0);
  const int hpk = a.hpk, Q = ntok * hpk, H = a.H, hd = a.hd, page = a.page, KV = a.KV, cmx = a.cmax;
  const float inv_sqrt_hd = a.inv_sqrt_hd;
  const float* kcache = a.kcache;
  const float* vcache = a.vcache;
  const int q0 = qg * QG;
  if (q0 >= Q) return;
  const int nq = min(QG, Q - q0);
  const int* bt = a.block_table + (size_t)a.slot[tok0] * a.bt_ld;
  // hd <= 128: lane owns dims 4*lane .. 4*lane+3 (lanes past hd/4 hold zeros, as the
  // idle lanes of attn_partial_kernel's dot products do)
  const bool dl = lane * 4 < hd;
  float4 qv[QG];
  int ctx[QG];
#pragma unroll
  for (int qq = 0; qq < QG; ++qq) {
    const bool on = qq < nq;
    const int qi = q0 + (on ? qq : 0), i = qi / hpk, h = kvh * hpk + qi % hpk;
    const float4* src = reinterpret_cast<const float4*>(a.q + (size_t)(tok0 + i) * a.ldq + (size_t)h * hd) + lane;
    qv[qq] = (on && dl) ? __ldcg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
    ctx[qq] = on ? a.pos[tok0 + i] + 1 : 0;
  }
  if (td && lane == 0) td[1] = gtimer();
  // scores: s[qq][r] holds key jj = r*32 + lane
  float s[QG][2];
#pragma unroll
  for (int qq = 0; qq < QG; ++qq) s[qq][0] = s[qq][1] = -INFINITY;
#pragma unroll 1
  for (int jb = 0; jb < nk; jb += kKB) {
    const int j = j0 + jb;  // kKB | page (checked on the host): one page per batch
    const size_t base = (((size_t)bt[j / page] * KV + kvh) * page + (j % page)) * hd;
    float4 kr[kKB];
#pragma unroll
    for (int u = 0; u < kKB; ++u) {
      const float4* src = reinterpret_cast<const float4*>(kcache + base + (size_t)u * hd) + lane;
      kr[u] = (jb + u < nk && dl) ? *src : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kKB; ++u) {
      const int jj = jb + u;
#pragma unroll
      for (int qq = 0; qq < QG; ++qq) {
        float p = 0.f;
        p = fmaf(qv[qq].x, kr[u].x, p);
        p = fmaf(qv[qq].y, kr[u].y, p);
        p = fmaf(qv[qq].z, kr[u].z, p);
        p = fmaf(qv[qq].w, kr[u].w, p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        const float sv = (jj < nk && j0 + jj < ctx[qq]) ? p * inv_sqrt_hd : -INFINITY;
        const bool mine = lane == (jj & 31);
        s[qq][0] = (mine && jj < 32) ? sv : s[qq][0];
        s[qq][1] = (mine && jj >= 32) ? sv : s[qq][1];
      }
    }
    if (td && lane == 0 && jb / kKB < 3) td[5 + jb / kKB] = gtimer();
  }
  if (td && lane == 0) td[2] = gtimer();
  // chunk softmax statistics (attn_partial_kernel: lane-strided max / sum + xor trees)
  float pr[QG][2];
#pragma unroll
  for (int qq = 0; qq < QG; ++qq) {
    float m = -INFINITY;
    m = (lane < nk) ? fmaxf(m, s[qq][0]) : m;
    m = (lane + 32 < nk) ? fmaxf(m, s[qq][1]) : m;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const bool on = lane + 32 * r < nk;
      const float e = (m == -INFINITY) ? 0.f : expf(s[qq][r] - m);
      pr[qq][r] = on ? e : 0.f;
      l = on ? l + e : l;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    if (lane == 0 && qq < nq) {
      const int qi = q0 + qq, i = qi / hpk, h = kvh * hpk + qi % hpk;
      float2* ml = reinterpret_cast<float2*>(a.part_ml) + ((size_t)(tok0 + i) * H + h) * cmx + ch;
      *ml = make_float2(m, l);
    }
  }
  if (td && lane == 0) td[3] = gtimer();
  // o_c[d] = sum_j p_j v_j[d], keys ascending
  float4 acc[QG];
#pragma unroll
  for (int qq = 0; qq < QG; ++qq) acc[qq] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int jb = 0; jb < nk; jb += kKB) {
    const int j = j0 + jb;
    const size_t base = (((size_t)bt[j / page] * KV + kvh) * page + (j % page)) * hd;
    float4 vr[kKB];
#pragma unroll
    for (int u = 0; u < kKB; ++u) {
      const float4* src = reinterpret_cast<const float4*>(vcache + base + (size_t)u * hd) + lane;
      vr[u] = (jb + u < nk && dl) ? *src : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kKB; ++u) {
      const int jj = jb + u;
      const bool on = jj < nk;
#pragma unroll
      for (int qq = 0; qq < QG; ++qq) {
        const float p0 = __shfl_sync(0xffffffffu, pr[qq][0], jj & 31);
        const float p1 = __shfl_sync(0xffffffffu, pr[qq][1], jj & 31);
        const float p = jj < 32 ? p0 : p1;
        acc[qq].x = on ? fmaf(p, vr[u].x, acc[qq].x) : acc[qq].x;
        acc[qq].y = on ? fmaf(p, vr[u].y, acc[qq].y) : acc[qq].y;
        acc[qq].z = on ? fmaf(p, vr[u].z, acc[qq].z) : acc[qq].z;
        acc[qq].w = on ? fmaf(p, vr[u].w, acc[qq].w) : acc[qq].w;
      }
    }
  }
#pragma unroll
  for (int qq = 0; qq < QG; ++qq) {
    if (qq < nq && dl) {
      const int qi = q0 + qq, i = qi / hpk, h = kvh * hpk + qi % hpk;
      float4* o = reinterpret_cast<float4*>(a.part_o + (((size_t)(tok0 + i) * H + h) * cmx + ch) * hd);
      o[lane] = acc[qq];
    }
  }
}

// CTA-wide split-KV attention partial of (block blk, kv head kvh, key chunk ch): the
// worker warps share the chunk's 64 keys, exactly as attn_partial_kernel's CTA does
// (score of key jj by one warp: lane-split dot + xor tree; softmax of query qi by one
// warp; o_c[qi][d] = sequential fma over keys by one thread) -- bit-identical to it,
// with each warp's K rows and each thread's V column fetched in one batch.
constexpr int kMkAttnQ = 16;  // queries (block tokens x GQA group) per CTA item
template <int NW>
__device__ __noinline__ void attn_cta_item(const AttnArgs& a, int blk, int kvh, int ch, int et, float* sm,
                                           unsigned long long* td) {
  constexpr int NT = NW * 32, KPW = kMkChunk / NW;  // keys per warp
  const int w = et >> 5, lane = et & 31;
  if (td && et == 0) td[0] = gtimer();
  const int ntok = a.blk_ntok[blk];
  if (ntok <= 0) return;
  const int tok0 = a.blk_tok0[blk];
  const int j0 = ch * kMkChunk;
  int cmax = 0;
  for (int i = 0; i < ntok; ++i) cmax = max(cmax, a.pos[tok0 + i] + 1);
  if (j0 >= cmax) return;
  const int nk = min(kMkChunk, cmax - j0);
  const int hpk = a.hpk, Q = ntok * hpk, H = a.H, hd = a.hd, page = a.page, KV = a.KV, cmx = a.cmax;
  const float inv_sqrt_hd = a.inv_sqrt_hd;
  const float* kcache = a.kcache;
  const float* vcache = a.vcache;
  const int* bt = a.block_table + (size_t)a.slot[tok0] * a.bt_ld;
  float* qv = sm;                       // [Q][hd]
  float* sc = qv + kMkAttnQ * 128;      // [Q][64]
  int* ctx_s = reinterpret_cast<int*>(sc + kMkAttnQ * kMkChunk);  // [Q]
  int* pg_s = ctx_s + kMkAttnQ;                                   // [64 / page] page ids of the chunk
  const bool dl = lane * 4 < hd;
  const int dv = et % hd;
  const int npg = (nk + page - 1) / page;
  if (et < npg) pg_s[et] = bt[(j0 + et * page) / page];
  // row offset (floats) of key jj of the chunk
  auto row = [&](int jj) -> size_t {
    const int j = j0 + jj;
    return (((size_t)pg_s[jj / page] * KV + kvh) * page + (j % page)) * hd;
  };
  // queries -> smem (cp.async 16 B), contexts
  for (int e = et; e < Q * (hd >> 2); e += NT) {
    const int qi = e / (hd >> 2), d4 = e - qi * (hd >> 2);
    const int i = qi / hpk, h = kvh * hpk + qi % hpk;
    cp_async16_cg(qv + qi * hd + d4 * 4, a.q + (size_t)(tok0 + i) * a.ldq + (size_t)h * hd + d4 * 4);
  }
  if (et < Q) ctx_s[et] = a.pos[tok0 + et / hpk] + 1;
  asm volatile("cp.async.wait_all;" ::: "memory");
  named_bar(1, NT);
  // V rows of the chunk toward L2 now (loaded after the scores): 128-byte lines
  {
    const int lpr = (hd * 4 + 127) / 128;
    for (int l = et; l < nk * lpr; l += NT)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(vcache + row(l / lpr) + (l % lpr) * 32));
  }
  if (td && et == 0) td[1] = gtimer();
  // ---- scores: warp w owns keys jj = w + NW*u (the key -> warp map does not change a score)
  {
    float4 kr[KPW];
#pragma unroll
    for (int u = 0; u < KPW; ++u) {
      const int jj = w + NW * u;
      const float4* src = reinterpret_cast<const float4*>(kcache + row(jj < nk ? jj : 0)) + lane;
      kr[u] = (jj < nk && dl) ? *src : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < KPW; ++u) {
      const int jj = w + NW * u, j = j0 + jj;
      for (int qi = 0; qi < Q; ++qi) {
        const float4 q4 = dl ? *reinterpret_cast<const float4*>(qv + qi * hd + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        float p = 0.f;
        p = fmaf(q4.x, kr[u].x, p);
        p = fmaf(q4.y, kr[u].y, p);
        p = fmaf(q4.z, kr[u].z, p);
        p = fmaf(q4.w, kr[u].w, p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        if (lane == 0 && jj < nk) sc[qi * kMkChunk + jj] = (j < ctx_s[qi]) ? p * inv_sqrt_hd : -INFINITY;
      }
    }
  }
  named_bar(1, NT);
  if (td && et == 0) td[2] = gtimer();
  // ---- chunk softmax statistics (warp per query)
  for (int qi = w; qi < Q; qi += NW) {
    float* s = sc + qi * kMkChunk;
    float m = -INFINITY;
    for (int jj = lane; jj < nk; jj += 32) m = fmaxf(m, s[jj]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
    for (int jj = lane; jj < nk; jj += 32) {
      const float e = (m == -INFINITY) ? 0.f : expf(s[jj] - m);
      s[jj] = e;
      l += e;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    if (lane == 0) {
      const int i = qi / hpk, h = kvh * hpk + qi % hpk;
      reinterpret_cast<float2*>(a.part_ml)[((size_t)(tok0 + i) * H + h) * cmx + ch] = make_float2(m, l);
    }
  }
  named_bar(1, NT);
  if (td && et == 0) td[3] = gtimer();
  // ---- o_c[qi][d] = sum_j p_j v_j[d], keys ascending; thread owns dimension dv
  if (et < hd * ((NT / hd) < Q ? (NT / hd) : Q)) {
    const int qstep = NT / hd;  // query stride between the threads sharing dv
    float vv[kMkChunk];
#pragma unroll
    for (int jj = 0; jj < kMkChunk; ++jj) {
      vv[jj] = jj < nk ? vcache[row(jj) + dv] : 0.f;
    }
    for (int qi = et / hd; qi < Q; qi += qstep) {
      const float* pp = sc + qi * kMkChunk;
      float acc = 0.f;
#pragma unroll
      for (int jj = 0; jj < kMkChunk; ++jj) acc = jj < nk ? fmaf(pp[jj], vv[jj], acc) : acc;
      const int i = qi / hpk, h = kvh * hpk + qi % hpk;
      a.part_o[(((size_t)(tok0 + i) * H + h) * cmx + ch) * hd + dv] = acc;
    }
  }
  named_bar(1, NT);  // smem reused by the next item
  if (td && et == 0) td[4] = gtimer();
}

template <int L>
__device__ __forceinline__ void pack_warp_item(const PackArgs& pk, int t, int gi, int lane) {
  const float inv = pk.rms_w != nullptr ? warp_inv_rms(pk, t, lane) : 1.0f;
  pack_group<L>(pk, t, gi, inv, lane);
}

// ------------------------------------------------------------------ the kernel
static_assert(sizeof(LinearArgs) <= 1024 && sizeof(PackArgs) <= 1024 && sizeof(AttnArgs) <= 1024, "phase args");

template <int L, int TMAX>
__global__ void __launch_bounds__(MkCfg<L, TMAX>::kThreads, 1) forward_mk_kernel(const MkArgs g) {
  using C = MkCfg<L, TMAX>;
  constexpr int CPS = C::kCPS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned base by pointer arithmetic on the __shared__ array (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* wfull = bars;                       // [kWSt] weights landed (tx)
  uint64_t* wempty = wfull + C::kWSt;           // [kWSt] unpack group has the weights in registers
  uint64_t* afull = wempty + C::kWSt;           // [kASt] image landed (tx)
  uint64_t* aempty = afull + C::kASt;           // [kASt] MMA commit
  uint64_t* tfull = aempty + C::kASt;           // [kASlots] unpack -> MMA
  uint64_t* tempty = tfull + C::kASlots;        // [kASlots] MMA commit -> unpack
  uint64_t* accfull = tempty + C::kASlots;      // [kAccBufs] MMA commit -> epilogue
  uint64_t* accempty = accfull + C::kAccBufs;   // [kAccBufs] epilogue -> MMA
  uint64_t* sfull = accempty + C::kAccBufs;     // [kSSt] scales landed (tx)
  uint64_t* sempty = sfull + C::kSSt;           // [kSSt] epilogue -> operand producer
  float* sring = reinterpret_cast<float*>(smem + C::kSOff);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);
  int* flag = reinterpret_cast<int*>(tmem_slot + 2);
  float* red_val = reinterpret_cast<float*>(smem + C::kWorkOff);  // [4][TMAX]
  int* red_idx = reinterpret_cast<int*>(red_val + 4 * TMAX);      // [4][TMAX]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x, NCTA = gridDim.x;
  // optional per-stage timeline of CTA 0 (stages < 256): [role][stage] after the phase records
  unsigned long long* sdbg = (g.dbg != nullptr && c == 0) ? g.dbg + 4 * 512 : nullptr;
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kWSt; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], C::kUnpackWarps);
    }
    for (int i = 0; i < C::kASt; ++i) {
      mbar_init(&afull[i], 32);  // cp.async arrive.noinc of every operand-producer lane
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < C::kASlots; ++i) {
      mbar_init(&tfull[i], C::kUnpackWarps);
      mbar_init(&tempty[i], 1);
    }
    for (int i = 0; i < C::kAccBufs; ++i) {
      mbar_init(&accfull[i], 1);
      mbar_init(&accempty[i], C::kEpiWarps);
    }
    for (int i = 0; i < C::kSSt; ++i) {
      mbar_init(&sfull[i], 33);  // weight-scale bulk copy (expect_tx) + 32 operand-producer lanes
      mbar_init(&sempty[i], C::kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const MkPhase* prog = g.prog;

  if (warp == 0) {
    // -------------------------------------------------------------- weight producer
    // Weights depend on nothing: stream them for the whole forward (no pdl_wait).
    int i = 0;
    for (int j = 0; j < g.n_lin; ++j) {
      const LinearArgs* a = &prog[__ldg(&g.lin_phase[j])].lin;
      const uint8_t* codes = ldg_ptr(&a->codes);
      MkIt it = mk_units_g(a, c, CPS);
      const int NC = it.NC;
      if (g.dbg != nullptr && c == 0 && lane == 0) g.dbg[4 * __ldg(&g.lin_phase[j]) + 3] = gtimer();
      for (; it.next(); ++i) {
        const int s = i % C::kWSt;
        if (i >= C::kWSt) mk_wait_warp(&wempty[s], ((i / C::kWSt) & 1) ^ 1);
        uint8_t* st = smem + s * C::kWStageBytes;
        mbar_arrive_expect_tx_elect(&wfull[s], (uint32_t)it.nq * kChunkBytes);
        bulk_g2s_elect(st, codes + ((size_t)it.tile * NC + it.ch0) * kChunkBytes, it.nq * kChunkBytes, &wfull[s]);
        if (sdbg && lane == 0 && i < 256) sdbg[0 * 256 + i] = gtimer();
      }
    }
  } else if (warp == 3) {
    // -------------------------------------------------------------- operand producer
    // Activation image + activation scales by cp.async (LSU path): they sit on the
    // critical path of every linear and must not queue behind the weight stream's
    // bulk copies in the TMA unit.
    pdl_wait();
    int i = 0;
    for (int j = 0; j < g.n_lin; ++j) {
      const MkPhase* ph = &prog[__ldg(&g.lin_phase[j])];
      const LinearArgs* a = &ph->lin;
      MkIt it = mk_units_g(a, c, CPS);
      if (it.u >= it.u1) continue;
      const uint8_t* act = ldg_ptr(&a->act);
      const float* ascale = ldg_ptr(&a->ascale);
      const int a_ld = __ldg(&a->a_ld);
      const uint32_t act_bytes = (uint32_t)__ldg(&a->r_pad) * 128u;
      const uint32_t a_bytes = (uint32_t)a_ld * 4u;
      const int dep = __ldg(&ph->dep), dep_count = __ldg(&ph->dep_count);
      mk_wait_count(&g.cnt[dep], dep_count);  // all lanes (one coalesced request per poll)
      __syncwarp();
      if (g.dbg != nullptr && c == 0 && lane == 0) g.dbg[4 * __ldg(&g.lin_phase[j]) + 1] = gtimer();
      for (; it.next(); ++i) {
        const int sa = i % C::kASt, ss = i % C::kSSt;
        if (i >= C::kASt) mk_wait_warp(&aempty[sa], ((i / C::kASt) & 1) ^ 1);
        if (sdbg && lane == 0 && i < 256) sdbg[8 * 256 + i] = gtimer();
        uint8_t* at = smem + C::kAOff + sa * C::kAStageBytes;
        const uint8_t* src = act + (size_t)it.ch0 * act_bytes;
        const uint32_t nb = (uint32_t)it.nq * act_bytes;
        for (uint32_t off = lane * 16u; off < nb; off += 512u) cp_async16_cg(at + off, src + off);
        cp_async_mbar_arrive(&afull[sa]);
        if (i >= C::kSSt) mk_wait_warp(&sempty[ss], ((i / C::kSSt) & 1) ^ 1);
        float* se = sring + ss * (C::kSEntry / 4) + CPS * 128;
        const float* ssrc = ascale + (size_t)it.ch0 * a_ld;
        for (uint32_t off = lane * 16u; off < (uint32_t)it.nq * a_bytes; off += 512u)
          cp_async16_cg(reinterpret_cast<uint8_t*>(se) + off, reinterpret_cast<const uint8_t*>(ssrc) + off);
        cp_async_mbar_arrive(&sfull[ss]);
        if (sdbg && lane == 0 && i < 256) sdbg[2 * 256 + i] = gtimer();
      }
    }
  } else if (warp == 2) {
    // -------------------------------------------------------------- weight-scale producer
    // Weight scales depend on nothing: bulk-copied into the scale ring ahead of use.
    int i = 0;
    for (int j = 0; j < g.n_lin; ++j) {
      const LinearArgs* a = &prog[__ldg(&g.lin_phase[j])].lin;
      const float* wscale = ldg_ptr(&a->wscale);
      MkIt it = mk_units_g(a, c, CPS);
      const int NC = it.NC;
      for (; it.next(); ++i) {
        const int ss = i % C::kSSt;
        if (i >= C::kSSt) mk_wait_warp(&sempty[ss], ((i / C::kSSt) & 1) ^ 1);
        float* se = sring + ss * (C::kSEntry / 4);
        mbar_arrive_expect_tx_elect(&sfull[ss], (uint32_t)it.nq * 512u);
        bulk_g2s_elect(se, wscale + ((size_t)it.tile * NC + it.ch0) * kTileN, it.nq * 512u, &sfull[ss]);
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    const uint32_t idesc = idesc_i8(128, (uint32_t)C::kRowsMax);
    int i = 0;
    for (int j = 0; j < g.n_lin; ++j) {
      MkIt it = mk_units_g(&prog[__ldg(&g.lin_phase[j])].lin, c, CPS);
      for (; it.next(); ++i) {
        const int sa = i % C::kASt, b = i % C::kAccBufs, as_ = i % C::kASlots;
        mk_wait_warp(&accempty[b], ((i / C::kAccBufs) & 1) ^ 1);
        if (sdbg && lane == 0 && i < 256) sdbg[5 * 256 + i] = gtimer();
        mk_wait_warp(&afull[sa], (i / C::kASt) & 1);
        if (sdbg && lane == 0 && i < 256) sdbg[6 * 256 + i] = gtimer();
        mk_wait_warp(&tfull[as_], (i / C::kASlots) & 1);
        if (sdbg && lane == 0 && i < 256) sdbg[7 * 256 + i] = gtimer();
        fence_proxy_async_smem();  // cp.async-written image -> tensor-core (async proxy) reads
        tc_fence_after();
        const uint64_t bdesc0 = sdesc_sw128(smem_u32(smem + C::kAOff + sa * C::kAStageBytes));
        const uint32_t d0 = tmem + b * CPS * C::kAccCols;
        const uint32_t a0 = tmem + C::kAColBase + as_ * CPS * 32;
#pragma unroll
        for (int q = 0; q < CPS; ++q) {
          if (q < it.nq) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_i8_ts_elect(d0 + q * C::kAccCols, a0 + q * 32 + kk * 8,
                              bdesc0 + (uint64_t)((q * C::kActBytes + kk * 32) >> 4), idesc, kk);
          }
        }
        if (sdbg && lane == 0 && i < 256) sdbg[9 * 256 + i] = gtimer();
        mma_commit_elect(&aempty[sa]);
        mma_commit_elect(&tempty[as_]);
        mma_commit_elect(&accfull[b]);
        if (sdbg && lane == 0 && i < 256) sdbg[3 * 256 + i] = gtimer();
      }
    }
  } else if (warp >= 4 && warp < 4 + C::kUnpackWarps) {
    // -------------------------------------------------------------- unpack
    // Warp (quadrant q4, half uh) unpacks pieces [uh*PPW, (uh+1)*PPW) of its 32 rows of
    // every chunk of the stage: piece j -> A words 4j..4j+3 (low nibbles, k = 16j..)
    // and 16+4j.. (high nibbles, k = 64+16j..).
    constexpr int UH = C::kUnpackHalves, PPW = 4 / UH;
    const int q4 = warp & 3, uh = (warp - 4) >> 2, r = q4 * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    int i = 0;
    for (int j = 0; j < g.n_lin; ++j) {
      MkIt it = mk_units_g(&prog[__ldg(&g.lin_phase[j])].lin, c, CPS);
      for (; it.next(); ++i) {
        const int s = i % C::kWSt, b = i % C::kASlots;
        mk_wait_warp(&wfull[s], (i / C::kWSt) & 1);
        uint4 wv[CPS][PPW];
#pragma unroll
        for (int q = 0; q < CPS; ++q) {
          if (q < it.nq) {
            const uint4* src = reinterpret_cast<const uint4*>(smem + s * C::kWStageBytes + q * kChunkBytes);
#pragma unroll
            for (int jp = 0; jp < PPW; ++jp) wv[q][jp] = src[(uh * PPW + jp) * 128 + r];
          }
        }
        mk_wait_warp(&tempty[b], ((i / C::kASlots) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < CPS; ++q) {
          if (q < it.nq) {
            uint32_t lo[4 * PPW], hi[4 * PPW];
#pragma unroll
            for (int jp = 0; jp < PPW; ++jp) {
              const uint32_t ww[4] = {wv[q][jp].x, wv[q][jp].y, wv[q][jp].z, wv[q][jp].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                lo[jp * 4 + e] = mk_sext_nib(ww[e] & 0x0F0F0F0Fu);
                hi[jp * 4 + e] = mk_sext_nib((ww[e] >> 4) & 0x0F0F0F0Fu);
              }
            }
            const uint32_t col = tmem + lane_base + C::kAColBase + (b * CPS + q) * 32 + uh * 4 * PPW;
            if constexpr (PPW == 4) {
              uint32_t v[32];
#pragma unroll
              for (int m = 0; m < 16; ++m) {
                v[m] = lo[m];
                v[16 + m] = hi[m];
              }
              tmem_st32(col, v);
            } else {
              tmem_st8(col, lo);
              tmem_st8(col + 16, hi);
            }
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&wempty[s]);  // every lane's weights were consumed by the stores above
          mbar_arrive(&tfull[b]);
          if (sdbg && q4 == 0 && uh == 0 && i < 256) sdbg[1 * 256 + i] = gtimer();
        }
      }
    }
  } else if (warp >= 4 + C::kUnpackWarps) {
    // -------------------------------------------------------------- workers
    constexpr int kH = C::kEpiHalves, kEpiT = C::kEpiThreads;
    const int q4 = warp & 3, h = (warp - 4 - C::kUnpackWarps) >> 2, r = q4 * 32 + lane;
    const int et = threadIdx.x - 32 * (4 + C::kUnpackWarps);
    const int ew = et >> 5;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    constexpr int kOwn = C::kOwnChunks;
    pdl_wait();
    int i = 0;  // global stage counter (same sequence as every other role)
    uint8_t* argbuf = smem + C::kWorkOff + 2048;  // this phase's arguments (smem copy)
    for (int p = 0; p < g.n_phases; ++p) {
      if (g.dbg != nullptr && et == 0 && p > 0) g.dbg[8192 + (p - 1) * NCTA + c] = gtimer();  // my share of p-1 done
      const MkPhase* php = &prog[p];
      const int kind = __ldg(&php->kind), dep = __ldg(&php->dep), dep_count = __ldg(&php->dep_count);
      {
        const int* src = kind == kMkLin ? reinterpret_cast<const int*>(&php->lin)
                         : kind == kMkPack ? reinterpret_cast<const int*>(&php->pk)
                                           : reinterpret_cast<const int*>(&php->at);
        const int words = (kind == kMkLin ? (int)sizeof(LinearArgs) : kind == kMkPack ? (int)sizeof(PackArgs)
                                                                                       : (int)sizeof(AttnArgs)) / 4;
        named_bar(1, kEpiT);  // every reader of the previous phase's arguments is done
        for (int w = et; w < words; w += kEpiT) reinterpret_cast<int*>(argbuf)[w] = __ldg(src + w);
        named_bar(1, kEpiT);
      }
      const bool dbg = g.dbg != nullptr && c == 0 && et == 0;
      if (dbg) g.dbg[4 * p + 0] = gtimer();
      if (kind != kMkLin) {
        if (dep >= 0) {
          if (et == 0) mk_wait_count(&g.cnt[dep], dep_count);
          named_bar(1, kEpiT);
        }
        if (dbg) g.dbg[4 * p + 1] = gtimer();
        if (kind == kMkPack) {
          const PackArgs& pk = *reinterpret_cast<const PackArgs*>(argbuf);
          const int n_items = pk.T * pk.G;
          for (int it = c * C::kEpiWarps + ew; it < n_items; it += NCTA * C::kEpiWarps) {
            const int t = it / pk.G, gi = it - t * pk.G;
            pack_warp_item<L>(pk, t, gi, lane);
          }
        } else {
          const AttnArgs& at = *reinterpret_cast<const AttnArgs*>(argbuf);
          const int qg_size = at.qmax * at.hpk == 1 ? 1 : 4;
          const int nqg = (at.qmax * at.hpk + qg_size - 1) / qg_size;
          const int nch = (at.ctx_cap + kMkChunk - 1) / kMkChunk;
          const int n_items = __ldg(&php->n_blk) * at.KV * nch * nqg;
          for (int it = c * C::kEpiWarps + ew; it < n_items; it += NCTA * C::kEpiWarps) {
            int rem = it;
            const int qg = rem % nqg;
            rem /= nqg;
            const int ch = rem % nch;
            rem /= nch;
            const int kvh = rem % at.KV;
            const int blk = rem / at.KV;
            unsigned long long* td = nullptr;
            if (sdbg && p < 12 && ew == 0) td = sdbg + 10 * 256 + 8 * ((it - c * C::kEpiWarps) / (NCTA * C::kEpiWarps));
            if (qg_size == 1)
              attn_warp_item<1>(at, blk, kvh, ch, qg, lane, td);
            else
              attn_warp_item<4>(at, blk, kvh, ch, qg, lane, td);
            if (td && lane == 0) td[4] = gtimer();
          }
        }
        named_bar(1, kEpiT);  // the release below is cumulative over the CTA's writes
        if (et == 0) red_release_add(&g.cnt[p], 1);
        if (dbg) g.dbg[4 * p + 2] = gtimer();
        continue;
      }
      // ------------------------------------------------------------ linear epilogue
      const LinearArgs& a = *reinterpret_cast<const LinearArgs*>(argbuf);
      const int NC = a.n_chunks;
      const int U = a.n_tiles * NC, P = a.n_cta;
      MkIt it = mk_units(a, c, CPS);
      const int u1 = it.u1;
      float acc[kOwn * 8];
#pragma unroll
      for (int t = 0; t < kOwn * 8; ++t) acc[t] = 0.f;
      for (; it.next(); ++i) {
        const int b = i % C::kAccBufs, ss = i % C::kSSt;
        const int tile = it.tile, n = tile * kTileN + r;
        mk_wait_warp(&sfull[ss], (i / C::kSSt) & 1);
        mk_wait_warp(&accfull[b], (i / C::kAccBufs) & 1);
        tc_fence_after();
        const float* se = sring + ss * (C::kSEntry / 4);
        bool released = false;  // accumulator buffer b handed back to the MMA
        {
          float sw[CPS];
#pragma unroll
          for (int q = 0; q < CPS; ++q) sw[q] = (q < it.nq) ? se[q * 128 + r] : 0.f;
#pragma unroll
          for (int lc = 0; lc < kOwn; ++lc) {
            const int tc = kH * lc + h;
            if (tc * 8 < a.T) {
              constexpr int kQB = (L == 3 && CPS == 4 && C::kTokChunk == 8) ? 2 : CPS;  // register budget
              constexpr int kCols = C::kTokChunk * L;  // accumulator columns of one token chunk
#pragma unroll
              for (int qb = 0; qb < CPS; qb += kQB) {
              uint32_t rr[kQB][kCols <= 8 ? 8 : 24];
#pragma unroll
              for (int qq = 0; qq < kQB; ++qq) {
                const int q = qb + qq;
                if (q < it.nq) {
                  const uint32_t col0 = tmem + lane_base + (b * CPS + q) * C::kAccCols;
                  if constexpr (kCols <= 8) {
                    tmem_ld8(col0 + tc * kCols, *reinterpret_cast<uint32_t(*)[8]>(rr[qq]));
                  } else {
                    tmem_ld16(col0 + tc * 24, rr[qq]);
                    tmem_ld8(col0 + tc * 24 + 16, *reinterpret_cast<uint32_t(*)[8]>(rr[qq] + 16));
                  }
                }
              }
              tmem_wait_ld();
              // last TMEM read of this stage by this warp: release the buffer before the math
              if (qb + kQB >= CPS && (lc == kOwn - 1 || (kH * (lc + 1) + h) * 8 >= a.T)) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&accempty[b]);
                released = true;
              }
#pragma unroll
              for (int qq = 0; qq < kQB; ++qq) {
                const int q = qb + qq;
                if (q < it.nq) {
                  const float* asc = se + CPS * 128 + q * a.a_ld;
                  const float4 s0 = *reinterpret_cast<const float4*>(asc + tc * 8);
                  const float4 s1 = *reinterpret_cast<const float4*>(asc + tc * 8 + 4);
                  const float as[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                  for (int e = 0; e < C::kTokChunk; ++e) {
                    float dv;
                    if constexpr (L == 1) {
                      dv = (float)(int32_t)rr[qq][e];
                    } else {
                      const int32_t lo = (int32_t)rr[qq][3 * e + 1] * 256 + (int32_t)rr[qq][3 * e];
                      dv = fmaf((float)(int32_t)rr[qq][3 * e + 2], 65536.0f, (float)lo);
                    }
                    acc[lc * 8 + e] = fmaf(dv, sw[q] * as[e], acc[lc * 8 + e]);
                  }
                }
              }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (!released) mbar_arrive(&accempty[b]);
          mbar_arrive(&sempty[ss]);
          if (sdbg && et == 0 && i < 256) sdbg[4 * 256 + i] = gtimer();
        }

        // ---- segment end: stream-K fixup + post-op (linear_tc.cu, same order)
        const int last_u = tile * NC + it.ch0 + it.nq - 1;
        const bool seg_end = (it.ch0 + it.nq == NC) || (last_u == u1 - 1);
        if (!seg_end) continue;
        const int c_lo = mk_cta_of_unit(tile * NC, U, P);
        const int c_hi = mk_cta_of_unit(tile * NC + NC - 1, U, P);
        if (c_hi > c_lo) {
          if (c != c_lo) {
            float* my = a.part + ((size_t)(c + tile) * TMAX) * kTileN;
#pragma unroll
            for (int lc = 0; lc < kOwn; ++lc)
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int t = (kH * lc + h) * 8 + e;
                if (t < a.T) __stcg(my + t * kTileN + r, acc[lc * 8 + e]);
              }
            named_bar(1, kEpiT);
            if (et == 0) red_release_add(&a.counters[tile], 1);
#pragma unroll
            for (int t = 0; t < kOwn * 8; ++t) acc[t] = 0.f;
            continue;
          }
          if (et == 0) {
            mk_wait_count(&a.counters[tile], c_hi - c_lo);
            a.counters[tile] = 0;
          }
          named_bar(1, kEpiT);
          constexpr int kPB = kOwn <= 1 ? 4 : (kOwn == 2 ? 2 : 1);
          for (int cb = c_lo + 1; cb <= c_hi; cb += kPB) {
            float pv[kPB][kOwn * 8];
#pragma unroll
            for (int u = 0; u < kPB; ++u) {
              const float* pp = a.part + ((size_t)(cb + u + tile) * TMAX) * kTileN;
#pragma unroll
              for (int lc = 0; lc < kOwn; ++lc)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const int t = (kH * lc + h) * 8 + e;
                  pv[u][lc * 8 + e] = (cb + u <= c_hi && t < a.T) ? __ldcg(pp + t * kTileN + r) : 0.f;
                }
            }
#pragma unroll
            for (int u = 0; u < kPB; ++u)
              if (cb + u <= c_hi)
#pragma unroll
                for (int k2 = 0; k2 < kOwn * 8; ++k2) acc[k2] = __fadd_rn(acc[k2], pv[u][k2]);
          }
        }
        // ---------------------------------------------------------- post-ops
        const bool valid = n < a.n;
#pragma unroll
        for (int lc = 0; lc < kOwn; ++lc) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int t = (kH * lc + h) * 8 + e;
            const float v = acc[lc * 8 + e];
            if (a.op == kOpStore || a.op == kOpResidual) {
              if (t < a.T && valid) {
                float* o = a.out + (size_t)t * a.ldo + n;
                *o = (a.op == kOpResidual) ? __fadd_rn(__ldcg(o), v) : v;
              }
            } else if (a.op == kOpSiluMul) {
              const float other = __shfl_xor_sync(0xffffffffu, v, 1);
              if (t < a.T && valid && (r & 1) == 0)
                a.out[(size_t)t * a.ldo + (n >> 1)] = __fmul_rn(mk_silu(v), other);
            } else if (a.op == kOpQkvRope) {
              const float other = __shfl_xor_sync(0xffffffffu, v, 1);
              if (t < a.T && valid) {
                const bool is_v = n >= a.n_q + a.n_k;
                const int loc = n < a.n_q ? n : (is_v ? n - a.n_q - a.n_k : n - a.n_q);
                const int d = loc % a.hd, head = loc / a.hd, half = a.hd >> 1, ip = d >> 1;
                const bool odd = (d & 1) != 0;
                const int pp = a.pos[t];
                float val = v;
                if (!is_v) {
                  const float cs = a.rope_cos[(size_t)pp * half + ip], sn = a.rope_sin[(size_t)pp * half + ip];
                  const float ev = odd ? other : v, ov = odd ? v : other;
                  val = odd ? __fadd_rn(__fmul_rn(ev, sn), __fmul_rn(ov, cs))
                            : __fsub_rn(__fmul_rn(ev, cs), __fmul_rn(ov, sn));
                }
                if (n < a.n_q) {
                  a.out[(size_t)t * a.ldo + n] = val;
                } else {
                  const int sl = a.slot[t];
                  const int pg = a.block_table[(size_t)sl * a.bt_ld + pp / a.page];
                  const size_t off = (((size_t)pg * a.n_kv_heads + head) * a.page + (pp % a.page)) * a.hd + d;
                  (is_v ? a.vcache : a.kcache)[off] = val;
                }
              }
            } else if (a.op == kOpLogits) {
              if (t < a.T) {
                if (a.out != nullptr && valid) a.out[(size_t)t * a.ldo + n] = v;
                float bv = valid ? v : -INFINITY;
                int bi = valid ? n : 0x7fffffff;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                  const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                  const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                  if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                }
                if (lane == 0) { red_val[q4 * TMAX + t] = bv; red_idx[q4 * TMAX + t] = bi; }
              }
            }
          }
        }
        if (a.op == kOpLogits) {
          named_bar(1, kEpiT);
          if (et < a.T) {
            float bv = red_val[et];
            int bi = red_idx[et];
            for (int w = 1; w < 4; ++w) {
              const float ov = red_val[w * TMAX + et];
              const int oi = red_idx[w * TMAX + et];
              if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            a.arg_val[(size_t)tile * TMAX + et] = bv;
            a.arg_idx[(size_t)tile * TMAX + et] = bi;
          }
          __threadfence();
          named_bar(1, kEpiT);
          if (et == 0) {
            const int old = atomicAdd(&a.counters[a.n_tiles], 1);
            *flag = (old == a.n_tiles - 1);
          }
          named_bar(1, kEpiT);
          const int last = *flag;
          named_bar(1, kEpiT);
          if (last) {
            __threadfence();
            if (et < a.T) {
              const volatile float* av = a.arg_val;
              const volatile int* ai = a.arg_idx;
              float bv = av[et];
              int bi = ai[et];
              for (int tt = 1; tt < a.n_tiles; ++tt) {
                const float ov = av[(size_t)tt * TMAX + et];
                const int oi = ai[(size_t)tt * TMAX + et];
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
              }
              a.argmax_out[et] = bi;
            }
            if (et == 0) a.counters[a.n_tiles] = 0;
          }
        }
        // tile complete: publish (phase count = n_tiles)
        named_bar(1, kEpiT);
        if (et == 0) red_release_add(&g.cnt[p], 1);
        if (dbg) g.dbg[4 * p + 2] = gtimer();
#pragma unroll
        for (int t = 0; t < kOwn * 8; ++t) acc[t] = 0.f;
      }
    }
    if (g.dbg != nullptr && et == 0) g.dbg[8192 + (g.n_phases - 1) * NCTA + c] = gtimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
  // last CTA out resets the phase counters for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    const int old = atomicAdd(&g.cnt[g.n_phases], 1);
    if (old == NCTA - 1) {
      for (int p = 0; p <= g.n_phases; ++p) g.cnt[p] = 0;
      __threadfence();
    }
  }
}

template <int L, int TMAX>
static cudaError_t launch_mk_t(const MkArgs& g, int n_cta, cudaStream_t st) {
  using C = MkCfg<L, TMAX>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(forward_mk_kernel<L, TMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_k(forward_mk_kernel<L, TMAX>, dim3(n_cta), dim3(C::kThreads), C::kSmemBytes, st, g);
}

// token bucket of the persistent kernel: the per-step buckets plus T <= 2 for the
// 3-limb verify / AR forward (6 image rows -> UMMA N = 8 instead of 32)
int mk_tmax_bucket(int T, int L) {
  if (L == 3 && T <= 2) return 2;
  return T <= 8 ? 8 : T <= 16 ? 16 : T <= 32 ? 32 : 64;
}

cudaError_t launch_forward_mk(int L, int T, const MkArgs& g, int n_cta, cudaStream_t st) {
  const int tm = mk_tmax_bucket(T, L);
  if (L == 1) {
    switch (tm) {
      case 8: return launch_mk_t<1, 8>(g, n_cta, st);
      case 16: return launch_mk_t<1, 16>(g, n_cta, st);
      case 32: return launch_mk_t<1, 32>(g, n_cta, st);
      default: return launch_mk_t<1, 64>(g, n_cta, st);
    }
  }
  switch (tm) {
    case 2: return launch_mk_t<3, 2>(g, n_cta, st);
    case 8: return launch_mk_t<3, 8>(g, n_cta, st);
    case 16: return launch_mk_t<3, 16>(g, n_cta, st);
    case 32: return launch_mk_t<3, 32>(g, n_cta, st);
    default: return launch_mk_t<3, 64>(g, n_cta, st);
  }
}

int mk_attn_chunk_len() { return kMkChunk; }

}  // namespace qs
