// W4A4 (draft) / W4A16 (verify) quantised linear on 5th-gen tensor cores.
//
// y[t, n] = sum_c  wscale[n, c] * ascale[c, t] * D[t, n, c]       (c = 128-wide K chunk)
// D[t, n, c] = sum_{k in c} code_w[n, k] * X[t, k]                 (exact int32, tcgen05 kind::i8)
//
//   draft  (L=1): X = int4 activation codes of the reference's per-(token, group)
//                 quantiser (quant.py:179-194); ascale = its scale.
//   verify (L=3): X = rint(x * 2^e) (24-bit fixed point per (token, group)),
//                 split into three int8 limbs that ride as three extra MMA
//                 columns; ascale = 2^-e.  Same weights, same kernel, same
//                 tensor-core instruction -- only the B operand changes.
//
// Persistent, warp-specialised, stream-K over (tile, chunk) units.  Units are
// processed in STAGES of up to CPS consecutive chunks of one tile so that every
// synchronisation (mbarrier wait / arrive / commit, bulk-copy issue -- each
// ~100 ns of latency on its issuing thread) is amortised over CPS x 8 KiB of
// weights:
//   warp 0      producer: one bulk copy of the stage's packed weights (CPS x 8 KiB,
//               contiguous) + one of its activation image
//   warp 1      MMA issuer (one thread): tcgen05.mma.kind::i8, A = weights in TMEM,
//               B = activation image in smem (128B swizzle), D = int32 in TMEM,
//               one accumulator column block per chunk of the stage
//   warp 2      TMEM allocator
//   warp 3      scale producer: per-stage bulk copies of weight / activation scales
//   warps 4-7   unpack: packed int4 (smem) -> int8 (registers) -> TMEM A operand
//   warps 8-15  epilogue (2 per TMEM lane quadrant, token chunks split): per-chunk
//               TMEM drain, fp32 scale-accumulate, stream-K fixup (fixed order =>
//               deterministic), fused post-op.
// The reduction order of every output depends only on (N, K, grid), never on T,
// so an n-token call is bit-identical to n single-token calls.
#include <type_traits>

#include "pack_dev.cuh"

// per-stage globaltimer stamps for scripts/linear_timeline.py (build with
// QS_NVCC_EXTRA=-DQS_LIN_TIMELINE=1); compiled out by default: the checks sit in
// the MMA issuer's loop
// largest token bucket that gets 8 unpack warps (and 4 epilogue warps)
#ifndef QS_UNPACK8_TMAX
#define QS_UNPACK8_TMAX 8
#endif
#ifndef QS_LIN_TIMELINE
#define QS_LIN_TIMELINE 0
#endif
#ifndef QS_CPS_SMALLN
#define QS_CPS_SMALLN 4
#endif
#ifndef QS_ONE_ACC
#define QS_ONE_ACC 0
#endif
#ifndef QS_EPI16_TMIN
#define QS_EPI16_TMIN 32
#endif
#ifndef QS_U8E8_T
#define QS_U8E8_T 0
#endif
// warp-2 contributor-partial prefetch for buckets T <= this (others: the owner polls and
// gathers).  Measured: B=1 AR 2.36 -> 2.34 ms, B=1 QSpec cycle 10.1 -> 9.9 ms at T <= 8; at
// T = 16 it first cost ~1 % (instruction footprint), and after the shared-space addressing
// of the rings it gains ~0.5 % (B=16 cycle 15.05 -> 15.04, AR B=16 3.21 -> 3.19 ms)
#ifndef QS_PART_PREFETCH_TMAX
#define QS_PART_PREFETCH_TMAX 16
#endif

// research ablations (scripts/lin_ablate.sh), 0 in the product build; bit 0: unpack skips
// LDS + ALU, 1: no MMAs (commits only), 2: epilogue skips TMEM loads + math, 3: unpack
// skips tcgen05.st, 4: no weight bulk copies (the ring fills without HBM traffic),
// 5: epilogue keeps its TMEM loads but skips the scale-accumulate math
#ifndef QS_AB
#define QS_AB 0
#endif
// offset-binary correction by a constant-A MMA where LinCfg::kCorrMma allows (1) or in the
// epilogue everywhere (0)
#ifndef QS_CORR_MMA
#define QS_CORR_MMA 1
#endif
// kEmitSilu group completed by the CTA's last owned tile: quantised after the final
// barrier on every warp (1) or by the epilogue warps in the tail (0)
#ifndef QS_DEFER_SILU
#define QS_DEFER_SILU 1
#endif

namespace qs {

constexpr size_t kPfPiece = 64 * 1024;  // bytes per cp.async.bulk.prefetch.L2

template <int L, int TMAX>
struct LinCfg {
  static constexpr int kRowsMax = (L * TMAX) <= 8 ? 8 : ((L * TMAX + 15) / 16) * 16;
  static constexpr int kAccCols = kRowsMax;  // one accumulator block (N columns) per chunk
  // chunks per stage: as many as TMEM allows with 2 acc buffers + 2 A slots
  // (QS_CPS_SMALLN=6 builds 6-chunk stages where TMEM allows: measured neutral)
  static constexpr int kCPS0 = (QS_CPS_SMALLN == 6 && 2 * 6 * kAccCols + 2 * 6 * 32 <= 512) ? 6
                               : (2 * 4 * kAccCols + 2 * 4 * 32 <= 512) ? 4
                               : (2 * 2 * kAccCols + 2 * 2 * 32 <= 512) ? 2 : 1;
  // wide buckets (N = 192): ONE accumulator buffer of 2-chunk stages instead of two of
  // 1-chunk stages -- half the unpack -> MMA hand-offs per weight byte; the epilogue
  // hands the buffer back right after its tcgen05.ld
  static constexpr bool kOneAcc = QS_ONE_ACC && kCPS0 == 1 && (2 * kAccCols + 2 * 2 * 32 <= 512);
  static constexpr int kCPS = kOneAcc ? 2 : kCPS0;
  // Offset-binary correction on the tensor core (small-token buckets, kUns below): after a
  // chunk's four K-steps, four more MMAs with a constant A of -8 bytes (8 TMEM columns,
  // written once) add -8 * sum_k x to every row, so D is the signed dot product and the
  // epilogue neither loads nor subtracts the per-(chunk, token) sums.  Measured: the
  // 3-limb T = 16 bucket gains (W4A16 AR B=16 3.31 -> 3.24 ms per step); the W4A4 T = 16
  // draft is neutral and the T <= 8 buckets lose (B=1 AR 2.13 -> 2.16 ms: the shallower
  // A ring and the extra MMA issue sit on their latency-bound stages), so only there.
  static constexpr bool kUns0 = TMAX <= 16;
  static constexpr bool kCorrMma = QS_CORR_MMA && L == 3 && TMAX == 16 &&
                                   ((kOneAcc ? 1 : 2) * kCPS * kAccCols + 2 * kCPS * 32 + 32 <= 512);
  static constexpr int kConstCols = kCorrMma ? 32 : 0;
  // spend leftover TMEM on deeper rings (lets unpack / epilogue run further ahead)
  static constexpr int kFree0 = 512 - (kOneAcc ? 1 : 2) * kCPS * kAccCols - 2 * kCPS * 32 - kConstCols;
  static constexpr int kASlots = 2 + (kFree0 >= kCPS * 32 ? 1 : 0);
  static constexpr int kFree1 = kFree0 - (kASlots - 2) * kCPS * 32;
  static constexpr int kAccBufs =
      kOneAcc ? 1 : 2 + (kFree1 / (kCPS * kAccCols) > 2 ? 2 : kFree1 / (kCPS * kAccCols));
  static constexpr int kAColBase = kAccBufs * kCPS * kAccCols;
  static constexpr int kAConst = kAColBase + kASlots * kCPS * 32;  // constant -8 A columns (kCorrMma)
  static constexpr int kTmemCols = 512;
  static_assert(kAConst + kConstCols <= kTmemCols, "TMEM budget");
  static constexpr int kActBytes = kRowsMax * 128;
  static constexpr int kStageBytes = kCPS * (kChunkBytes + kActBytes);
  // 16 warps: 4 control, then unpack and epilogue warps (2 or 1 per TMEM lane
  // quadrant each).  Small T is unpack-bound -> 8 unpack warps; large T is
  // epilogue-bound -> 8 epilogue warps.
  // QS_U8E8_T: buckets of exactly this T get 8 unpack AND 8 epilogue warps (640 threads)
  static constexpr bool kU8E8 = TMAX == QS_U8E8_T;
  static constexpr int kUnpackWarps = (TMAX <= QS_UNPACK8_TMAX || kU8E8) ? 8 : 4;
  // T >= 32 buckets are epilogue-latency bound (one 3-limb chunk drain + scale-accumulate
  // per stage, only two accumulator buffers fit TMEM): 16 epilogue warps (4 per TMEM lane
  // quadrant, 2 token chunks each) in a 768-thread CTA halve each warp's per-chunk chain
  static constexpr int kEpiWarps = TMAX >= QS_EPI16_TMIN ? 16 : (kU8E8 ? 8 : 12 - kUnpackWarps);
  static constexpr int kThreads = 32 * (4 + kUnpackWarps + kEpiWarps);
  static constexpr int kEpiHalves = kEpiWarps / 4;
  static constexpr int kUnpackHalves = kUnpackWarps / 4;
  // residual-emit staging: the tile's new residual rows [T][128] + 1/rms per token
  // (+ the tile's 128 RMSNorm weights for the deferred emit quantiser)
  static constexpr int kStgBytes = ((TMAX < 8 ? 8 : TMAX) * 129 + 128) * 4;
  static constexpr int kStages0 = (196 * 1024 - kStgBytes) / kStageBytes;
  // Unpack group g takes the stages i with i % kUnpackHalves == g and waits on
  // wfull[i % kStages] by parity.  kStages must be a multiple of kUnpackHalves so
  // that each weight slot is only ever consumed by ONE group, which then observes
  // every phase of that slot's barrier; otherwise a group that skipped a phase can
  // read a parity two phases stale and unpack a slot whose bulk copy is in flight.
  static constexpr int kStagesCap = kStages0 > 8 ? 8 : kStages0;
  static constexpr int kStages = kStagesCap - kStagesCap % kUnpackHalves;
  static_assert(kStages >= 2, "pipeline depth");
  static_assert(kStages % kUnpackHalves == 0, "unpack groups must own whole weight slots");
  static constexpr int kSStages = kStages + 2;
  // Offset-binary weights (qs_common.cuh): small-token buckets feed the tensor core the
  // unsigned bytes u = c + 8 straight from one mask (3 ALU ops per 8 codes instead of 7)
  // and subtract 8 * sum(x) per (chunk, token, limb) in the epilogue; buckets with
  // T >= 32 are epilogue-bound, so they convert to signed bytes in the unpack instead
  // (measured: the correction cost T=64 draft 79 -> 89 us on 28672x8192).
  static constexpr bool kUns = kUns0;
  static constexpr int kALd = TMAX < 8 ? 8 : TMAX;  // ascale rows are a_ld = roundup(T, 8) <= kALd
  // scale ring entry: [kCPS][128] weight scales | [kCPS][a_ld] activation scales | (kUns)
  // [kCPS][a_ld][4] correction sums
  static constexpr int kSEntry = kCPS * (128 + kALd + (kUns ? 4 * kALd : 0)) * 4;
  static constexpr int kCorrOff = kCPS * (128 + kALd);  // floats
  static constexpr int kEpiThreads = kEpiWarps * 32;
  static constexpr int kTokChunk = TMAX < 8 ? TMAX : 8;  // tokens per epilogue token chunk (T <= 4 buckets: fewer)
  static constexpr int kOwnChunks = ((TMAX < 8 ? 8 : TMAX) / 8 + kEpiHalves - 1) / kEpiHalves;  // per epilogue warp
  static constexpr int kScaleOff = kStages * kStageBytes;
  static constexpr int kBarOff = kScaleOff + kSStages * kSEntry;
  static constexpr bool kPref = TMAX <= QS_PART_PREFETCH_TMAX;  // warp-2 partial prefetch compiled in
  static constexpr int kNumBars = 3 * kStages + 2 * kASlots + 2 * kAccBufs + 2 * kSStages + (kPref ? 1 : 0);
  static constexpr int kStgOff = ((kBarOff + kNumBars * 8 + 16 + 4 * TMAX * 8 + 4 * 4 + 32 * 4) + 15) / 16 * 16;
  // the rest of the 227 KB: contributor partials of the owned last tile, bulk-copied in by
  // warp 2 while the owner still streams its own stages
  static constexpr int kPartOff = kPref ? (kStgOff + kStgBytes + 127) / 128 * 128 : kStgOff + kStgBytes;
  static constexpr int kPartBytes0 = kPref ? 227 * 1024 - 1024 - kPartOff : 0;
  static constexpr int kPartBytes = kPartBytes0 > 0 ? kPartBytes0 / 512 * 512 : 0;
  static constexpr int kSmemBytes = kPartOff + kPartBytes + 1024;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

// 4 offset-binary nibbles (one per byte, u = c + 8) -> 4 int8 codes c = u - 8 (no borrow
// crosses a byte: (u | 0x80) - 8 >= 0x78)
__device__ __forceinline__ uint32_t ob_to_s8(uint32_t n) {
  return ((n | 0x80808080u) - 0x08080808u) ^ 0x80808080u;
}

// Packed fp32x2 (sm_100): d = a * b + d and d = d * b per lane pair, each element rounded
// exactly as fmaf / __fmul_rn.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 A, B, D;\n\tmov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\tmov.b64 D, {%0, %1};\n\t"
      "fma.rn.f32x2 D, A, B, D;\n\tmov.b64 {%0, %1}, D;\n\t}"
      : "+f"(d0), "+f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fmul2(float& d0, float& d1, float b0, float b1) {
  asm("{\n\t.reg .b64 B, D;\n\tmov.b64 B, {%2, %3};\n\tmov.b64 D, {%0, %1};\n\t"
      "mul.rn.f32x2 D, D, B;\n\tmov.b64 {%0, %1}, D;\n\t}"
      : "+f"(d0), "+f"(d1)
      : "f"(b0), "f"(b1));
}

// Order register uses after an asynchronous TMEM load's tcgen05.wait::ld: an empty
// volatile asm that "rewrites" each register (volatile asms keep their order).
template <int N>
__device__ __forceinline__ void reg_dep(uint32_t (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}

// 32-bit unsigned: a * b < 2^31 for every launch (launch_linear checks n_units * n_cta);
// a 64-bit division is a ~70-instruction dependent chain and the segment-end lookups
// below sit on the owners' critical path
__device__ __forceinline__ unsigned umul_div(unsigned a, unsigned b, unsigned c) { return a * b / c; }

// CTA c of P covers units [bnd(c), bnd(c+1)) of U = n_tiles * n_chunks.
__device__ __forceinline__ int unit_bound(int c, int U, int P) { return (int)umul_div(c, U, P); }
__device__ __forceinline__ int cta_of_unit(int u, int U, int P) {
  int c = (int)umul_div(u, P, U);
  while (c + 1 < P && unit_bound(c + 1, U, P) <= u) ++c;
  while (c > 0 && unit_bound(c, U, P) > u) --c;
  return c;
}

__device__ __forceinline__ float silu_ref(float g) {
  // numerics.py:89-94: x / (1 + exp(-x)), float32, no contraction
  return __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
}

// Stage iterator shared by every role: runs of <= CPS chunks of one tile.  The (tile,
// chunk) position advances incrementally -- one division at construction only (a
// per-stage u / NC in every warp's loop showed up at ~10 % of the linear's samples).
struct StageIt {
  int u, u1, NC, cps;
  int tile, ch0, nq;
  int ntile, nch;  // position of u
  __device__ __forceinline__ StageIt(int u0_, int u1_, int NC_, int cps_) : u(u0_), u1(u1_), NC(NC_), cps(cps_) {
    ntile = u0_ / NC_;
    nch = u0_ - ntile * NC_;
  }
  __device__ __forceinline__ bool next() {
    if (u >= u1) return false;
    tile = ntile;
    ch0 = nch;
    int n = NC - nch;
    if (n > cps) n = cps;
    if (n > u1 - u) n = u1 - u;
    nq = n;
    u += n;
    nch += n;
    if (nch == NC) {
      nch = 0;
      ++ntile;
    }
    return true;
  }
};

// Post-op class fixed at compile time so a launch only carries its own epilogue
// tail (the tail runs once per CTA with a cold instruction cache): OPC = kOpStore
// covers store / residual / dump (runtime a.op), every other class is exact.
template <int OPC, int O>
__device__ __forceinline__ bool op_is(const LinearArgs& a) {
  constexpr bool in_class = OPC == kOpStore ? (O == kOpStore || O == kOpResidual || O == kOpDump) : O == OPC;
  if constexpr (!in_class) return false;
  if constexpr (OPC != kOpStore) return true;
  return a.op == O;
}

// ---------------------------------------------------------------- next-operand emits
// kEmitRms (residual linears): stg = this tile's new residual rows [T][128] (+ [T] 1/rms
// after them).  Leaf = tile: numpy's pairwise sum (numerics.py:60) over a 128 * 2^k row
// splits down to 128-element leaves, each summed with 8 strided accumulators and the
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) bracket; leaves combine as a balanced tree
// (token_inv_rms in pack_dev.cuh states the same order).
// Each leaf is published as ~bits(sum) into a zero-cleared slot, so the owners wait for
// their tokens' leaves by polling the leaves themselves: the last owner's publish reaches
// every owner in one round trip (no counter barrier followed by a second round of loads).
template <int L, int TMAX, int kEpiT, int kEpiWarps>
__device__ __forceinline__ void emit_rms(const LinearArgs& a, float* stg, int tile, int et, int* pending) {
  const int lane = et & 31, ew = et >> 5;
  constexpr int kTW = (TMAX + kEpiWarps - 1) / kEpiWarps;  // tokens per warp
  // this tile's RMSNorm weights do not depend on the leaves: in flight across the wait,
  // parked in shared memory for the deferred quantiser
  float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (TMAX <= 8 || ew == 0) wv = *reinterpret_cast<const float4*>(a.e_rms_w + (size_t)tile * 128 + 4 * lane);
  // clear this tile's column of the other leaf buffer (its readers' launch has completed)
  for (int t = et; t < kLeafRows; t += kEpiT) a.e_leaf_clr[t * kLeafLd + tile] = 0u;
  named_bar(1, kEpiT);
  for (int base = 0; base < a.T * 8; base += kEpiT) {
    const int item = base + et, t = item >> 3, j = item & 7;
    const bool on = t < a.T;
    float rs = 0.f;
    if (on) {
      const float* xr = stg + t * 128;
      rs = __fmul_rn(xr[j], xr[j]);
#pragma unroll
      for (int i = 1; i < 16; ++i) rs = __fadd_rn(rs, __fmul_rn(xr[8 * i + j], xr[8 * i + j]));
    }
    rs = __fadd_rn(rs, __shfl_xor_sync(0xffffffffu, rs, 1));
    rs = __fadd_rn(rs, __shfl_xor_sync(0xffffffffu, rs, 2));
    rs = __fadd_rn(rs, __shfl_xor_sync(0xffffffffu, rs, 4));
    // ~bits is never 0: sums of squares are >= +0 or a NaN other than 0xffffffff
    if (on && j == 0) st_relaxed_u32(a.e_leaf + t * kLeafLd + tile, ~__float_as_uint(rs));
  }
  float* inv = stg + 128 * (a.T > 8 ? a.T : 8);
  const int nl = a.n_tiles, per = nl > 32 ? nl >> 5 : 1, lanes = nl > 32 ? 32 : nl;
  // every leaf of this warp's tokens polled at once until all are published
  float s[kTW][4];
  {
    const unsigned long long t0 = gtimer();
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < kTW; ++k) {
        const int t = ew + k * kEpiWarps;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          s[k][i] = 0.f;
          if (t < a.T && i < per && lane * per + i < nl) {
            const unsigned w = ld_relaxed_u32(a.e_leaf + t * kLeafLd + lane * per + i);
            ok = ok && w != 0u;
            s[k][i] = __uint_as_float(~w);
          }
        }
      }
      if (__all_sync(0xffffffffu, ok)) break;
      if (gtimer() - t0 > 5000000000ull) __trap();
    }
  }
  if (QS_LIN_TIMELINE && a.dbg && et == 0) a.dbg[7168 + blockIdx.x] = gtimer();  // every leaf seen
#pragma unroll
  for (int k = 0; k < kTW; ++k) {
    const int t = ew + k * kEpiWarps;
    if (t >= a.T) break;
    if (per >= 2) s[k][0] = __fadd_rn(s[k][0], s[k][1]);
    if (per >= 4) {
      s[k][2] = __fadd_rn(s[k][2], s[k][3]);
      s[k][0] = __fadd_rn(s[k][0], s[k][2]);
    }
    float v = s[k][0];
    for (int off = 1; off < lanes; off <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) {
      const float ms = __fdiv_rn(v, (float)a.e_n);
      inv[t] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, a.e_eps)));
    }
  }
  if (QS_LIN_TIMELINE && a.dbg && et == 0) a.dbg[7936 + blockIdx.x] = gtimer();  // 1/rms known
  if constexpr (TMAX >= 16) {
    // the group quantiser runs after the CTA's final barrier, spread over all warps
    // (emit_rms_quantise): every other role is idle by then.  Measured: T = 16 draft
    // forward 3.16 -> 3.12 ms; for T <= 8 (a token or two per epilogue warp) the extra
    // barrier costs more than it spreads (B = 1 AR 2.16 -> 2.20 ms), so they quantise here.
    if (ew == 0) reinterpret_cast<float4*>(stg + 129 * TMAX)[lane] = wv;
    if (et == 0) *pending = tile + 1;
  } else {
    __syncwarp();  // inv[t] of this warp's tokens: written and read by this warp only
#pragma unroll 1
    for (int k = 0; k < kTW; ++k) {
      const int t = ew + k * kEpiWarps;
      if (t >= a.T) break;
      const float iv = inv[t];
      const float4 xv = *reinterpret_cast<const float4*>(stg + t * 128 + 4 * lane);
      const float v[4] = {__fmul_rn(__fmul_rn(xv.x, iv), wv.x), __fmul_rn(__fmul_rn(xv.y, iv), wv.y),
                          __fmul_rn(__fmul_rn(xv.z, iv), wv.z), __fmul_rn(__fmul_rn(xv.w, iv), wv.w)};
      quant_group_warp<L>(v, t, tile, lane, a.e_img, a.e_ascale, a.e_acorr, a.r_pad, a.a_ld, a.e_rotate != 0);
    }
    if (QS_LIN_TIMELINE && a.dbg && et == 0) a.dbg[7680 + blockIdx.x] = gtimer();  // quantised
  }
}

// The owned tile's group of the RMSNorm'd rows, one token per warp of the whole CTA (the
// tile is the owner's last segment, so this is the CTA's last work).
template <int L, int TMAX>
__device__ __forceinline__ void emit_rms_quantise(const LinearArgs& a, const float* stg, int tile, int warp,
                                                  int nwarps, int lane) {
  const float* inv = stg + 128 * (a.T > 8 ? a.T : 8);
  const float4 wv = reinterpret_cast<const float4*>(stg + 129 * (TMAX < 8 ? 8 : TMAX))[lane];  // parked by emit_rms
#pragma unroll 1
  for (int t = warp; t < a.T; t += nwarps) {
    const float iv = inv[t];
    const float4 xv = *reinterpret_cast<const float4*>(stg + t * 128 + 4 * lane);
    const float v[4] = {__fmul_rn(__fmul_rn(xv.x, iv), wv.x), __fmul_rn(__fmul_rn(xv.y, iv), wv.y),
                        __fmul_rn(__fmul_rn(xv.z, iv), wv.z), __fmul_rn(__fmul_rn(xv.w, iv), wv.w)};
    quant_group_warp<L>(v, t, tile, lane, a.e_img, a.e_ascale, a.e_acorr, a.r_pad, a.a_ld, a.e_rotate != 0);
  }
}

// kEmitSilu (gate_up): tiles 2q, 2q+1 hold silu outputs 128q..128q+127 = group q of
// down_proj's input.  Each owner publishes its half; the second one quantises the group.
template <int L, int TMAX, int kEpiT, int kEpiWarps>
__device__ __forceinline__ void emit_silu(const LinearArgs& a, int tile, int et, int* flag, bool last, int* pending) {
  constexpr int kTW = (TMAX + kEpiWarps - 1) / kEpiWarps;  // tokens per warp
  const int lane = et & 31, ew = et >> 5, q = tile >> 1;
  named_bar(1, kEpiT);  // the CTA's h writes, then et 0's acq_rel add (cumulative release)
  if (et == 0) *flag = atom_add_acq_rel(&a.e_cnt[8 + q], 1);
  named_bar(1, kEpiT);
  const int second = *flag;
  named_bar(1, kEpiT);
  if (second != 1) return;
  if (TMAX >= 16 && QS_DEFER_SILU && last) {  // the CTA's last work: quantised after the final barrier on every warp
    if (et == 0) *pending = q + 1;
    return;
  }
  float4 hv[kTW];  // all of this warp's rows in flight at once
#pragma unroll
  for (int k = 0; k < kTW; ++k) {
    const int t = ew + k * kEpiWarps;
    hv[k] = t < a.T ? __ldcg(reinterpret_cast<const float4*>(a.out + (size_t)t * a.ldo + 128 * q) + lane)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll 1  // (see emit_rms)
  for (int k = 0; k < kTW; ++k) {
    const int t = ew + k * kEpiWarps;
    if (t >= a.T) break;
    const float v[4] = {hv[k].x, hv[k].y, hv[k].z, hv[k].w};
    quant_group_warp<L>(v, t, q, lane, a.e_img, a.e_ascale, a.e_acorr, a.r_pad, a.a_ld, a.e_rotate != 0);
  }
  if (et == 0) a.e_cnt[8 + q] = 0;
}

// Deferred kEmitSilu group q (the CTA's last owned tile completed it): one token per warp.
template <int L>
__device__ __forceinline__ void emit_silu_quantise(const LinearArgs& a, int q, int warp, int nwarps, int lane) {
#pragma unroll 1
  for (int t = warp; t < a.T; t += nwarps) {
    const float4 hv = __ldcg(reinterpret_cast<const float4*>(a.out + (size_t)t * a.ldo + 128 * q) + lane);
    const float v[4] = {hv.x, hv.y, hv.z, hv.w};
    quant_group_warp<L>(v, t, q, lane, a.e_img, a.e_ascale, a.e_acorr, a.r_pad, a.a_ld, a.e_rotate != 0);
  }
  if (warp == 0 && lane == 0) a.e_cnt[8 + q] = 0;
}

// The linear kernel body (A = the launch's argument block).
template <int L, int TMAX, int OPC>
__device__ __forceinline__ void linear_body(const LinearArgs* __restrict__ A) {
  using C = LinCfg<L, TMAX>;
  constexpr int CPS = C::kCPS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base.  For T >= 32 as an OFFSET from the shared array: the compiler
  // keeps the shared address space, so the ring / scale / staging accesses are LDS / STS
  // (verify forward 6.25 -> 6.09 ms).  The small-token buckets form `smem` through an
  // integer round trip (generic LD / ST) and address only the scale ring and the unpack's
  // weight-ring loads through `smem_sh` below: with the whole kernel (or just the owner
  // tail's staging / partial buffers) in the shared space the compiler batches more shared
  // loads ahead in the tail, which costs registers (T <= 2: 116 -> 128) and measured slower
  // (B=1 AR 2.13 -> 2.24 ms, AR B=16 3.22 -> 3.29 ms).
  uint8_t* smem;
  if constexpr (TMAX >= 32)
    smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  else
    smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* wfull = bars;                      // [kStages] stage weights landed (tx bytes)
  uint64_t* afull = wfull + C::kStages;        // [kStages] stage activation image landed
  uint64_t* empty = afull + C::kStages;        // [kStages] MMA commit -> producer
  uint64_t* tfull = empty + C::kStages;        // [kASlots] unpack -> MMA
  uint64_t* tempty = tfull + C::kASlots;       // [kASlots] MMA commit -> unpack
  uint64_t* accfull = tempty + C::kASlots;     // [kAccBufs] MMA commit -> epilogue
  uint64_t* accempty = accfull + C::kAccBufs;  // [kAccBufs] epilogue -> MMA
  uint64_t* sfull = accempty + C::kAccBufs;    // [kSStages] scales landed
  uint64_t* sempty = sfull + C::kSStages;      // [kSStages] epilogue -> scale producer
  uint64_t* pbar = sempty + C::kSStages;       // [1] prefetched contributor partials landed
  // the scale ring (read by the epilogue every stage) and the weight ring's unpack loads
  // always through the shared space
  uint8_t* const smem_sh = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* sring = reinterpret_cast<float*>(smem_sh + C::kScaleOff);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);
  int* flag = reinterpret_cast<int*>(tmem_slot + 2);
  int* emit_pending = reinterpret_cast<int*>(tmem_slot + 3);  // deferred emit: kEmitRms tile + 1 / kEmitSilu group + 1
  float* red_val = reinterpret_cast<float*>(tmem_slot + 4);  // [4][TMAX]
  int* red_idx = reinterpret_cast<int*>(red_val + 4 * TMAX);  // [4][TMAX]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const bool dbg0 = QS_LIN_TIMELINE && A[0].dbg != nullptr && c == 0;
  if (QS_LIN_TIMELINE && A[0].dbg && threadIdx.x == 0) A[0].dbg[1024 + c] = gtimer();
  ktrace_enter(A[0].kt);
  pdl_launch_dependents();

  // Warp 0 initialises the weight-ring barriers and requests the first stages of weights
  // (independent of the previous kernel) BEFORE the CTA-wide barrier, so a CTA that enters
  // late -- its SM was held by one of the predecessor's owners -- starts its HBM stream
  // without waiting for the other roles' set-up and the TMEM allocation.
  int w_npro = 0;  // warp 0: weight stages already requested
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < C::kStages; ++i) {
        mbar_init(&wfull[i], 1);
        mbar_init(&afull[i], 1);
        mbar_init(&empty[i], 1);
      }
      fence_mbar_init();
    }
    __syncwarp();
    const LinearArgs& a = A[0];
    const int NC = a.n_chunks, U = a.n_tiles * NC, P = a.n_cta;
    StageIt it{unit_bound(c, U, P), unit_bound(c + 1, U, P), NC, CPS};
    for (; w_npro < C::kStages && it.next(); ++w_npro) {
      uint8_t* st = smem + w_npro * C::kStageBytes;
      if (QS_AB & 16) {
        if (lane == 0) mbar_arrive(&wfull[w_npro]);
      } else {
        mbar_arrive_expect_tx_elect(&wfull[w_npro], (uint32_t)it.nq * kChunkBytes);
        bulk_g2s_elect(st, a.codes + ((size_t)it.tile * NC + it.ch0) * kChunkBytes, it.nq * kChunkBytes,
                       &wfull[w_npro]);
      }
    }
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < C::kASlots; ++i) {
      mbar_init(&tfull[i], 4);
      mbar_init(&tempty[i], 1);
    }
    for (int i = 0; i < C::kAccBufs; ++i) {
      mbar_init(&accfull[i], 1);
      mbar_init(&accempty[i], C::kEpiWarps);
    }
    for (int i = 0; i < C::kSStages; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], C::kEpiWarps); }
    if (C::kPref) mbar_init(pbar, 1);
    *emit_pending = 0;
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the launch's unit partition
#define QS_LIN_GEOM(j)                                   \
  const LinearArgs& a = A[j];                            \
  const int NC = a.n_chunks;                             \
  const int U = a.n_tiles * NC, P = a.n_cta;             \
  const int u0 = unit_bound(c, U, P), u1 = unit_bound(c + 1, U, P); \
  (void)u0;                                              \
  (void)u1;
  if (warp == 0) {
    // ------------------------------------------------------------ weight/act producer (warp-wide, elected issue)
    // Weights do not depend on the previous kernel: the first kStages stages of
    // weights are requested before griddepcontrol.wait (PDL overlap); activation
    // images only after it.
    {
      QS_LIN_GEOM(0)
      const uint32_t act_bytes = (uint32_t)a.r_pad * 128u;
      StageIt it{u0, u1, NC, CPS};
      const int npro = w_npro;  // requested before the CTA barrier
      for (int k = 0; k < npro; ++k) it.next();
      // L2 prefetch (no smem, no barrier): the rest of this CTA's own weight range, then
      // its share of the forward's look-ahead window (later linears' weights)
      if (lane == 0) {
        if (a.pf_own) {
          const size_t b0 = ((size_t)it.u) * kChunkBytes, b1 = (size_t)u1 * kChunkBytes;
          for (size_t o = b0; o < b1; o += kPfPiece)
            prefetch_l2(a.codes + o, (uint32_t)(b1 - o < kPfPiece ? b1 - o : kPfPiece));
          const size_t s0 = (size_t)u0 * kTileN * 4, s1 = (size_t)u1 * kTileN * 4;
          if (s1 > s0) prefetch_l2(reinterpret_cast<const uint8_t*>(a.wscale) + s0, (uint32_t)(s1 - s0));
        }
        if (a.pf_n > 0) {
          size_t tot = 0;
          for (int r = 0; r < a.pf_n; ++r) tot += a.pf_len[r];
          // CTA c takes [c*tot/P, (c+1)*tot/P) of the concatenated ranges, 16-byte aligned
          size_t lo = (tot * (size_t)c / P) & ~(size_t)15, hi = (tot * (size_t)(c + 1) / P) & ~(size_t)15;
          if (c == P - 1) hi = tot;
          size_t base = 0;
          for (int r = 0; r < a.pf_n && lo < hi; ++r) {
            const size_t e = base + a.pf_len[r];
            if (lo < e) {
              const size_t x0 = lo - base, x1 = (hi < e ? hi : e) - base;
              for (size_t o = x0; o < x1; o += kPfPiece)
                prefetch_l2(a.pf_ptr[r] + o, (uint32_t)(x1 - o < kPfPiece ? x1 - o : kPfPiece));
              lo = base + x1;
            }
            base = e;
          }
        }
      }
      __syncwarp();
      pdl_wait();
      if (QS_LIN_TIMELINE && a.dbg && lane == 0) a.dbg[4096 + c] = gtimer();
      StageIt ia{u0, u1, NC, CPS};
      for (int i = 0; i < npro && ia.next(); ++i) {
        uint8_t* st = smem + i * C::kStageBytes;
        mbar_arrive_expect_tx_elect(&afull[i], (uint32_t)ia.nq * act_bytes);
        bulk_g2s_elect(st + CPS * kChunkBytes, a.act + (size_t)ia.ch0 * act_bytes, ia.nq * act_bytes, &afull[i]);
        if (dbg0 && i < 64 && lane == 0) a.dbg[0 * 64 + i] = gtimer();
      }
      for (int i = npro; it.next(); ++i) {
        const int s = i % C::kStages;
        mbar_wait(&empty[s], ((i / C::kStages) & 1) ^ 1);
        uint8_t* st = smem + s * C::kStageBytes;
        if (QS_AB & 16) {
          if (lane == 0) mbar_arrive(&wfull[s]);
        } else {
          mbar_arrive_expect_tx_elect(&wfull[s], (uint32_t)it.nq * kChunkBytes);
          bulk_g2s_elect(st, a.codes + ((size_t)it.tile * NC + it.ch0) * kChunkBytes, it.nq * kChunkBytes,
                         &wfull[s]);
        }
        mbar_arrive_expect_tx_elect(&afull[s], (uint32_t)it.nq * act_bytes);
        bulk_g2s_elect(st + CPS * kChunkBytes, a.act + (size_t)it.ch0 * act_bytes, it.nq * act_bytes, &afull[s]);
        if (dbg0 && i < 64 && lane == 0) a.dbg[0 * 64 + i] = gtimer();
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ scale producer (warp-wide, elected issue)
    // Weight scales do not depend on the previous kernel: the first kSStages entries'
    // weight scales are requested before griddepcontrol.wait (with the whole entry's
    // byte count expected up front), the activation scales / correction sums after it.
    {
      QS_LIN_GEOM(0)
      const uint32_t a_bytes = (uint32_t)a.a_ld * 4u;
      const uint32_t e_bytes = 512u + ((C::kUns && !C::kCorrMma) ? 5u : 1u) * a_bytes;  // per chunk
      auto act_part = [&](float* se, const StageIt& st, int ss) {
        bulk_g2s_elect(se + CPS * 128, a.ascale + (size_t)st.ch0 * a.a_ld, st.nq * a_bytes, &sfull[ss]);
        if (C::kUns && !C::kCorrMma)
          bulk_g2s_elect(se + C::kCorrOff, a.acorr + (size_t)st.ch0 * a.a_ld * 4, st.nq * 4u * a_bytes, &sfull[ss]);
      };
      StageIt it{u0, u1, NC, CPS};
      int npro = 0;
      for (; npro < C::kSStages && it.next(); ++npro) {
        float* se = sring + npro * (C::kSEntry / 4);
        mbar_arrive_expect_tx_elect(&sfull[npro], (uint32_t)it.nq * e_bytes);
        bulk_g2s_elect(se, a.wscale + ((size_t)it.tile * NC + it.ch0) * kTileN, it.nq * 512u, &sfull[npro]);
      }
      pdl_wait();
      StageIt ia{u0, u1, NC, CPS};
      for (int i = 0; i < npro && ia.next(); ++i) act_part(sring + i * (C::kSEntry / 4), ia, i);
      for (int i = npro; it.next(); ++i) {
        const int ss = i % C::kSStages;
        mbar_wait(&sempty[ss], ((i / C::kSStages) & 1) ^ 1);
        float* se = sring + ss * (C::kSEntry / 4);
        mbar_arrive_expect_tx_elect(&sfull[ss], (uint32_t)it.nq * e_bytes);
        bulk_g2s_elect(se, a.wscale + ((size_t)it.tile * NC + it.ch0) * kTileN, it.nq * 512u, &sfull[ss]);
        act_part(se, it, ss);
      }
    }
  } else if (C::kPref && warp == 2) {
    // ------------------------------------------------------------ partial prefetch
    // The owner of a split tile processes that tile's first chunks as its LAST segment;
    // the contributors processed the rest as their FIRST segments and published long
    // before.  Warp 2 (idle after the TMEM allocation) waits for them and bulk-copies
    // their partials into shared memory while the owner still streams, so the owner's
    // fixup is one mbarrier wait instead of a counter poll plus a gather round trip.
    QS_LIN_GEOM(0)
    if (u1 > u0 && !op_is<OPC, kOpDump>(a)) {  // dumps keep per-CTA partials, no fixup
      const int lt = (u1 - 1) / NC;
      const int lo = cta_of_unit(lt * NC, U, P), hi = cta_of_unit(lt * NC + NC - 1, U, P);
      const int np = hi - lo;
      if (lo == c && np > 0 && np * a.T * kTileN * 4 <= C::kPartBytes && lane == 0) {
        pdl_wait();  // counters and partial slots are reused across launches
        const unsigned long long t0 = gtimer();
        while (ld_acquire(&a.counters[lt]) != np) {
          if (gtimer() - t0 > 5000000000ull) __trap();
          __nanosleep(64);
        }
        a.counters[lt] = 0;
        fence_proxy_async_global();  // acquired generic writes -> async-proxy reads
        const uint32_t rb = (uint32_t)a.T * kTileN * 4u;
        mbar_arrive_expect_tx(pbar, (uint32_t)np * rb);
        float* dst = reinterpret_cast<float*>(smem + C::kPartOff);
        for (int u = 0; u < np; ++u)
          bulk_g2s(dst + (size_t)u * a.T * kTileN, a.part + ((size_t)(lo + 1 + u + lt) * TMAX) * kTileN, rb, pbar);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (warp-wide, elected issue)
    int i = 0;
    {
      QS_LIN_GEOM(0)
      const uint32_t idesc = idesc_i8(128, (uint32_t)a.r_pad, !C::kUns);
      const uint32_t idesc_s = idesc_i8(128, (uint32_t)a.r_pad, true);  // the constant -8 A is signed
      StageIt it{u0, u1, NC, CPS};
      for (; it.next(); ++i) {
        const int s = i % C::kStages, b = i % C::kAccBufs, as_ = i % C::kASlots;
        if (dbg0 && i < 64 && lane == 0) a.dbg[4 * 64 + i] = gtimer();
        mbar_wait(&accempty[b], ((i / C::kAccBufs) & 1) ^ 1);
        if (dbg0 && i < 64 && lane == 0) a.dbg[5 * 64 + i] = gtimer();
        mbar_wait(&afull[s], (i / C::kStages) & 1);
        if (QS_LIN_TIMELINE && a.dbg && i == 0 && lane == 0) a.dbg[4608 + c] = gtimer();
        if (dbg0 && i < 64 && lane == 0) a.dbg[6 * 64 + i] = gtimer();
        mbar_wait(&tfull[as_], (i / C::kASlots) & 1);
        tc_fence_after();
        if (dbg0 && i < 64 && lane == 0) a.dbg[7 * 64 + i] = gtimer();
        // per-stage bases; every per-MMA offset below is a compile-time constant
        // (the image chunk stride is kActBytes because r_pad == kRowsMax)
        const uint64_t bdesc0 = sdesc_sw128(smem_u32(smem + s * C::kStageBytes + CPS * kChunkBytes));
        const uint32_t d0 = tmem + b * CPS * C::kAccCols;
        const uint32_t a0 = tmem + C::kAColBase + as_ * CPS * 32;
#pragma unroll
        for (int q = 0; q < CPS; ++q)
          if (!(QS_AB & 2) && q < it.nq) {
            mma_i8_ts_chunk4_elect(d0 + q * C::kAccCols, a0 + q * 32,
                                   bdesc0 + (uint64_t)((q * C::kActBytes) >> 4), idesc);
            if constexpr (C::kCorrMma)
              mma_i8_ts_const4_elect(d0 + q * C::kAccCols, tmem + C::kAConst,
                                     bdesc0 + (uint64_t)((q * C::kActBytes) >> 4), idesc_s);
          }
        if (dbg0 && i < 64 && lane == 0) a.dbg[8 * 64 + i] = gtimer();
        mma_commit_elect(&empty[s]);
        mma_commit_elect(&tempty[as_]);
        mma_commit_elect(&accfull[b]);
        if (dbg0 && i < 64 && lane == 0) a.dbg[2 * 64 + i] = gtimer();
      }
    }
  } else if (warp >= 4 && warp < 4 + C::kUnpackWarps) {
    // ------------------------------------------------------------ unpack
    // kUnpackHalves groups of 4 warps (one per TMEM lane quadrant); group ug
    // unpacks the stages i with i % kUnpackHalves == ug, so consecutive stages'
    // latency chains (LDS -> ALU -> tcgen05.st -> wait) overlap.
    const int q4 = warp & 3, ug = (warp - 4) >> 2, r = q4 * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    if (C::kCorrMma && ug == 0) {
      // the constant -8 A operand: waited for (tcgen05.wait::st) with the group's first
      // stage, which the MMA issuer waits for before any MMA reads it
      const uint32_t m8[8] = {0xF8F8F8F8u, 0xF8F8F8F8u, 0xF8F8F8F8u, 0xF8F8F8F8u,
                              0xF8F8F8F8u, 0xF8F8F8F8u, 0xF8F8F8F8u, 0xF8F8F8F8u};
      tmem_st8(tmem + lane_base + C::kAConst, m8);
    }
    int i = 0;
    {
    QS_LIN_GEOM(0)
    StageIt it{u0, u1, NC, CPS};
    for (; it.next(); ++i) {
      if ((i % C::kUnpackHalves) != ug) continue;
      const int s = i % C::kStages, b = i % C::kASlots;
      mbar_wait_warp(&wfull[s], (i / C::kStages) & 1, 0);
      if (QS_LIN_TIMELINE && a.dbg && i == 0 && r == 0) a.dbg[3072 + c] = gtimer();
      mbar_wait_warp(&tempty[b], ((i / C::kASlots) & 1) ^ 1, 0);
      tc_fence_after();
      if (dbg0 && i < 64 && r == 0) a.dbg[9 * 64 + i] = gtimer();
      // all LDS of the stage first (latency overlap), then unpack + TMEM stores
      constexpr int kPre = C::kThreads > 640 ? 1 : (C::kThreads > 512 ? 2 : (CPS <= 4 ? CPS : 1));  // register budget
      uint4 wv[CPS][4];
#pragma unroll
      for (int q = 0; q < kPre; ++q) {
        if (!(QS_AB & 1) && q < it.nq) {
          const uint4* src = reinterpret_cast<const uint4*>(smem_sh + s * C::kStageBytes + q * kChunkBytes);
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) wv[q][jp] = src[jp * 128 + r];
        }
      }
#pragma unroll
      for (int q = 0; q < CPS; ++q) {
        if (q < it.nq) {
          if (!(QS_AB & 1) && q >= kPre) {
            const uint4* src = reinterpret_cast<const uint4*>(smem_sh + s * C::kStageBytes + q * kChunkBytes);
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) wv[q][jp] = src[jp * 128 + r];
          }
          uint32_t v[32];
          if (QS_AB & 1) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = (uint32_t)(r + m);
          } else
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) {
            const uint32_t ww[4] = {wv[q][jp].x, wv[q][jp].y, wv[q][jp].z, wv[q][jp].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int m = jp * 4 + e;
              if constexpr (C::kUns) {
                v[m] = ww[e] & 0x0F0F0F0Fu;
                v[16 + m] = (ww[e] >> 4) & 0x0F0F0F0Fu;
              } else {
                v[m] = ob_to_s8(ww[e] & 0x0F0F0F0Fu);
                v[16 + m] = ob_to_s8((ww[e] >> 4) & 0x0F0F0F0Fu);
              }
            }
          }
          if (!(QS_AB & 8)) tmem_st32(tmem + lane_base + C::kAColBase + (b * CPS + q) * 32, v);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfull[b]);
      if (dbg0 && i < 64 && r == 0) a.dbg[1 * 64 + i] = gtimer();
    }
    }
  } else if (warp >= 4 + C::kUnpackWarps) {
    // ------------------------------------------------------------ epilogue
    // lane quadrant q4 = warp & 3 (TMEM lanes 32q4.. = tile rows); half h owns the
    // token chunks tc with (tc & 1) == h.
    constexpr int kH = C::kEpiHalves, kEpiT = C::kEpiThreads;
    const int q4 = warp & 3, h = (warp - 4 - C::kUnpackWarps) >> 2, r = q4 * 32 + lane;
    const int et = threadIdx.x - 32 * (4 + C::kUnpackWarps);
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    constexpr int kOwn = C::kOwnChunks;
    pdl_wait();  // epilogue reads / writes predecessor-owned buffers
    float acc[kOwn * 8];
#pragma unroll
    for (int t = 0; t < kOwn * 8; ++t) acc[t] = 0.f;
    int i = 0;
    {
    QS_LIN_GEOM(0)
    StageIt it{u0, u1, NC, CPS};
    for (; it.next(); ++i) {
      const int b = i % C::kAccBufs, ss = i % C::kSStages;
      const int tile = it.tile, n = tile * kTileN + r;
      mbar_wait_warp(&sfull[ss], (i / C::kSStages) & 1, 0);
      mbar_wait_warp(&accfull[b], (i / C::kAccBufs) & 1, 0);
      tc_fence_after();
      if (dbg0 && i < 64 && et == 0) a.dbg[10 * 64 + i] = gtimer();
      const float* se = sring + ss * (C::kSEntry / 4);
      bool released = false;  // accumulator buffer b handed back to the MMA
      if (op_is<OPC, kOpDump>(a)) {
        if (h == 0) {
          for (int q = 0; q < it.nq; ++q) {
            const uint32_t col0 = tmem + lane_base + (b * CPS + q) * C::kAccCols;
            const int ch = it.ch0 + q;
            for (int c0 = 0; c0 < a.r_pad; c0 += 8) {
              uint32_t rr[8];
              tmem_ld8(col0 + c0, rr);
              tmem_wait_ld();
              for (int e = 0; e < 8; ++e) {
                const int col = c0 + e, tt = col / L, l = col - tt * L;
                const int32_t corr =
                    (C::kUns && !C::kCorrMma && tt < a.T) ? a.acorr[((size_t)ch * a.a_ld + tt) * 4 + l] : 0;
                a.dump[((size_t)n * NC + ch) * a.r_pad + col] = (int32_t)rr[e] - corr;
              }
            }
          }
        }
      } else {
        float sw[CPS];
#pragma unroll
        for (int q = 0; q < CPS; ++q) sw[q] = (q < it.nq) ? se[q * 128 + r] : 0.f;
        // Software pipeline over this warp's token chunks: the TMEM loads of chunk lc+1
        // are in flight while chunk lc's scale-accumulate runs (one tcgen05.ld -> wait
        // round trip per token chunk was the 3-limb epilogue's critical path).  Only the
        // columns of the chunk's tokens are drained (kCols = tokens x limbs).
        constexpr int kCols = C::kTokChunk * L;
        constexpr int KC = kCols <= 8 ? 8 : (kCols <= 16 ? 16 : 24);
        // double-buffer only where the registers allow (no spills under the 128 cap)
        constexpr bool kPipe = C::kThreads <= 512 && 2 * CPS * KC <= 64;
        uint32_t rb[kPipe ? 2 : 1][CPS][KC];
        auto issue = [&](int lc, uint32_t (&rr)[CPS][KC]) {
#pragma unroll
          for (int q = 0; q < CPS; ++q) {
            if (q < it.nq) {
              const uint32_t col0 = tmem + lane_base + (b * CPS + q) * C::kAccCols + (kH * lc + h) * 8 * L;
              if constexpr (kCols <= 8) {
                tmem_ld8(col0, *reinterpret_cast<uint32_t(*)[8]>(rr[q]));
              } else if constexpr (kCols <= 16) {
                tmem_ld16(col0, rr[q]);
              } else {
                tmem_ld16(col0, rr[q]);
                tmem_ld8(col0 + 16, *reinterpret_cast<uint32_t(*)[8]>(rr[q] + 16));
              }
            }
          }
        };
        const bool any = !(QS_AB & 4) && h * 8 < a.T;
        if (any) issue(0, rb[0]);
#pragma unroll
        for (int lc = 0; lc < kOwn; ++lc) {
          const int tc = kH * lc + h;
          if (!any || tc * 8 >= a.T) break;
          uint32_t(&rr)[CPS][KC] = rb[kPipe ? (lc & 1) : 0];
          if (!kPipe && lc > 0) issue(lc, rr);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < CPS; ++q) reg_dep(rr[q]);  // uses of rr stay after the wait
          const bool more = lc + 1 < kOwn && (kH * (lc + 1) + h) * 8 < a.T;
          if (more) {
            if (kPipe) issue(lc + 1, rb[(lc + 1) & (kPipe ? 1 : 0)]);
          } else {
            // every accumulator column this warp reads is in registers: hand the TMEM
            // buffer back to the MMA now, before the scale-accumulate math
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[b]);
            released = true;
          }
#pragma unroll
          for (int q = 0; q < CPS; ++q) {
            if (!(QS_AB & 32) && q < it.nq) {
              const float* asc = se + CPS * 128 + q * a.a_ld;
              const float4 s0 = *reinterpret_cast<const float4*>(asc + tc * 8);
              const float4 s1 = *reinterpret_cast<const float4*>(asc + tc * 8 + 4);
              const float as[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
              const int* corr = reinterpret_cast<const int*>(se + C::kCorrOff) + (q * a.a_ld + tc * 8) * 4;
              // T >= 32 (epilogue-issue bound): token pairs on the packed fp32x2 pipe (fma /
              // mul .f32x2: two IEEE fmas / products per instruction, the same per-element
              // roundings as fmaf; measured verify forward 6.41 -> 6.26 ms with the attention
              // change of the same commit).  Smaller buckets keep the scalar chain (the packed
              // form measured slower there).
              if constexpr (TMAX >= 32) {
#pragma unroll
              for (int e = 0; e < C::kTokChunk; e += 2) {
                float dv[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  // offset-binary correction (kUns): D = D' - 8 * S per limb
                  if constexpr (L == 1) {
                    const int c0 = (C::kUns && !C::kCorrMma) ? corr[4 * (e + u)] : 0;
                    dv[u] = (float)((int32_t)rr[q][e + u] - c0);
                  } else {
                    // token-major, limb-minor columns: X = l2*2^16 + l1*2^8 + l0.
                    // d1*256+d0 is exact in int32; one rounding in the fma.
                    const int2 cr = (C::kUns && !C::kCorrMma) ? *reinterpret_cast<const int2*>(corr + 4 * (e + u) + 2)
                                                              : make_int2(0, 0);
                    const int32_t lo = (int32_t)rr[q][3 * (e + u) + 1] * 256 + (int32_t)rr[q][3 * (e + u)] - cr.y;
                    dv[u] = (float)lo;
                    rr[q][3 * (e + u) + 2] = __float_as_uint((float)((int32_t)rr[q][3 * (e + u) + 2] - cr.x));
                  }
                }
                if constexpr (L != 1)
                  ffma2(dv[0], dv[1], __uint_as_float(rr[q][3 * e + 2]), __uint_as_float(rr[q][3 * e + 5]), 65536.0f,
                        65536.0f);
                float s0 = sw[q], s1 = sw[q];
                fmul2(s0, s1, as[e], as[e + 1]);
                ffma2(acc[lc * 8 + e], acc[lc * 8 + e + 1], dv[0], dv[1], s0, s1);
              }
              } else {
#pragma unroll
              for (int e = 0; e < C::kTokChunk; ++e) {
                float dv;
                // offset-binary correction (kUns): D = D' - 8 * S per limb
                if constexpr (L == 1) {
                  const int c0 = (C::kUns && !C::kCorrMma) ? corr[4 * e] : 0;
                  dv = (float)((int32_t)rr[q][e] - c0);
                } else {
                  // token-major, limb-minor columns: X = l2*2^16 + l1*2^8 + l0.
                  // d1*256+d0 is exact in int32; one rounding in the fma.
                  const int2 cr = (C::kUns && !C::kCorrMma) ? *reinterpret_cast<const int2*>(corr + 4 * e + 2)
                                                            : make_int2(0, 0);
                  const int32_t lo = (int32_t)rr[q][3 * e + 1] * 256 + (int32_t)rr[q][3 * e] - cr.y;
                  dv = fmaf((float)((int32_t)rr[q][3 * e + 2] - cr.x), 65536.0f, (float)lo);
                }
                acc[lc * 8 + e] = fmaf(dv, sw[q] * as[e], acc[lc * 8 + e]);
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
      }
      if (dbg0 && i < 64 && et == 0) a.dbg[3 * 64 + i] = gtimer();

      // ---- segment end (stages never straddle tiles): stream-K fixup + post-op
      const int last_u = tile * NC + it.ch0 + it.nq - 1;
      const bool seg_end = (it.ch0 + it.nq == NC) || (last_u == u1 - 1);
      if (!seg_end || op_is<OPC, kOpDump>(a)) continue;
      if (QS_LIN_TIMELINE && a.dbg && et == 0) a.dbg[3584 + c] = gtimer();
      const int c_lo = cta_of_unit(tile * NC, U, P);
      const int c_hi = cta_of_unit(tile * NC + NC - 1, U, P);
      // The tail is a chain of dependent global round trips, each ~1-2 us while the next
      // launch streams its weights: the residual rows (independent of the contributors)
      // and then every contributor partial go out as 16-byte async copies, one wait each.
      float* const stg = reinterpret_cast<float*>(smem + C::kStgOff);
      bool res_staged = false;
      if constexpr (OPC == kOpStore) {
        res_staged = a.op == kOpResidual && (a.n & 3) == 0 && !(c_hi > c_lo && c != c_lo);
        if (res_staged) {
          named_bar(1, kEpiT);  // the previous tile's readers of the staging rows are done
          const int n0 = tile * kTileN;
          for (int idx = et; idx < a.T * 32; idx += kEpiT) {
            const int t = idx >> 5, q = idx & 31;
            if (n0 + 4 * q < a.n) cp_async16_cg(stg + t * 128 + 4 * q, a.out + (size_t)t * a.ldo + n0 + 4 * q);
          }
        }
      }
      if (c_hi > c_lo) {
        // Tile split across CTAs c_lo..c_hi.  Non-owners publish their partial and
        // leave (release-increment, no round trip); the owner c_lo -- whose segment
        // of this tile is the last one it processes -- waits for the others and sums
        // in CTA order (deterministic: acc(c_lo) + p(c_lo+1) + ... + p(c_hi)).
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
        const bool prefetched = C::kPref && (c_hi - c_lo) * a.T * kTileN * 4 <= C::kPartBytes;
        if (prefetched) {
          // warp 2 gathered them (the owner's split tile is always its last segment)
          mbar_wait_warp(pbar, 0, 0);
          if (QS_LIN_TIMELINE && a.dbg && et == 0) a.dbg[5120 + c] = gtimer();
          const float* pp = reinterpret_cast<const float*>(smem + C::kPartOff);
          for (int u = 0; u < c_hi - c_lo; ++u) {
#pragma unroll
            for (int lc = 0; lc < kOwn; ++lc)
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int t = (kH * lc + h) * 8 + e;
                if (t < a.T) acc[lc * 8 + e] = __fadd_rn(acc[lc * 8 + e], pp[(u * a.T + t) * kTileN + r]);
              }
          }
        } else {
        if (et == 0) {
          // same 5 s trap guard as the mbarrier waits: a missing contributor (CTAs not
          // co-resident) fails the launch instead of wedging the GPU
          const unsigned long long t0 = gtimer();
          while (ld_acquire(&a.counters[tile]) != c_hi - c_lo) {
            if (gtimer() - t0 > 5000000000ull) __trap();
          }
          a.counters[tile] = 0;
          if (QS_LIN_TIMELINE && a.dbg) a.dbg[5120 + c] = gtimer();
        }
        named_bar(1, kEpiT);
        // the owner's segment is its last one: the whole stage ring is drained and free
        float* const pst = reinterpret_cast<float*>(smem);
        constexpr int kRing = C::kStages * C::kStageBytes / 4;  // floats
        static_assert(kRing >= (TMAX < 8 ? 8 : TMAX) * kTileN, "one partial must fit the ring");
        const int rowsz = a.T * kTileN, np = c_hi - c_lo, maxp = kRing / rowsz;
        for (int p0 = 0; p0 < np; p0 += maxp) {
          const int pn = np - p0 < maxp ? np - p0 : maxp;
          for (int idx = et; idx < pn * a.T * 32; idx += kEpiT) {
            const int u = idx / (a.T * 32), rem = idx - u * a.T * 32, t = rem >> 5, q = rem & 31;
            cp_async16_cg(pst + u * rowsz + t * kTileN + 4 * q,
                          a.part + ((size_t)(c_lo + 1 + p0 + u + tile) * TMAX + t) * kTileN + 4 * q);
          }
          cp_async_wait_all();
          named_bar(1, kEpiT);
          for (int u = 0; u < pn; ++u) {
#pragma unroll
            for (int lc = 0; lc < kOwn; ++lc)
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int t = (kH * lc + h) * 8 + e;
                if (t < a.T) acc[lc * 8 + e] = __fadd_rn(acc[lc * 8 + e], pst[u * rowsz + t * kTileN + r]);
              }
          }
          if (p0 + maxp < np) named_bar(1, kEpiT);  // before the next batch overwrites the ring
        }
        }
      }
      if (res_staged) {
        cp_async_wait_all();
        named_bar(1, kEpiT);
      }
      if (QS_LIN_TIMELINE && a.dbg && et == 0) a.dbg[6144 + c] = gtimer();  // partials summed
      // ---------------------------------------------------------- post-ops
      // the post-op class is a template parameter: a launch carries only its own tail
      auto post = [&](auto opc) {
        constexpr int OP = decltype(opc)::value;
        const bool valid = n < a.n;
        // Every load of the tail is issued before its first store (a load behind a store
        // to a may-alias pointer would wait a full L2 round trip per element).
        float pre[kOwn * 8];  // store class: residual rows
        if constexpr (OP == kOpStore) {
          const bool res = op_is<OP, kOpResidual>(a);
  #pragma unroll
          for (int k = 0; k < kOwn * 8; ++k) {
            const int t = (kH * (k >> 3) + h) * 8 + (k & 7);
            pre[k] = (res && t < a.T && valid) ? (res_staged ? stg[t * 128 + r] : __ldcg(a.out + (size_t)t * a.ldo + n))
                                                : 0.f;
          }
        }
  #pragma unroll
        for (int lc = 0; lc < kOwn; ++lc) {
          float pc[8], ps[8];  // qkv: cos / sin of the chunk's 8 tokens
          int pr[8], prow[8];  // qkv: KV page and in-page row
          if constexpr (OP == kOpQkvRope) {
            const bool is_v = n >= a.n_q + a.n_k;
            const int loc = n < a.n_q ? n : (is_v ? n - a.n_q - a.n_k : n - a.n_q);
            const int half = a.hd >> 1, ip = (loc % a.hd) >> 1;
  #pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int t = (kH * lc + h) * 8 + e;
              pr[e] = (t < a.T) ? a.pos[t] : 0;  // position (uniform per warp)
            }
  #pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int t = (kH * lc + h) * 8 + e;
              const bool on = t < a.T && valid;
              const int p = pr[e];
              pc[e] = (on && !is_v) ? a.rope_cos[(size_t)p * half + ip] : 0.f;
              ps[e] = (on && !is_v) ? a.rope_sin[(size_t)p * half + ip] : 0.f;
              // page / row of the token's KV slot (page is a power of two: a shift and a mask,
              // not two integer divisions per token on the tail's critical path)
              pr[e] = (on && n >= a.n_q) ? a.block_table[(size_t)a.slot[t] * a.bt_ld + (p >> a.page_shift)] : 0;
              prow[e] = p & (a.page - 1);
            }
          }
  #pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int t = (kH * lc + h) * 8 + e;
            const float v = acc[lc * 8 + e];
            if (op_is<OP, kOpStore>(a) || op_is<OP, kOpResidual>(a)) {
              if (t < a.T && valid) {
                const float nv = (op_is<OP, kOpResidual>(a)) ? __fadd_rn(pre[lc * 8 + e], v) : v;
                a.out[(size_t)t * a.ldo + n] = nv;
                if (OP == kOpStore && a.emit == kEmitRms)
                  reinterpret_cast<float*>(smem + C::kStgOff)[t * 128 + r] = nv;
              }
            } else if (op_is<OP, kOpSiluMul>(a)) {
              const float other = __shfl_xor_sync(0xffffffffu, v, 1);
              if (t < a.T && valid && (r & 1) == 0)
                a.out[(size_t)t * a.ldo + (n >> 1)] = __fmul_rn(silu_ref(v), other);
            } else if (op_is<OP, kOpQkvRope>(a)) {
              const float other = __shfl_xor_sync(0xffffffffu, v, 1);
              if (t < a.T && valid) {
                const bool is_v = n >= a.n_q + a.n_k;
                const int loc = n < a.n_q ? n : (is_v ? n - a.n_q - a.n_k : n - a.n_q);
                const int d = loc % a.hd, head = loc / a.hd;
                const bool odd = (d & 1) != 0;
                float val = v;
                if (!is_v) {
                  // model.py:243-252: even' = e*c - o*s ; odd' = e*s + o*c
                  const float cs = pc[e], sn = ps[e];
                  const float ev = odd ? other : v, ov = odd ? v : other;
                  val = odd ? __fadd_rn(__fmul_rn(ev, sn), __fmul_rn(ov, cs))
                            : __fsub_rn(__fmul_rn(ev, cs), __fmul_rn(ov, sn));
                }
                if (n < a.n_q) {
                  a.out[(size_t)t * a.ldo + n] = val;
                } else {
                  const int pg = pr[e], row = prow[e];
                  const size_t off = (((size_t)pg * a.n_kv_heads + head) * a.page + row) * a.hd + d;
                  (is_v ? a.vcache : a.kcache)[off] = val;
                }
              }
            } else if (op_is<OP, kOpLogits>(a)) {
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
        if (op_is<OP, kOpLogits>(a)) {
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
          named_bar(1, kEpiT);
          if (et == 0) {
            const int old = atom_add_acq_rel(&a.counters[a.n_tiles], 1);
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
              if (a.arg_rec != nullptr)
                a.arg_rec[et] = make_int2(__float_as_int(bv), bi + a.arg_off);
              else
                a.argmax_out[et] = bi;
            }
            if (et == 0) a.counters[a.n_tiles] = 0;
          }
        }
        if (QS_LIN_TIMELINE && a.dbg && et == 0) a.dbg[6656 + c] = gtimer();  // post-op stores issued
        if constexpr (OP == kOpStore) {
          if (a.emit == kEmitRms)
            emit_rms<L, TMAX, kEpiT, C::kEpiWarps>(a, reinterpret_cast<float*>(smem + C::kStgOff), tile, et,
                                                   emit_pending);
        }
        if constexpr (OP == kOpSiluMul) {
          if (a.emit == kEmitSilu)
            emit_silu<L, TMAX, kEpiT, C::kEpiWarps>(a, tile, et, flag, last_u == u1 - 1, emit_pending);
        }
      };
      post(std::integral_constant<int, OPC>{});
#pragma unroll
      for (int t = 0; t < kOwn * 8; ++t) acc[t] = 0.f;
    }
    }
  }
#undef QS_LIN_GEOM
  if (QS_LIN_TIMELINE && A[0].dbg && warp == 4 + C::kUnpackWarps && lane == 0) A[0].dbg[5632 + c] = gtimer();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
  if constexpr (OPC == kOpSiluMul) {
    if (*emit_pending) emit_silu_quantise<L>(A[0], *emit_pending - 1, warp, C::kThreads / 32, lane);
  }
  if constexpr (OPC == kOpStore) {
    if (*emit_pending) {
      emit_rms_quantise<L, TMAX>(A[0], reinterpret_cast<const float*>(smem + C::kStgOff), *emit_pending - 1, warp,
                           C::kThreads / 32, lane);
      if (QS_LIN_TIMELINE && A[0].dbg && threadIdx.x == 0) A[0].dbg[7680 + c] = gtimer();  // quantised
    }
  }
  if (QS_LIN_TIMELINE && A[0].dbg && threadIdx.x == 0) A[0].dbg[2048 + c] = gtimer();
  ktrace_exit(A[0].kt);
}

template <int L, int TMAX, int OPC>
__global__ void __launch_bounds__(LinCfg<L, TMAX>::kThreads, 1) linear_tc_kernel(const __grid_constant__ LinearArgs a) {
  linear_body<L, TMAX, OPC>(&a);
}

template <int L, int TMAX, int OPC>
static cudaError_t launch_linear_op(const LinearArgs& a, cudaStream_t st) {
  using C = LinCfg<L, TMAX>;
  static bool attr[kMaxDevices] = {};  // the attribute is per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= kMaxDevices || !attr[dev]) {
    e = cudaFuncSetAttribute(linear_tc_kernel<L, TMAX, OPC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::kSmemBytes);
    if (e != cudaSuccess) return e;
    if (dev < kMaxDevices) attr[dev] = true;
  }
  return launch_k(linear_tc_kernel<L, TMAX, OPC>, dim3(a.n_cta), dim3(C::kThreads), C::kSmemBytes, st, a);
}

template <int L, int TMAX>
static cudaError_t launch_linear_t(const LinearArgs& a, cudaStream_t st) {
  if (a.r_pad != LinCfg<L, TMAX>::kRowsMax) return cudaErrorInvalidValue;  // image rows are padded to the bucket
  switch (a.op) {
    case kOpSiluMul: return launch_linear_op<L, TMAX, kOpSiluMul>(a, st);
    case kOpQkvRope: return launch_linear_op<L, TMAX, kOpQkvRope>(a, st);
    case kOpLogits: return launch_linear_op<L, TMAX, kOpLogits>(a, st);
    default: return launch_linear_op<L, TMAX, kOpStore>(a, st);
  }
}

// token buckets; the 3-limb (verify / AR) path adds T <= 2 and T <= 4 (6 / 12 image
// rows -> UMMA N = 8 / 16, a quarter / half of the TMEM drain of the T <= 8 bucket)
int linear_tmax_bucket(int T, int L) {
  if (L == 3 && T <= 2) return 2;
  if (L == 3 && T <= 4) return 4;
  return T <= 8 ? 8 : T <= 16 ? 16 : T <= 32 ? 32 : 64;
}

cudaError_t launch_linear(int L, const LinearArgs& a, cudaStream_t st) {
  const int tm = linear_tmax_bucket(a.T, L);
  if ((long long)a.n_tiles * a.n_chunks * (a.n_cta + 1) >= (1ll << 31)) return cudaErrorInvalidValue;  // umul_div range
  if (L == 1) {
    switch (tm) {
      case 8: return launch_linear_t<1, 8>(a, st);
      case 16: return launch_linear_t<1, 16>(a, st);
      case 32: return launch_linear_t<1, 32>(a, st);
      default: return launch_linear_t<1, 64>(a, st);
    }
  }
  switch (tm) {
    case 2: return launch_linear_t<3, 2>(a, st);
    case 4: return launch_linear_t<3, 4>(a, st);
    case 8: return launch_linear_t<3, 8>(a, st);
    case 16: return launch_linear_t<3, 16>(a, st);
    case 32: return launch_linear_t<3, 32>(a, st);
    default: return launch_linear_t<3, 64>(a, st);
  }
}

}  // namespace qs
