// Device-side operand packing shared by the standalone act_pack kernel and the
// pack pre-phase fused into the tensor-core linear (linear_tc.cu).
#pragma once
#include "ptx.cuh"
#include "qs_common.cuh"

namespace qs {

__device__ __forceinline__ float snap_group_max(float m) {
  // quant.py:163-176 (fixed point of m -> f32(7*f32(m/7)), <= 8 passes)
  for (int it = 0; it < 8; ++it) {
    const float nx = __fmul_rn(7.0f, __fdiv_rn(m, 7.0f));
    if (nx == m) break;
    m = nx;
  }
  return m;
}

// element k of the token's input row (gather / plain / attention combine)
__device__ __forceinline__ float pack_load(const PackArgs& a, int t, int k, const float* src_row) {
  if (a.att_o == nullptr) return src_row[k];
  const int H = a.K / a.att_hd;
  const int h = k / a.att_hd, d = k - h * a.att_hd;
  const int nch = (a.att_pos[t] + a.att_chunk) / a.att_chunk;  // ceil((pos+1)/chunk)
  const float2* ml = reinterpret_cast<const float2*>(a.att_ml) + ((size_t)t * H + h) * a.att_cmax;
  const float* o = a.att_o + (((size_t)t * H + h) * a.att_cmax) * a.att_hd + d;
  float M = -INFINITY;
  for (int c = 0; c < nch; ++c) M = fmaxf(M, ml[c].x);
  float Ls = 0.f, acc = 0.f;
  for (int c = 0; c < nch; ++c) {
    const float w = expf(ml[c].x - M);
    Ls = fmaf(w, ml[c].y, Ls);
    acc = fmaf(w, o[(size_t)c * a.att_hd], acc);
  }
  return __fdiv_rn(acc, Ls);
}

// pack_load's attention combine for 4 consecutive elements k..k+3 of one head, with
// every chunk statistic / partial fetched in batches (same per-element association:
// max over chunks, then one sequential fma chain over chunks).
__device__ __forceinline__ float4 merge4(const PackArgs& a, int t, int k) {
  const int H = a.K / a.att_hd;
  const int h = k / a.att_hd, d = k - h * a.att_hd;
  const int nch = (a.att_pos[t] + a.att_chunk) / a.att_chunk;
  const float2* ml = reinterpret_cast<const float2*>(a.att_ml) + ((size_t)t * H + h) * a.att_cmax;
  const float* o = a.att_o + (((size_t)t * H + h) * a.att_cmax) * a.att_hd + d;
  float M = -INFINITY;
  for (int c0 = 0; c0 < nch; c0 += 8) {
    float2 mv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) mv[u] = (c0 + u < nch) ? __ldcg(ml + c0 + u) : make_float2(-INFINITY, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) M = (c0 + u < nch) ? fmaxf(M, mv[u].x) : M;
  }
  float Ls = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int c0 = 0; c0 < nch; c0 += 4) {
    float2 mv[4];
    float4 ov[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool on = c0 + u < nch;
      mv[u] = on ? __ldcg(ml + c0 + u) : make_float2(0.f, 0.f);
      ov[u] = on ? __ldcg(reinterpret_cast<const float4*>(o + (size_t)(c0 + u) * a.att_hd)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c0 + u < nch) {
        const float w = expf(mv[u].x - M);
        Ls = fmaf(w, mv[u].y, Ls);
        acc[0] = fmaf(w, ov[u].x, acc[0]);
        acc[1] = fmaf(w, ov[u].y, acc[1]);
        acc[2] = fmaf(w, ov[u].z, acc[2]);
        acc[3] = fmaf(w, ov[u].w, acc[3]);
      }
    }
  }
  return make_float4(__fdiv_rn(acc[0], Ls), __fdiv_rn(acc[1], Ls), __fdiv_rn(acc[2], Ls), __fdiv_rn(acc[3], Ls));
}

// numpy's pairwise float32 sum (numpy/_core/src/umath/loops_utils.h.src, pairwise_sum),
// which np.mean(x * x, dtype=float32) uses along a contiguous row (numerics.py:60):
//   n < 8     sequential from 0;
//   n <= 128  8 strided accumulators r[j] = a[j] + a[8+j] + ... in order, then
//             ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail sequentially;
//   n > 128   split at n2 = n/2 - (n/2)%8 and add the two halves' sums.
// Serial restatement (one thread), for shapes whose recursion is not a balanced tree.
static __device__ float pairwise_sumsq_serial(const float* x, int n) {
  if (n < 8) {
    float r = 0.f;
    for (int i = 0; i < n; ++i) r = __fadd_rn(r, __fmul_rn(x[i], x[i]));
    return r;
  }
  if (n <= 128) {
    float r[8];
    for (int j = 0; j < 8; ++j) r[j] = __fmul_rn(x[j], x[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], __fmul_rn(x[i + j], x[i + j]));
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __fadd_rn(res, __fmul_rn(x[i], x[i]));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __fadd_rn(pairwise_sumsq_serial(x, n2), pairwise_sumsq_serial(x + n2, n - n2));
}

// 1/sqrt(mean(x^2) + eps) of token t's input row (numerics.py:46-62), bit-exact with
// numpy: the row is cut into the pairwise recursion's leaves (n = Lf * 2^lev, Lf <= 128),
// 8 lanes per leaf run its 8 accumulators in numpy's order and combine them with an xor
// tree (= numpy's bracketing), and the leaf sums are combined by the balanced tree of the
// recursion.  Unbalanced recursions (n/2 not a multiple of 8 somewhere) run serially.
// nthreads (a multiple of 32) threads cooperate; red holds >= 130 floats; bar_id is a
// named barrier for those threads.
__device__ __forceinline__ float token_inv_rms(const PackArgs& a, int t, int tid, int nthreads, int bar_id,
                                               float* red) {
  const float* row = a.gather_ids != nullptr ? a.emb + (size_t)a.gather_ids[t] * a.K : a.x + (size_t)t * a.ldx;
  const int n = a.K;
  int Lf = n, lev = 0;
  bool bal = true;
  while (Lf > 128) {
    int h = Lf >> 1;
    h -= h % 8;
    if (2 * h != Lf || lev >= 7) {
      bal = false;
      break;
    }
    Lf = h;
    ++lev;
  }
  float* total = red + 128;
  if (!bal) {
    if (tid == 0) *total = pairwise_sumsq_serial(row, n);
  } else {
    const int nl = 1 << lev, ngroups = nthreads >> 3, gi = tid >> 3, j = tid & 7;
    for (int base = 0; base < nl; base += ngroups) {
      const int b = base + gi;
      const float* x = row + (size_t)(b < nl ? b : 0) * Lf;
      float res = 0.f;
      if (Lf < 8) {
        for (int i = 0; i < Lf; ++i) res = __fadd_rn(res, __fmul_rn(x[i], x[i]));
      } else {
        const int m = Lf >> 3;  // <= 16 accumulator steps
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = i < m ? x[8 * i + j] : 0.f;
        float r = __fmul_rn(v[0], v[0]);
#pragma unroll
        for (int i = 1; i < 16; ++i)
          if (i < m) r = __fadd_rn(r, __fmul_rn(v[i], v[i]));
        r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
        r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
        r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
        res = r;
        for (int i = 8 * m; i < Lf; ++i) res = __fadd_rn(res, __fmul_rn(x[i], x[i]));
      }
      if (j == 0 && b < nl) red[b] = res;
    }
    named_bar(bar_id, nthreads);
    if (tid < 32) {
      // lane l holds the balanced sub-tree of leaves [l*per, (l+1)*per), then an xor tree
      const int per = nl > 32 ? nl >> 5 : 1;
      float s[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) s[i] = (i < per && tid * per + i < nl) ? red[tid * per + i] : 0.f;
      if (per >= 2) s[0] = __fadd_rn(s[0], s[1]);
      if (per >= 4) {
        s[2] = __fadd_rn(s[2], s[3]);
        s[0] = __fadd_rn(s[0], s[2]);
      }
      float v = s[0];
      const int lanes = nl > 32 ? 32 : nl;
      for (int off = 1; off < lanes; off <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
      if (tid == 0) *total = v;
    }
  }
  named_bar(bar_id, nthreads);
  const float ss = *total;
  named_bar(bar_id, nthreads);  // red is reused by the next call
  const float ms = __fdiv_rn(ss, (float)n);
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, a.eps)));
}

// Opt-in block rotation (ModelConfig.hadamard, default off; the reference has none --
// SPEC.md:17): the orthonormal 128-point Walsh-Hadamard transform of one group, lane
// holding elements 4*lane..+3.  Butterfly stages over index bits 0..6 in order (pair
// (i, i | 2^b): a + c, a - c), then * f32(1/sqrt(128)) -- the order oracle/
// qspec_oracle.py wht128 restates, so rotated codes are bit-exact too.
constexpr float kInvSqrt128 = 0.08838834764831845f;
__device__ __forceinline__ void wht128_warp(float (&v)[4], int lane) {
  float t0 = __fadd_rn(v[0], v[1]), t1 = __fsub_rn(v[0], v[1]);
  float t2 = __fadd_rn(v[2], v[3]), t3 = __fsub_rn(v[2], v[3]);
  v[0] = __fadd_rn(t0, t2);
  v[2] = __fsub_rn(t0, t2);
  v[1] = __fadd_rn(t1, t3);
  v[3] = __fsub_rn(t1, t3);
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const bool hi = (lane & m) != 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float o = __shfl_xor_sync(0xffffffffu, v[e], m);
      v[e] = hi ? __fsub_rn(o, v[e]) : __fadd_rn(v[e], o);
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) v[e] = __fmul_rn(v[e], kInvSqrt128);
}

// One warp quantises one 128-element group of token t (lane holds elements 4*lane..+3,
// already normalised) into chunk `ch` of the operand image + its activation scale and
// offset-binary correction sums -- the same arithmetic as pack_group's plain path (the
// linear epilogues use it to emit the NEXT linear's operand; tests check the fused and
// the act_pack operands are bit-identical).
template <int L>
__device__ __forceinline__ void quant_group_warp(const float (&vin)[4], int t, int ch, int lane, uint8_t* img,
                                                 float* ascale, int32_t* acorr, int r_pad, int a_ld,
                                                 bool rotate = false) {
  float v[4] = {vin[0], vin[1], vin[2], vin[3]};
  if (rotate) wht128_warp(v, lane);
  float m = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
  m = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));
  float s, mul;
  int e2 = 0;
  if constexpr (L == 1) {
    m = snap_group_max(m);
    s = __fdiv_rn(m, 7.0f);
    mul = s;
  } else {
    if (m > 0.f) {
      int E;
      frexpf(m, &E);
      e2 = 22 - E;
      mul = ldexpf(1.0f, -e2);
    } else {
      mul = 0.f;
    }
    s = mul;
  }
  uint32_t w[L];
  int lsum[L];
#pragma unroll
  for (int l = 0; l < L; ++l) w[l] = 0, lsum[l] = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int code[L];
    const float x = v[e];
    if constexpr (L == 1) {
      float qv = 0.f;
      if (s != 0.f) qv = fminf(fmaxf(rintf(__fdiv_rn(x, s)), -8.0f), 7.0f);
      code[0] = (int)qv;
    } else {
      const int X = (m > 0.f) ? __float2int_rn(ldexpf(x, e2)) : 0;
      const int l0 = ((X + 128) & 255) - 128;
      const int X1 = (X - l0) >> 8;
      const int l1 = ((X1 + 128) & 255) - 128;
      code[0] = l0;
      code[1 % L] = l1;
      code[2 % L] = (X1 - l1) >> 8;
    }
#pragma unroll
    for (int l = 0; l < L; ++l) w[l] |= ((uint32_t)(code[l] & 0xFF)) << (8 * e), lsum[l] += code[l];
  }
  const size_t chunk_stride = (size_t)r_pad * 128;
#pragma unroll
  for (int l = 0; l < L; ++l)
    *reinterpret_cast<uint32_t*>(img + ch * chunk_stride + sw128_off(t * L + l, lane * 4)) = w[l];
  int S[3] = {0, 0, 0};
#pragma unroll
  for (int l = 0; l < L; ++l) S[l] = __reduce_add_sync(0xffffffffu, lsum[l]);
  if (lane == 0) {
    ascale[(size_t)ch * a_ld + t] = mul;
    *reinterpret_cast<int4*>(acorr + ((size_t)ch * a_ld + t) * 4) =
        make_int4(8 * S[0], 8 * S[1], 8 * S[2], 8 * (256 * S[1] + S[0]));
  }
}

// One warp quantises group gi of token t into the operand image (+ scales).
// kPlain: the common operand (no attention combine, g % 4 == 0, gp == 128) -- one
// float4 per lane and none of the general paths, so the kernel's code stays small
// (the general instantiation is ~12k instructions; instruction fetch dominated it).
// kAttPlain: the same for the attention-combine operand (att_hd % 4 == 0).
template <int L, bool kPlain = false, bool kAttPlain = false>
__device__ __forceinline__ void pack_group(const PackArgs& a, int t, int gi, float inv, int lane) {
  constexpr bool kLean = kPlain || kAttPlain;
  const int K = a.K;
  const float* src_row = a.gather_ids != nullptr ? a.emb + (size_t)a.gather_ids[t] * K : a.x + (size_t)t * a.ldx;
  const int g = a.g, cpg = kLean ? 1 : a.gp >> 7;
  constexpr int kMaxIter = kLean ? 1 : 4;  // gp <= 512
  float val[kMaxIter][4];
  float m = 0.f;
  const bool vec = kPlain || (!kAttPlain && (a.att_o == nullptr) && ((g & 3) == 0));
  const bool att4 = kAttPlain || (!kPlain && (a.att_o != nullptr) && ((g & 3) == 0) && ((a.att_hd & 3) == 0));
#pragma unroll
  for (int it = 0; it < kMaxIter; ++it) {
    const int o0 = it * 128 + lane * 4;
    float4 raw = make_float4(0.f, 0.f, 0.f, 0.f);
    if (vec && o0 < g) raw = *reinterpret_cast<const float4*>(src_row + gi * g + o0);
    if constexpr (!kPlain) {
      if (att4 && o0 < g) raw = merge4(a, t, gi * g + o0);
    }
    const float rv[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int o = o0 + e;
      float v = 0.f;
      if (o < g) {
        const int k = gi * g + o;
        if constexpr (kLean) {
          v = rv[e];
        } else {
          v = (vec || att4) ? rv[e] : pack_load(a, t, k, src_row);
        }
        if (a.x_out) a.x_out[(size_t)t * K + k] = v;
        if (a.rms_w != nullptr) v = __fmul_rn(__fmul_rn(v, inv), a.rms_w[k]);
        if (a.y_out) a.y_out[(size_t)t * K + k] = v;
      }
      val[it][e] = v;
      m = fmaxf(m, fabsf(v));
    }
  }
  if (kLean && a.rotate) {  // opt-in Hadamard rotation of the group (g == gp == 128)
    wht128_warp(val[0], lane);
    m = fmaxf(fmaxf(fabsf(val[0][0]), fabsf(val[0][1])), fmaxf(fabsf(val[0][2]), fabsf(val[0][3])));
  }
  // group max|x| in one warp reduction: non-negative floats order like their bit patterns
  m = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));
  float s, mul;
  int e2 = 0;
  if constexpr (L == 1) {
    m = snap_group_max(m);
    s = __fdiv_rn(m, 7.0f);
    mul = s;
  } else {
    if (m > 0.f) {
      int E;
      frexpf(m, &E);
      e2 = 22 - E;
      mul = ldexpf(1.0f, -e2);
    } else {
      mul = 0.f;
    }
    s = mul;
  }
  if (lane == 0) {
    if (a.ascale)  // per 128-wide chunk (a group spans gp/128 chunks)
      for (int cc = 0; cc < cpg; ++cc) a.ascale[(size_t)(gi * cpg + cc) * a.a_ld + t] = mul;
    if (a.scales_out) a.scales_out[(size_t)t * a.G + gi] = s;
  }
  const size_t chunk_stride = (size_t)a.r_pad * 128;
#pragma unroll
  for (int it = 0; it < kMaxIter; ++it) {
    const int o = it * 128 + lane * 4;
    if (!kLean && it * 128 >= a.gp) break;
    uint32_t w[L];
    int lsum[L];  // this lane's part of the chunk's limb sums (offset-binary correction)
#pragma unroll
    for (int l = 0; l < L; ++l) w[l] = 0, lsum[l] = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int code[L];
#pragma unroll
      for (int l = 0; l < L; ++l) code[l] = 0;
      if (o + e < g) {
        const float x = val[it][e];
        if constexpr (L == 1) {
          float qv = 0.f;
          if (s != 0.f) qv = fminf(fmaxf(rintf(__fdiv_rn(x, s)), -8.0f), 7.0f);
          code[0] = (int)qv;
          const size_t kk = (size_t)gi * g + o + e;
          if (a.codes_out) a.codes_out[(size_t)t * K + kk] = (int8_t)code[0];
          if (a.fq_out) a.fq_out[(size_t)t * K + kk] = __fmul_rn((float)code[0], s);
        } else {
          const int X = (m > 0.f) ? __float2int_rn(ldexpf(x, e2)) : 0;
          const int l0 = ((X + 128) & 255) - 128;
          const int X1 = (X - l0) >> 8;
          const int l1 = ((X1 + 128) & 255) - 128;
          code[0] = l0;
          code[1 % L] = l1;
          code[2 % L] = (X1 - l1) >> 8;
        }
      }
#pragma unroll
      for (int l = 0; l < L; ++l) w[l] |= ((uint32_t)(code[l] & 0xFF)) << (8 * e), lsum[l] += code[l];
    }
    if (a.img) {
      const int kp = gi * a.gp + o;
      const int ch = kp >> 7, byte = kp & 127;
#pragma unroll
      for (int l = 0; l < L; ++l)
        *reinterpret_cast<uint32_t*>(a.img + ch * chunk_stride + sw128_off(t * L + l, byte)) = w[l];
      if (a.acorr) {
        int S[3] = {0, 0, 0};
#pragma unroll
        for (int l = 0; l < L; ++l) S[l] = __reduce_add_sync(0xffffffffu, lsum[l]);
        if (lane == 0)
          *reinterpret_cast<int4*>(a.acorr + ((size_t)ch * a.a_ld + t) * 4) =
              make_int4(8 * S[0], 8 * S[1], 8 * S[2], 8 * (256 * S[1] + S[0]));
      }
    }
  }
}

}  // namespace qs
