// W4A4 (draft) / W4A16 (verify) quantised linear on 5th-gen tensor cores.
//
// y[t, n] = sum_g  wscale[g, n] * ascale[g, t] * D[t, n, g]
// D[t, n, g] = sum_{k in g} code_w[n, k] * X[t, k]       (exact int32 on tcgen05 kind::i8)
//
//   draft  (L=1): X = int4 activation codes of the reference's per-(token, group)
//                 quantiser (quant.py:179-194); ascale = its scale.
//   verify (L=3): X = rint(x * 2^e) (24-bit fixed point per (token, group)),
//                 split into three int8 limbs that ride as three extra MMA
//                 columns; ascale = 2^-e.  Same weights, same kernel, same
//                 tensor-core instruction -- only the B operand changes.
//
// Persistent, warp-specialised, stream-K over (tile, group) units:
//   warp 0      producer: bulk-async copies of packed weight chunks + activation image
//   warp 1      MMA issuer (one thread): tcgen05.mma.kind::i8, A from TMEM, B from smem
//   warp 2      TMEM allocator
//   warps 4-7   unpack: packed int4 (smem) -> int8 (registers) -> TMEM A operand
//   warps 8-11  epilogue: per-group TMEM drain, fp32 scale-accumulate, stream-K
//               fixup (fixed order => deterministic), fused post-op.
// The reduction order of every output depends only on (N, K, grid), never on T,
// so an n-token call is bit-identical to n single-token calls.
#include "ptx.cuh"
#include "qs_common.cuh"

namespace qs {

template <int L, int TMAX>
struct LinCfg {
  static constexpr int kRowsMax = (L * TMAX) <= 8 ? 8 : ((L * TMAX + 15) / 16) * 16;
  static constexpr int kActBytes = kRowsMax * 128;
  static constexpr int kStageBytes = kChunkBytes + kActBytes;
  static constexpr int kStages = (200 * 1024 / kStageBytes) > 10 ? 10 : (200 * 1024 / kStageBytes);
  static constexpr int kTStages = 4;                 // TMEM A-operand slots (32 cols each)
  static constexpr int kAccCols = kRowsMax < 32 ? 32 : kRowsMax;
  static constexpr int kAColBase = 2 * kAccCols;
  static constexpr int kTmemCols = 512;
  static_assert(2 * kAccCols + kTStages * 32 <= kTmemCols, "TMEM budget");
  static constexpr int kBarOff = kStages * kStageBytes;
  static constexpr int kNumBars = 2 * kStages + 2 * kTStages + 4;
  static constexpr int kSmemBytes = kBarOff + kNumBars * 8 + 16 + 4 * TMAX * 8 + 1024;
};

__device__ __forceinline__ uint32_t sext_nib(uint32_t n) {  // 4 nibbles (one per byte) -> 4 int8
  return ((n ^ 0x88888888u) - 0x08080808u) ^ 0x80808080u;
}

__device__ __forceinline__ long long umul_div(long long a, long long b, long long c) { return a * b / c; }

// CTA c of P covers units [bnd(c), bnd(c+1)) of U = n_tiles * G.
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

template <int L, int TMAX>
__global__ void __launch_bounds__(384, 1) linear_tc_kernel(const LinearArgs a) {
  using C = LinCfg<L, TMAX>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;                       // [kStages] producer -> MMA/unpack (tx bytes)
  uint64_t* empty = bars + C::kStages;         // [kStages] MMA commit -> producer
  uint64_t* tfull = empty + C::kStages;        // [kTStages] unpack -> MMA
  uint64_t* tempty = tfull + C::kTStages;      // [kTStages] MMA commit -> unpack
  uint64_t* accfull = tempty + C::kTStages;    // [2] MMA commit -> epilogue
  uint64_t* accempty = accfull + 2;            // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);
  int* flag = reinterpret_cast<int*>(tmem_slot + 2);
  float* red_val = reinterpret_cast<float*>(tmem_slot + 4);  // [4][TMAX]
  int* red_idx = reinterpret_cast<int*>(red_val + 4 * TMAX);  // [4][TMAX]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int U = a.n_tiles * a.G, P = a.n_cta, c = blockIdx.x;
  const int u0 = unit_bound(c, U, P), u1 = unit_bound(c + 1, U, P);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < C::kTStages; ++i) { mbar_init(&tfull[i], 4); mbar_init(&tempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&accfull[i], 1); mbar_init(&accempty[i], 4); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int cpg = a.cpg;
  const uint32_t act_bytes = (uint32_t)a.r_pad * 128u;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int i = 0;
      for (int u = u0; u < u1; ++u) {
        const int tile = u / a.G, gi = u % a.G;
        for (int cc = 0; cc < cpg; ++cc, ++i) {
          const int ch = gi * cpg + cc, s = i % C::kStages;
          mbar_wait(&empty[s], ((i / C::kStages) & 1) ^ 1);
          uint8_t* st = smem + s * C::kStageBytes;
          mbar_arrive_expect_tx(&full[s], kChunkBytes + act_bytes);
          bulk_g2s(st, a.codes + ((size_t)tile * a.n_chunks + ch) * kChunkBytes, kChunkBytes, &full[s]);
          bulk_g2s(st + kChunkBytes, a.act + (size_t)ch * act_bytes, act_bytes, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_i8(128, (uint32_t)a.r_pad);
      int i = 0, j = 0;
      for (int u = u0; u < u1; ++u, ++j) {
        const int b = j & 1;
        mbar_wait(&accempty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + b * C::kAccCols;
        for (int cc = 0; cc < cpg; ++cc, ++i) {
          const int s = i % C::kStages, ts = i % C::kTStages;
          mbar_wait(&full[s], (i / C::kStages) & 1);
          mbar_wait(&tfull[ts], (i / C::kTStages) & 1);
          tc_fence_after();
          const uint32_t b_base = smem_u32(smem + s * C::kStageBytes + kChunkBytes);
          const uint32_t a_tmem = tmem + C::kAColBase + ts * 32;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_i8_ts(d_tmem, a_tmem + kk * 8, sdesc_sw128(b_base + kk * 32), idesc, (cc | kk) != 0);
          }
          mma_commit(&empty[s]);
          mma_commit(&tempty[ts]);
        }
        mma_commit(&accfull[b]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ unpack
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int i = 0;
    for (int u = u0; u < u1; ++u) {
      for (int cc = 0; cc < cpg; ++cc, ++i) {
        const int s = i % C::kStages, ts = i % C::kTStages;
        mbar_wait(&full[s], (i / C::kStages) & 1);
        mbar_wait(&tempty[ts], ((i / C::kTStages) & 1) ^ 1);
        tc_fence_after();
        const uint4* src = reinterpret_cast<const uint4*>(smem + s * C::kStageBytes);
        uint32_t v[32];
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const uint4 w = src[jp * 128 + r];
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int m = jp * 4 + e;
            v[m] = sext_nib(ww[e] & 0x0F0F0F0Fu);
            v[16 + m] = sext_nib((ww[e] >> 4) & 0x0F0F0F0Fu);
          }
        }
        tmem_st32(tmem + lane_base + C::kAColBase + ts * 32, v);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tfull[ts]);
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3, r = q * 32 + lane, et = threadIdx.x - 256;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float acc[TMAX];
#pragma unroll
    for (int t = 0; t < TMAX; ++t) acc[t] = 0.f;
    int j = 0;
    for (int u = u0; u < u1; ++u, ++j) {
      const int tile = u / a.G, gi = u % a.G, b = j & 1;
      const int n = tile * kTileN + r;
      const float sw = a.wscale[(size_t)gi * a.n_pad + n];
      const float* asc = a.ascale + (size_t)gi * a.a_ld;
      mbar_wait(&accfull[b], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t col0 = tmem + lane_base + b * C::kAccCols;
      if (a.op == kOpDump) {
        for (int c0 = 0; c0 < a.r_pad; c0 += 8) {
          uint32_t rr[8];
          tmem_ld8(col0 + c0, rr);
          tmem_wait_ld();
          for (int e = 0; e < 8; ++e)
            a.dump[((size_t)n * a.G + gi) * a.r_pad + c0 + e] = (int32_t)rr[e];
        }
      } else {
#pragma unroll
        for (int tc = 0; tc < TMAX / 8; ++tc) {
          if (tc * 8 < a.T) {
            uint32_t rr[L][8];
#pragma unroll
            for (int l = 0; l < L; ++l) tmem_ld8(col0 + tc * 8 * L + l * 8, rr[l]);
            tmem_wait_ld();
            const float4 s0 = *reinterpret_cast<const float4*>(asc + tc * 8);
            const float4 s1 = *reinterpret_cast<const float4*>(asc + tc * 8 + 4);
            const float as[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float dv;
              if constexpr (L == 1) {
                dv = (float)(int32_t)rr[0][e];
              } else {
                // column order within the 24-column block: token-major, limb-minor
                const int cidx = e * 3;
                const int32_t d0 = (int32_t)rr[(cidx + 0) / 8][(cidx + 0) % 8];
                const int32_t d1 = (int32_t)rr[(cidx + 1) / 8][(cidx + 1) % 8];
                const int32_t d2 = (int32_t)rr[(cidx + 2) / 8][(cidx + 2) % 8];
                const long long dd = ((long long)d2 << 16) + ((long long)d1 << 8) + (long long)d0;
                dv = (float)dd;
              }
              acc[tc * 8 + e] = __fadd_rn(acc[tc * 8 + e], __fmul_rn(dv, __fmul_rn(sw, as[e])));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[b]);

      // ---- segment end: stream-K fixup + post-op
      const bool seg_end = (gi == a.G - 1) || (u == u1 - 1);
      if (!seg_end || a.op == kOpDump) continue;
      const int c_lo = cta_of_unit(tile * a.G, U, P);
      const int c_hi = cta_of_unit(tile * a.G + a.G - 1, U, P);
      if (c_hi > c_lo) {
        float* my = a.part + ((size_t)(c + tile) * TMAX) * kTileN;
#pragma unroll
        for (int t = 0; t < TMAX; ++t)
          if (t < a.T) my[t * kTileN + r] = acc[t];
        __threadfence();
        named_bar(1, 128);
        if (et == 0) {
          const int old = atomicAdd(&a.counters[tile], 1);
          *flag = (old == c_hi - c_lo);
        }
        named_bar(1, 128);
        const int last = *flag;
        named_bar(1, 128);
        if (!last) {
#pragma unroll
          for (int t = 0; t < TMAX; ++t) acc[t] = 0.f;
          continue;
        }
        __threadfence();
#pragma unroll
        for (int t = 0; t < TMAX; ++t) acc[t] = 0.f;
        for (int cc2 = c_lo; cc2 <= c_hi; ++cc2) {
          const volatile float* pp = a.part + ((size_t)(cc2 + tile) * TMAX) * kTileN;
#pragma unroll
          for (int t = 0; t < TMAX; ++t)
            if (t < a.T) acc[t] = __fadd_rn(acc[t], pp[t * kTileN + r]);
        }
        if (et == 0) a.counters[tile] = 0;
      }
      // ---------------------------------------------------------- post-ops
      const bool valid = n < a.n;
      if (a.op == kOpStore || a.op == kOpResidual) {
#pragma unroll
        for (int t = 0; t < TMAX; ++t) {
          if (t < a.T && valid) {
            float* o = a.out + (size_t)t * a.ldo + n;
            *o = (a.op == kOpResidual) ? __fadd_rn(*o, acc[t]) : acc[t];
          }
        }
      } else if (a.op == kOpSiluMul) {
#pragma unroll
        for (int t = 0; t < TMAX; ++t) {
          const float other = __shfl_xor_sync(0xffffffffu, acc[t], 1);
          if (t < a.T && valid && (r & 1) == 0)
            a.out[(size_t)t * a.ldo + (n >> 1)] = __fmul_rn(silu_ref(acc[t]), other);
        }
      } else if (a.op == kOpQkvRope) {
        const bool is_v = n >= a.n_q + a.n_k;
        const int loc = n < a.n_q ? n : (is_v ? n - a.n_q - a.n_k : n - a.n_q);
        const int d = loc % a.hd, head = loc / a.hd, half = a.hd >> 1, ip = d >> 1;
        const bool odd = (d & 1) != 0;
#pragma unroll
        for (int t = 0; t < TMAX; ++t) {
          const float other = __shfl_xor_sync(0xffffffffu, acc[t], 1);
          if (t < a.T && valid) {
            const int p = a.pos[t];
            float val = acc[t];
            if (!is_v) {
              // model.py:243-252: even' = e*c - o*s ; odd' = e*s + o*c
              const float cs = a.rope_cos[(size_t)p * half + ip], sn = a.rope_sin[(size_t)p * half + ip];
              const float e = odd ? other : acc[t], o = odd ? acc[t] : other;
              val = odd ? __fadd_rn(__fmul_rn(e, sn), __fmul_rn(o, cs)) : __fsub_rn(__fmul_rn(e, cs), __fmul_rn(o, sn));
            }
            if (n < a.n_q) {
              a.out[(size_t)t * a.ldo + n] = val;
            } else {
              const int sl = a.slot[t];
              const int pg = a.block_table[(size_t)sl * a.bt_ld + p / a.page];
              const size_t off = (((size_t)pg * a.n_kv_heads + head) * a.page + (p % a.page)) * a.hd + d;
              (is_v ? a.vcache : a.kcache)[off] = val;
            }
          }
        }
      } else if (a.op == kOpLogits) {
        // store logits, then first-index argmax over this tile, then over tiles
#pragma unroll
        for (int t = 0; t < TMAX; ++t) {
          if (t < a.T) {
            if (a.out != nullptr && valid) a.out[(size_t)t * a.ldo + n] = acc[t];
            float bv = valid ? acc[t] : -INFINITY;
            int bi = valid ? n : 0x7fffffff;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
              if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) { red_val[q * TMAX + t] = bv; red_idx[q * TMAX + t] = bi; }
          }
        }
        named_bar(1, 128);
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
        named_bar(1, 128);
        if (et == 0) {
          const int old = atomicAdd(&a.counters[a.n_tiles], 1);
          *flag = (old == a.n_tiles - 1);
        }
        named_bar(1, 128);
        const int last = *flag;
        named_bar(1, 128);
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
#pragma unroll
      for (int t = 0; t < TMAX; ++t) acc[t] = 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

template <int L, int TMAX>
static cudaError_t launch_linear_t(const LinearArgs& a, cudaStream_t st) {
  using C = LinCfg<L, TMAX>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(linear_tc_kernel<L, TMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  linear_tc_kernel<L, TMAX><<<a.n_cta, 384, C::kSmemBytes, st>>>(a);
  return cudaGetLastError();
}

int linear_tmax_bucket(int T) { return T <= 8 ? 8 : T <= 16 ? 16 : T <= 32 ? 32 : 64; }

cudaError_t launch_linear(int L, const LinearArgs& a, cudaStream_t st) {
  const int tm = linear_tmax_bucket(a.T);
  if (L == 1) {
    switch (tm) {
      case 8: return launch_linear_t<1, 8>(a, st);
      case 16: return launch_linear_t<1, 16>(a, st);
      case 32: return launch_linear_t<1, 32>(a, st);
      default: return launch_linear_t<1, 64>(a, st);
    }
  }
  switch (tm) {
    case 8: return launch_linear_t<3, 8>(a, st);
    case 16: return launch_linear_t<3, 16>(a, st);
    case 32: return launch_linear_t<3, 32>(a, st);
    default: return launch_linear_t<3, 64>(a, st);
  }
}

}  // namespace qs
