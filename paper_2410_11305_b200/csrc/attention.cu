// Decode / verify attention over the shared paged fp32 KV cache (K6), split-KV.
//
// Grid (query block, kv head, key chunk of kAttnChunk positions).  A query block
// is a run of consecutive tokens of one sequence (1 token per draft step, gamma+1
// per verify, a prompt slice for prefill), so each K/V row is fetched once per
// CTA and shared by all its queries and the GQA heads of this kv head.  Per
// (query, chunk) the CTA writes the chunk max m_c, the chunk sum l_c of
// exp(s - m_c) and the unnormalised o_c = sum_j exp(s_j - m_c) v_j; the o_proj
// operand pack (act_pack.cu) merges chunks in ascending order.
//
// Chunk boundaries are absolute positions, so a query's arithmetic depends only
// on its own context, never on how many queries share the pass (batch
// invariance).  Semantics: model.py:322-330 (scores * f32(1/sqrt(hd)), softmax
// with max subtraction, probability-weighted V), fp32 throughout.
#include "ptx.cuh"
#include "qs_common.cuh"

namespace qs {

#ifndef QS_ATTN_CHUNK
#define QS_ATTN_CHUNK 64
#endif
constexpr int kAttnChunk = QS_ATTN_CHUNK;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) { cp_async16_cg(smem, gmem); }

// Scores of keys jj = warp + 8u (u < KPW) for every query, QB queries at a time:
// per (key, query) a lane-ordered fma chain, then the xor-butterfly total of the lanes'
// partials (computed by recursive halving, see below).
template <int QB, int KPW>
__device__ __forceinline__ void score_block(const float* kt, const float* qv, float* sc, const int* ctx_s, int hd,
                                            int Q, int nk, int j0, int warp, int lane, float inv_sqrt_hd) {
  for (int q0 = 0; q0 < Q; q0 += QB) {
    float p[KPW][QB];
#pragma unroll
    for (int u = 0; u < KPW; ++u)
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) p[u][qq] = 0.f;
    for (int d = lane * 4; d < hd; d += 128) {
#pragma unroll
      for (int u = 0; u < KPW; ++u) {
        const int jj = warp + 8 * u;
        const float4 k4 = *reinterpret_cast<const float4*>(kt + jj * hd + d);
#pragma unroll
        for (int qq = 0; qq < QB; ++qq) {
          const int qi = q0 + qq < Q ? q0 + qq : Q - 1;
          const float4 q4 = *reinterpret_cast<const float4*>(qv + qi * hd + d);
          p[u][qq] = fmaf(q4.x, k4.x, p[u][qq]);
          p[u][qq] = fmaf(q4.y, k4.y, p[u][qq]);
          p[u][qq] = fmaf(q4.z, k4.z, p[u][qq]);
          p[u][qq] = fmaf(q4.w, k4.w, p[u][qq]);
        }
      }
    }
    // Reduce the NP = KPW * QB (key, query) partials across the lanes.  The reference
    // arithmetic is the xor butterfly p += shfl_xor(p, 16), 8, 4, 2, 1 (every lane ends
    // with every pair's total); here the levels with offset >= NP stay butterflies and the
    // rest are recursive halving -- at offset o a lane keeps the half of its pairs selected
    // by its lane bit o and adds the partner's value of the same pair, which is exactly the
    // butterfly's v_l + v_(l^o) for the pairs it keeps.  Lane l ends with pair l % NP:
    // bit-identical totals for ~31 shuffles per lane instead of 5 * NP.
    constexpr int NP = KPW * QB;
    static_assert((NP & (NP - 1)) == 0 && NP <= 32, "pairs per warp: a power of two <= 32");
    float v[NP];
#pragma unroll
    for (int u = 0; u < KPW; ++u)
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) v[u * QB + qq] = p[u][qq];
#pragma unroll
    for (int off = 16; off >= NP; off >>= 1)
#pragma unroll
      for (int i = 0; i < NP; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
#pragma unroll
    for (int n = NP; n > 1; n >>= 1) {
      const int h = n >> 1;
      const bool hi = (lane & h) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const float keep = hi ? v[i + h] : v[i], send = hi ? v[i] : v[i + h];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
      }
    }
    if (lane < NP) {
      const int u = lane / QB, qq = lane % QB;
      const int jj = warp + 8 * u, j = j0 + jj, qi = q0 + qq;
      if (jj < nk && qi < Q) sc[qi * kAttnChunk + jj] = (j < ctx_s[qi]) ? v[0] * inv_sqrt_hd : -INFINITY;
    }
  }
}

__global__ void __launch_bounds__(256) attn_partial_kernel(const AttnArgs a) {
  extern __shared__ __align__(16) float sm[];
  KTraceScope kts(a.kt);
  pdl_launch_dependents();
  pdl_wait();
  const int blk = blockIdx.x, kvh = blockIdx.y, ch = blockIdx.z, tid = threadIdx.x;
  // the prologue is a chain of dependent global round trips: block -> positions + slot
  // -> page table -> K / V rows; each level's loads are issued together
  // uniform blocks (blk_tok0 == nullptr, the decode engine's batches): no block-table load
  const int ntok = a.blk_tok0 ? a.blk_ntok[blk] : a.qmax, tok0 = a.blk_tok0 ? a.blk_tok0[blk] : blk * a.qmax;
  if (ntok <= 0) return;
  const int j0 = ch * kAttnChunk;
  const int sl = a.slot[tok0];
  int cmax = 0;
  for (int i = 0; i < ntok; ++i) cmax = max(cmax, a.pos[tok0 + i] + 1);
  if (j0 >= cmax) return;
  const int nk = min(kAttnChunk, cmax - j0);
  const int hd = a.hd, hpk = a.hpk, Q = ntok * hpk, H = a.H;
  float* qv = sm;                             // [Q][hd]
  float* kt = qv + a.qmax * hpk * hd;         // [chunk][hd]
  float* vt = kt + kAttnChunk * hd;           // [chunk][hd]
  float* sc = vt + kAttnChunk * hd;           // [Q][chunk]
  __shared__ int ctx_s[64];
  __shared__ __align__(8) uint64_t kv_bar[2];  // [0] K rows landed, [1] V rows landed

  const int* bt = a.block_table + (size_t)sl * a.bt_ld;
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  if (tid < Q) ctx_s[tid] = a.pos[tok0 + tid / hpk] + 1;
  if (tid == 0) {
    mbar_init(&kv_bar[0], 1);
    mbar_init(&kv_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // The chunk's K and V rows are runs of whole page rows, contiguous within a page
  // ([page][kv_head][row][hd]): warp 0 walks the page table once per page and issues one
  // bulk copy per (page, K|V) on two barriers, so the scores start as soon as K has
  // landed while V is still in flight.  The queries go in with 16-byte async copies.
  if (warp == 0) {
    const uint32_t bytes = (uint32_t)nk * hd * 4u;
    if (lane == 0) {
      mbar_arrive_expect_tx(&kv_bar[0], bytes);
      mbar_arrive_expect_tx(&kv_bar[1], bytes);
    }
    __syncwarp();
    const int ps = __ffs(a.page) - 1;  // page is a power of two (qs_forward checks)
    const int p_first = j0 >> ps, p_last = (j0 + nk - 1) >> ps;
    for (int pi = p_first + lane; pi <= p_last; pi += 32) {
      const int r0 = max(j0, pi * a.page), r1 = min(j0 + nk, (pi + 1) * a.page);
      const size_t off = (((size_t)bt[pi] * a.KV + kvh) * a.page + (r0 - pi * a.page)) * hd;
      const uint32_t nb = (uint32_t)(r1 - r0) * hd * 4u;
      bulk_g2s(kt + (r0 - j0) * hd, a.kcache + off, nb, &kv_bar[0]);
      bulk_g2s(vt + (r0 - j0) * hd, a.vcache + off, nb, &kv_bar[1]);
    }
  }
  const int hd4 = hd >> 2;
  const int hs = (hd >= 4 && (hd & (hd - 1)) == 0) ? __ffs(hd) - 1 : -1;  // head_dim shift (power of two)
  for (int e = tid; e < Q * hd4; e += blockDim.x) {
    const int qi = hs >= 0 ? e >> (hs - 2) : e / hd4, d4 = e - qi * hd4;
    const int i = qi / hpk, h = kvh * hpk + qi % hpk;
    cp_async16(qv + qi * hd + d4 * 4, a.q + (size_t)(tok0 + i) * a.ldq + (size_t)h * hd + d4 * 4);
  }
  cp_async_wait_all();
  __syncthreads();
  mbar_wait(&kv_bar[0], 0);

  // ---- scores: warp per key, lanes split the head dimension, all queries.  Each
  // warp owns keys jj = warp + nw*u; the (key, query) dot products of a 4-query block
  // are independent, so their xor trees are interleaved (same per-pair arithmetic:
  // lane-ordered fma chain, then p += shfl_xor(p, 16..1)).
  constexpr int kKPW = kAttnChunk / 8;  // keys per warp at 8 warps
  if (nw == 8) {
    if (Q == 1)
      score_block<1, kKPW>(kt, qv, sc, ctx_s, hd, Q, nk, j0, warp, lane, a.inv_sqrt_hd);
    else
      score_block<4, kKPW>(kt, qv, sc, ctx_s, hd, Q, nk, j0, warp, lane, a.inv_sqrt_hd);
  } else {
    for (int jj = warp; jj < nk; jj += nw) {
      const int j = j0 + jj;
      for (int qi = 0; qi < Q; ++qi) {
        float p = 0.f;
        for (int d = lane * 4; d < hd; d += 128) {
          const float4 k4 = *reinterpret_cast<const float4*>(kt + jj * hd + d);
          const float4 q4 = *reinterpret_cast<const float4*>(qv + qi * hd + d);
          p = fmaf(q4.x, k4.x, p);
          p = fmaf(q4.y, k4.y, p);
          p = fmaf(q4.z, k4.z, p);
          p = fmaf(q4.w, k4.w, p);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        if (lane == 0) sc[qi * kAttnChunk + jj] = (j < ctx_s[qi]) ? p * a.inv_sqrt_hd : -INFINITY;
      }
    }
  }
  __syncthreads();

  // ---- chunk-local softmax statistics (warp per query)
  for (int qi = warp; qi < Q; qi += nw) {
    float* s = sc + qi * kAttnChunk;
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
      float2* ml = reinterpret_cast<float2*>(a.part_ml) + ((size_t)(tok0 + i) * H + h) * a.cmax + ch;
      *ml = make_float2(m, l);
    }
  }
  __syncthreads();

  // ---- o_c = sum_j p_j v_j: per (query, dim) one sequential fma chain over the chunk's
  // keys.  Thread (g, d) owns dim d of queries g, g + G, ... (G = 256 / hd), four at a
  // time, so each V element is read once per four queries and the probabilities four keys
  // per 16-byte load; the chains themselves are unchanged.
  mbar_wait(&kv_bar[1], 0);
  if (hd <= (int)blockDim.x && blockDim.x % hd == 0) {
    const int G = blockDim.x / hd, g = tid / hd, d = tid - g * hd;
    if (Q <= G) {  // one query per thread (decode steps): a single chain
      if (g < Q) {
        const float* pq = sc + g * kAttnChunk;
        float acc = 0.f;
        int jj = 0;
        for (; jj + 4 <= nk; jj += 4) {
          const float4 pp = *reinterpret_cast<const float4*>(pq + jj);
          acc = fmaf(pp.x, vt[jj * hd + d], acc);
          acc = fmaf(pp.y, vt[(jj + 1) * hd + d], acc);
          acc = fmaf(pp.z, vt[(jj + 2) * hd + d], acc);
          acc = fmaf(pp.w, vt[(jj + 3) * hd + d], acc);
        }
        for (; jj < nk; ++jj) acc = fmaf(pq[jj], vt[jj * hd + d], acc);
        const int i = g / hpk, h = kvh * hpk + g % hpk;
        a.part_o[(((size_t)(tok0 + i) * H + h) * a.cmax + ch) * hd + d] = acc;
      }
    } else
    for (int q0 = g; q0 < Q; q0 += 4 * G) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* pr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) pr[u] = sc + min(q0 + u * G, Q - 1) * kAttnChunk;
      int jj = 0;
      for (; jj + 4 <= nk; jj += 4) {
        const float v0 = vt[jj * hd + d], v1 = vt[(jj + 1) * hd + d], v2 = vt[(jj + 2) * hd + d],
                    v3 = vt[(jj + 3) * hd + d];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 pp = *reinterpret_cast<const float4*>(pr[u] + jj);
          acc[u] = fmaf(pp.x, v0, acc[u]);
          acc[u] = fmaf(pp.y, v1, acc[u]);
          acc[u] = fmaf(pp.z, v2, acc[u]);
          acc[u] = fmaf(pp.w, v3, acc[u]);
        }
      }
      for (; jj < nk; ++jj) {
        const float vj = vt[jj * hd + d];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = fmaf(pr[u][jj], vj, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int qi = q0 + u * G;
        if (qi < Q) {
          const int i = qi / hpk, h = kvh * hpk + qi % hpk;
          a.part_o[(((size_t)(tok0 + i) * H + h) * a.cmax + ch) * hd + d] = acc[u];
        }
      }
    }
  } else {
    for (int e = tid; e < Q * hd; e += blockDim.x) {
      const int qi = hs >= 0 ? e >> hs : e / hd, d = e - qi * hd;
      const float* p = sc + qi * kAttnChunk;
      float acc = 0.f;
      for (int jj = 0; jj < nk; ++jj) acc = fmaf(p[jj], vt[jj * hd + d], acc);
      const int i = qi / hpk, h = kvh * hpk + qi % hpk;
      a.part_o[(((size_t)(tok0 + i) * H + h) * a.cmax + ch) * hd + d] = acc;
    }
  }
}

size_t attention_smem_bytes(int qmax, int hpk, int hd, int ctx_cap) {
  (void)ctx_cap;
  return sizeof(float) * ((size_t)qmax * hpk * hd + 2 * (size_t)kAttnChunk * hd + (size_t)qmax * hpk * kAttnChunk);
}

int attention_chunks(int ctx_cap) { return (ctx_cap + kAttnChunk - 1) / kAttnChunk; }
int attention_chunk_len() { return kAttnChunk; }

cudaError_t launch_attention(const AttnArgs& a, int n_blk, cudaStream_t st) {
  const size_t smem = attention_smem_bytes(a.qmax, a.hpk, a.hd, a.ctx_cap);
  static size_t attr[kMaxDevices] = {};  // the attribute is per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  // static shared memory (ctx_s, row_s) comes on top of the dynamic bytes: opt in above
  // 47 KB, not at 48 KB exactly (a 32-query block of head_dim 64 is exactly 48 KB dynamic)
  if (smem > 47 * 1024 && (dev >= kMaxDevices || smem > attr[dev])) {
    e = cudaFuncSetAttribute(attn_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev < kMaxDevices) attr[dev] = smem;
  }
  return launch_k(attn_partial_kernel, dim3(n_blk, a.KV, attention_chunks(a.ctx_cap)), dim3(256), smem, st, a);
}

}  // namespace qs
