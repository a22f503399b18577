// Decode / verify attention over the shared paged fp32 KV cache (K6).
//
// One CTA per (query block, kv head): a query block is a run of consecutive
// tokens of one sequence (1 token for a draft step, gamma+1 for a verify, a
// prompt chunk for prefill), so K and V of the sequence are read once per CTA
// and shared by all its queries and the GQA heads mapped to this kv head.
// Per query the arithmetic follows model.py:322-330 and is independent of how
// many queries share the CTA (batch invariance):
//   s_j = (sum_d q_d k_jd, ascending d, no FMA) * f32(1/sqrt(hd))
//   p_j = exp(s_j - max) / sum(exp(...))        (numerics.py:73-78)
//   o_d = sum_j p_j v_jd, ascending j, no FMA
#include "ptx.cuh"
#include "qs_common.cuh"

namespace qs {

constexpr int kAttnKeys = 32;  // key rows staged per smem tile
constexpr int kAttnMaxAcc = 32;

__global__ void __launch_bounds__(256) attention_kernel(const AttnArgs a) {
  extern __shared__ float sm[];
  const int blk = blockIdx.x, kvh = blockIdx.y, tid = threadIdx.x;
  const int ntok = a.blk_ntok[blk];
  if (ntok <= 0) return;
  const int tok0 = a.blk_tok0[blk];
  const int hd = a.hd, hpk = a.hpk, Q = ntok * hpk;
  const int ld_kv = hd + 1;
  float* qv = sm;                                // [Q][hd]
  float* kt = qv + a.qmax * hpk * hd;            // [kAttnKeys][hd+1]
  float* sc = kt + kAttnKeys * ld_kv;            // [Q][ctx_cap]
  __shared__ int ctx_s[64];

  const int sl = a.slot[tok0];
  const int* bt = a.block_table + (size_t)sl * a.bt_ld;
  int cmax = 0;
  for (int i = 0; i < ntok; ++i) cmax = max(cmax, a.pos[tok0 + i] + 1);
  if (tid < Q) ctx_s[tid] = a.pos[tok0 + tid / hpk] + 1;
  for (int e = tid; e < Q * hd; e += blockDim.x) {
    const int qi = e / hd, d = e % hd;
    const int i = qi / hpk, h = kvh * hpk + qi % hpk;
    qv[e] = a.q[(size_t)(tok0 + i) * a.ldq + (size_t)h * hd + d];
  }
  __syncthreads();

  // ---- scores
  for (int j0 = 0; j0 < cmax; j0 += kAttnKeys) {
    const int nk = min(kAttnKeys, cmax - j0);
    for (int e = tid; e < nk * hd; e += blockDim.x) {
      const int jj = e / hd, d = e % hd, j = j0 + jj;
      const int pg = bt[j / a.page];
      kt[jj * ld_kv + d] = a.kcache[(((size_t)pg * a.KV + kvh) * a.page + (j % a.page)) * hd + d];
    }
    __syncthreads();
    for (int e = tid; e < Q * kAttnKeys; e += blockDim.x) {
      const int qi = e / kAttnKeys, jj = e % kAttnKeys, j = j0 + jj;
      if (jj < nk && j < ctx_s[qi]) {
        const float* qq = qv + qi * hd;
        const float* kk = kt + jj * ld_kv;
        float acc = 0.f;
        for (int d = 0; d < hd; ++d) acc = __fadd_rn(acc, __fmul_rn(qq[d], kk[d]));
        sc[(size_t)qi * a.ctx_cap + j] = __fmul_rn(acc, a.inv_sqrt_hd);
      }
    }
    __syncthreads();
  }

  // ---- softmax per query (one warp per query)
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  for (int qi = warp; qi < Q; qi += nw) {
    float* s = sc + (size_t)qi * a.ctx_cap;
    const int n = ctx_s[qi];
    float m = -INFINITY;
    for (int j = lane; j < n; j += 32) m = fmaxf(m, s[j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float z = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float e = expf(__fsub_rn(s[j], m));
      s[j] = e;
      z = __fadd_rn(z, e);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) z = __fadd_rn(z, __shfl_xor_sync(0xffffffffu, z, off));
    for (int j = lane; j < n; j += 32) s[j] = __fdiv_rn(s[j], z);
  }
  __syncthreads();

  // ---- P . V
  float acc[kAttnMaxAcc];
#pragma unroll
  for (int k = 0; k < kAttnMaxAcc; ++k) acc[k] = 0.f;
  const int n_own = (Q * hd + blockDim.x - 1) / blockDim.x;
  for (int j0 = 0; j0 < cmax; j0 += kAttnKeys) {
    const int nk = min(kAttnKeys, cmax - j0);
    for (int e = tid; e < nk * hd; e += blockDim.x) {
      const int jj = e / hd, d = e % hd, j = j0 + jj;
      const int pg = bt[j / a.page];
      kt[jj * ld_kv + d] = a.vcache[(((size_t)pg * a.KV + kvh) * a.page + (j % a.page)) * hd + d];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kAttnMaxAcc; ++k) {
      if (k < n_own) {
        const int e = tid + k * blockDim.x;
        if (e < Q * hd) {
          const int qi = e / hd, d = e % hd;
          const int lim = min(nk, ctx_s[qi] - j0);
          const float* p = sc + (size_t)qi * a.ctx_cap + j0;
          float v = acc[k];
          for (int jj = 0; jj < lim; ++jj) v = __fadd_rn(v, __fmul_rn(p[jj], kt[jj * ld_kv + d]));
          acc[k] = v;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < kAttnMaxAcc; ++k) {
    if (k < n_own) {
      const int e = tid + k * blockDim.x;
      if (e < Q * hd) {
        const int qi = e / hd, d = e % hd;
        const int i = qi / hpk, h = kvh * hpk + qi % hpk;
        a.out[(size_t)(tok0 + i) * a.ldo + (size_t)h * hd + d] = acc[k];
      }
    }
  }
}

size_t attention_smem_bytes(int qmax, int hpk, int hd, int ctx_cap) {
  return sizeof(float) * ((size_t)qmax * hpk * hd + (size_t)kAttnKeys * (hd + 1) + (size_t)qmax * hpk * ctx_cap);
}

cudaError_t launch_attention(const AttnArgs& a, int n_blk, cudaStream_t st) {
  const size_t smem = attention_smem_bytes(a.qmax, a.hpk, a.hd, a.ctx_cap);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  attention_kernel<<<dim3(n_blk, a.KV), 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace qs
