// Activation operand producer (K1 + K4 + K7 fused): optional embedding gather,
// optional RMSNorm, then per-(token, group) quantisation into the 128B-swizzled
// int8 image the tensor-core linear streams.
//
//   draft  (L=1): reference activation quantiser, bit-exact given the same fp32
//                 input (quant.py:163-194): m = max|x|, snap m <- f32(7*f32(m/7)),
//                 s = m/7, c = clip(rint(x/s), -8, 7), s == 0 -> c = 0.
//   verify (L=3): X = rint(x * 2^e), e = 22 - exponent(max|x|); three signed
//                 byte limbs X = l2*2^16 + l1*2^8 + l0, ascale = 2^-e.
// RMSNorm follows numerics.py:46-62: y = (x * (1/sqrt(mean(x^2)+eps))) * w.
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

__device__ __forceinline__ float block_sum_fixed(float v, float* red) {
  // deterministic: warp xor-tree, then warps summed in index order
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < nw; ++w) s = __fadd_rn(s, red[w]);
  return s;
}

template <int L>
__global__ void __launch_bounds__(256) act_pack_kernel(const PackArgs a) {
  extern __shared__ float row[];  // [K]
  __shared__ float red[32];
  const int t = blockIdx.x, tid = threadIdx.x;
  const int K = a.K;
  if (a.gather_ids != nullptr) {
    const int id = a.gather_ids[t];
    const float* src = a.emb + (size_t)id * K;
    for (int k = tid; k < K; k += blockDim.x) {
      const float v = src[k];
      row[k] = v;
      if (a.x_out) a.x_out[(size_t)t * K + k] = v;
    }
  } else {
    for (int k = tid; k < K; k += blockDim.x) row[k] = a.x[(size_t)t * a.ldx + k];
  }
  __syncthreads();
  if (a.rms_w != nullptr) {
    float part = 0.f;
    for (int k = tid; k < K; k += blockDim.x) part = __fadd_rn(part, __fmul_rn(row[k], row[k]));
    const float ss = block_sum_fixed(part, red);
    const float ms = __fdiv_rn(ss, (float)K);
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, a.eps)));
    __syncthreads();
    for (int k = tid; k < K; k += blockDim.x) row[k] = __fmul_rn(__fmul_rn(row[k], inv), a.rms_w[k]);
    __syncthreads();
  }
  if (a.y_out)
    for (int k = tid; k < K; k += blockDim.x) a.y_out[(size_t)t * K + k] = row[k];

  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const size_t chunk_stride = (size_t)a.r_pad * 128;
  for (int gi = warp; gi < a.G; gi += nw) {
    const float* gx = row + (size_t)gi * a.g;
    float m = 0.f;
    for (int o = lane; o < a.g; o += 32) m = fmaxf(m, fabsf(gx[o]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float s, mul;
    int e = 0;
    if constexpr (L == 1) {
      m = snap_group_max(m);
      s = __fdiv_rn(m, 7.0f);
      mul = s;
    } else {
      if (m > 0.f) {
        int E;
        frexpf(m, &E);
        e = 22 - E;
        mul = ldexpf(1.0f, -e);
      } else {
        mul = 0.f;
      }
      s = mul;
    }
    if (lane == 0) {
      if (a.ascale) a.ascale[(size_t)gi * a.a_ld + t] = mul;
      if (a.scales_out) a.scales_out[(size_t)t * a.G + gi] = s;
    }
    // quantise 4 consecutive (padded) positions per lane per step
    for (int o = lane * 4; o < a.gp; o += 128) {
      uint32_t w[L];
#pragma unroll
      for (int l = 0; l < L; ++l) w[l] = 0;
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4) {
        const int oo = o + e4;
        int code[L];
#pragma unroll
        for (int l = 0; l < L; ++l) code[l] = 0;
        if (oo < a.g) {
          const float x = gx[oo];
          if constexpr (L == 1) {
            float qv = 0.f;
            if (s != 0.f) qv = fminf(fmaxf(rintf(__fdiv_rn(x, s)), -8.0f), 7.0f);
            code[0] = (int)qv;
            const size_t kk = (size_t)gi * a.g + oo;
            if (a.codes_out) a.codes_out[(size_t)t * K + kk] = (int8_t)code[0];
            if (a.fq_out) a.fq_out[(size_t)t * K + kk] = __fmul_rn((float)code[0], s);
          } else {
            const int X = (m > 0.f) ? __float2int_rn(ldexpf(x, e)) : 0;
            const int l0 = ((X + 128) & 255) - 128;
            const int X1 = (X - l0) >> 8;
            const int l1 = ((X1 + 128) & 255) - 128;
            code[0] = l0;
            code[1 % L] = l1;
            code[2 % L] = (X1 - l1) >> 8;
          }
        }
#pragma unroll
        for (int l = 0; l < L; ++l) w[l] |= ((uint32_t)(code[l] & 0xFF)) << (8 * e4);
      }
      if (a.img) {
        const int kp = gi * a.gp + o;
        const int ch = kp >> 7, byte = kp & 127;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const int rr = t * L + l;
          *reinterpret_cast<uint32_t*>(a.img + ch * chunk_stride + sw128_off(rr, byte)) = w[l];
        }
      }
    }
  }
}

cudaError_t launch_act_pack(int L, const PackArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)a.K * sizeof(float);
  if (L == 1) {
    static bool attr1 = false;
    if (!attr1) {
      cudaFuncSetAttribute(act_pack_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr1 = true;
    }
    act_pack_kernel<1><<<a.T, 256, smem, st>>>(a);
  } else {
    static bool attr3 = false;
    if (!attr3) {
      cudaFuncSetAttribute(act_pack_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr3 = true;
    }
    act_pack_kernel<3><<<a.T, 256, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace qs
