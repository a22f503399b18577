// Activation operand producer (K1 + K4 + K7 fused): optional embedding gather,
// optional RMSNorm, optional split-KV attention combine, then per-(token, group)
// quantisation into the 128B-swizzled int8 image the tensor-core linear streams.
//
//   draft  (L=1): reference activation quantiser, bit-exact given the same fp32
//                 input (quant.py:163-194): m = max|x|, snap m <- f32(7*f32(m/7)),
//                 s = m/7, c = clip(rint(x/s), -8, 7), s == 0 -> c = 0.
//   verify (L=3): X = rint(x * 2^e), e = 22 - exponent(max|x|); three signed
//                 byte limbs X = l2*2^16 + l1*2^8 + l0, ascale = 2^-e.
// RMSNorm follows numerics.py:46-62: y = (x * (1/sqrt(mean(x^2)+eps))) * w.
//
// Grid: (token, block of kGroupsPerCta groups), 32 threads per group.  A CTA
// that needs RMSNorm re-reads the whole row for the sum of squares (L2-resident,
// numpy's pairwise order, so every CTA of a token computes the reference's scale
// bit for bit).
#include "pack_dev.cuh"

namespace qs {

constexpr int kGroupsPerCta = 4;
constexpr int kPackThreads = 32 * kGroupsPerCta;

template <int L, bool kPlain, bool kAttPlain>
__global__ void __launch_bounds__(kPackThreads) act_pack_kernel(const PackArgs a) {
  __shared__ float red[132];
  KTraceScope kts(a.kt);
  pdl_launch_dependents();
  pdl_wait();
  const int t = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float inv = 1.0f;
  if (a.rms_w != nullptr) inv = token_inv_rms(a, t, tid, kPackThreads, 1, red);
  const int gi = blockIdx.y * kGroupsPerCta + warp;
  if (gi >= a.G) return;
  pack_group<L, kPlain, kAttPlain>(a, t, gi, inv, lane);
}

cudaError_t launch_act_pack(int L, const PackArgs& a, cudaStream_t st) {
  if (a.gp > 512) return cudaErrorInvalidValue;
  const dim3 grid(a.T, (a.G + kGroupsPerCta - 1) / kGroupsPerCta);
  const bool lean = (a.g & 3) == 0 && a.gp == 128 && a.g <= 128;
  if (lean && a.att_o == nullptr) {
    if (L == 1) return launch_k(act_pack_kernel<1, true, false>, grid, dim3(kPackThreads), 0, st, a);
    return launch_k(act_pack_kernel<3, true, false>, grid, dim3(kPackThreads), 0, st, a);
  }
  if (lean && (a.att_hd & 3) == 0) {
    if (L == 1) return launch_k(act_pack_kernel<1, false, true>, grid, dim3(kPackThreads), 0, st, a);
    return launch_k(act_pack_kernel<3, false, true>, grid, dim3(kPackThreads), 0, st, a);
  }
  if (L == 1) return launch_k(act_pack_kernel<1, false, false>, grid, dim3(kPackThreads), 0, st, a);
  return launch_k(act_pack_kernel<3, false, false>, grid, dim3(kPackThreads), 0, st, a);
}

// qs_hadamard_rows: one warp per (row, 128-block), in place (the weight rotation of the
// opt-in ModelConfig.hadamard, and the standalone API's activation rotation)
__global__ void __launch_bounds__(256) hadamard_rows_kernel(float* __restrict__ x, long long blocks) {
  const long long b = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= blocks) return;
  float4* p = reinterpret_cast<float4*>(x + b * 128) + lane;
  const float4 in = *p;
  float v[4] = {in.x, in.y, in.z, in.w};
  wht128_warp(v, lane);
  *p = make_float4(v[0], v[1], v[2], v[3]);
}

cudaError_t launch_hadamard_rows(float* x, long long rows, int cols, cudaStream_t st) {
  const long long blocks = rows * (cols / 128);
  hadamard_rows_kernel<<<(unsigned)((blocks + 7) / 8), 256, 0, st>>>(x, blocks);
  return cudaGetLastError();
}

}  // namespace qs
