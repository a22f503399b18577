// Weight construction on the device (K10): the reference's seeded 64-bit LCG
// (storage.py:62-101, 135-149) with per-thread jump-ahead, followed by the
// group-wise int4 quantiser (quant.py:163-218), written straight into the
// chunk layout the tensor-core linear streams.  Bit-exact with the reference:
// draws, the f32(1/sqrt(d)) multiply, max-abs snap, IEEE division and
// round-half-even are all reproduced with explicit _rn intrinsics.
#include "ptx.cuh"
#include "qs_common.cuh"

namespace qs {

constexpr unsigned long long kLcgMul = 6364136223846793005ull;
constexpr unsigned long long kLcgInc = 1442695040888963407ull;

__host__ __device__ inline unsigned long long lcg_jump(unsigned long long state, unsigned long long n) {
  unsigned long long mul = kLcgMul, inc = kLcgInc, am = 1, ai = 0;
  while (n) {
    if (n & 1ull) { am = am * mul; ai = ai * mul + inc; }
    inc = inc * mul + inc;
    mul = mul * mul;
    n >>= 1;
  }
  return am * state + ai;
}

__device__ __forceinline__ float lcg_float(unsigned long long st) {
  // storage.py:83-85: f32(state >> 40) / 2^23 - 1
  return __fsub_rn(__fdiv_rn((float)(unsigned)(st >> 40), 8388608.0f), 1.0f);
}



__global__ void quantize_weight_kernel(const QuantWArgs a) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)a.rows * a.G;
  if (idx >= total) return;
  const int n = (int)(idx / a.G), gi = (int)(idx % a.G);
  const long long e0 = (long long)n * a.cols + (long long)gi * a.g;
  const int g = a.g;
  // pass 1: group max (quant.py:179-194)
  float m = 0.f;
  unsigned long long st0 = 0;
  if (a.src == nullptr) st0 = lcg_jump(a.seed, a.offset + (unsigned long long)e0);
  {
    unsigned long long st = st0;
    for (int o = 0; o < g; ++o) {
      float w;
      if (a.src) {
        w = a.src[e0 + o];
      } else {
        st = st * kLcgMul + kLcgInc;
        w = __fmul_rn(lcg_float(st), a.scale);
      }
      m = fmaxf(m, fabsf(w));
    }
  }
  for (int it = 0; it < 8; ++it) {
    const float nx = __fmul_rn(7.0f, __fdiv_rn(m, 7.0f));
    if (nx == m) break;
    m = nx;
  }
  const float s = __fdiv_rn(m, 7.0f);
  const int dst_row = a.row_off + n * a.row_stride;
  const int tile = dst_row / kTileN, r = dst_row % kTileN;
  const int cpg = a.gp / kChunkK;
  for (int cc = 0; cc < cpg; ++cc)  // scales per 128-wide chunk, tile-major [n_tiles][n_chunks][128]
    a.scales[((size_t)tile * a.n_chunks + gi * cpg + cc) * kTileN + r] = s;
  if (a.ref_scales) a.ref_scales[(size_t)n * a.G + gi] = s;
  // pass 2: codes -> chunk layout.  Padded positions (o >= g) stay zero (buffer pre-zeroed).
  unsigned long long st = st0;
  uint8_t prev_ref = 0;
  for (int o = 0; o < g; ++o) {
    float w;
    if (a.src) {
      w = a.src[e0 + o];
    } else {
      st = st * kLcgMul + kLcgInc;
      w = __fmul_rn(lcg_float(st), a.scale);
    }
    int c = 0;
    if (s != 0.f) c = (int)fminf(fmaxf(rintf(__fdiv_rn(w, s)), -8.0f), 7.0f);
    const uint32_t nib = (uint32_t)c & 0xFu;     // reference nibble (two's complement)
    const uint32_t dnib = nib ^ 0x8u;            // device nibble: offset binary, code + 8
    const int kp = gi * a.gp + o;
    const int ch = kp >> 7, kl = kp & 127;
    const int pb = kl & 63, hi = kl >> 6;
    const int piece = pb >> 4, b = pb & 15;
    uint8_t* dst = a.codes + ((((size_t)tile * a.n_chunks + ch) * 4 + piece) * kTileN + r) * 16 + b;
    // each (row, chunk) byte is owned by exactly this thread: plain RMW is safe
    *dst = (uint8_t)(hi ? ((*dst & 0x0F) | (dnib << 4)) : ((*dst & 0xF0) | dnib));
    if (a.ref_codes) {
      const long long fe = e0 + o;
      if (fe & 1) {
        a.ref_codes[fe >> 1] = (uint8_t)(prev_ref | (nib << 4));
      } else {
        prev_ref = (uint8_t)nib;
        if (o == g - 1) a.ref_codes[fe >> 1] = prev_ref;  // odd-sized tail (pairs straddling groups)
      }
    }
  }
}

__global__ void lcg_fill_kernel(float* out, unsigned long long seed, unsigned long long offset, long long count,
                                float scale, int per_thread) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long e0 = t * per_thread;
  if (e0 >= count) return;
  unsigned long long st = lcg_jump(seed, offset + (unsigned long long)e0);
  const long long e1 = min(count, e0 + per_thread);
  for (long long e = e0; e < e1; ++e) {
    st = st * kLcgMul + kLcgInc;
    out[e] = __fmul_rn(lcg_float(st), scale);
  }
}

// reference packed codes + scales -> chunk layout (checkpoint load path)
__global__ void repack_ref_kernel(const uint8_t* ref_codes, const float* ref_scales, int rows, int cols, int g,
                                  uint8_t* codes, float* scales, int n_pad, int n_chunks, int gp, int G,
                                  int row_off, int row_stride) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * G) return;
  const int n = (int)(idx / G), gi = (int)(idx % G);
  const int dst_row = row_off + n * row_stride;
  const int tile = dst_row / kTileN, r = dst_row % kTileN;
  const int cpg = gp / kChunkK;
  for (int cc = 0; cc < cpg; ++cc)
    scales[((size_t)tile * n_chunks + gi * cpg + cc) * kTileN + r] = ref_scales[(size_t)n * G + gi];
  for (int o = 0; o < g; ++o) {
    const long long fe = (long long)n * cols + (long long)gi * g + o;
    const uint8_t byte = ref_codes[fe >> 1];
    const uint32_t nib = ((fe & 1) ? (byte >> 4) : (byte & 0xF)) ^ 0x8u;  // -> offset binary
    const int kp = gi * gp + o;
    const int ch = kp >> 7, kl = kp & 127;
    const int pb = kl & 63, hi = kl >> 6;
    uint8_t* dst = codes + ((((size_t)tile * n_chunks + ch) * 4 + (pb >> 4)) * kTileN + r) * 16 + (pb & 15);
    *dst = (uint8_t)(hi ? ((*dst & 0x0F) | (nib << 4)) : ((*dst & 0xF0) | nib));
  }
}

cudaError_t launch_quantize_weight(const QuantWArgs& a, cudaStream_t st) {
  const long long total = (long long)a.rows * a.G;
  const int bs = 128;
  quantize_weight_kernel<<<(unsigned)((total + bs - 1) / bs), bs, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lcg_fill(float* out, unsigned long long seed, unsigned long long offset, long long count,
                            float scale, cudaStream_t st) {
  const int per = 64, bs = 256;
  const long long threads = (count + per - 1) / per;
  lcg_fill_kernel<<<(unsigned)((threads + bs - 1) / bs), bs, 0, st>>>(out, seed, offset, count, scale, per);
  return cudaGetLastError();
}

cudaError_t launch_repack_ref(const uint8_t* ref_codes, const float* ref_scales, int rows, int cols, int g,
                              uint8_t* codes, float* scales, int n_pad, int n_chunks, int gp, int G, int row_off,
                              int row_stride, cudaStream_t st) {
  const long long total = (long long)rows * G;
  repack_ref_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(ref_codes, ref_scales, rows, cols, g, codes,
                                                                     scales, n_pad, n_chunks, gp, G, row_off,
                                                                     row_stride);
  return cudaGetLastError();
}

}  // namespace qs
