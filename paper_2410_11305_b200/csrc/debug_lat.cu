// Diagnostic: memory round-trip latency of a warp issuing rounds of 8 independent
// 512-byte row loads (the split-KV attention access pattern), timed with %globaltimer.
#include "ptx.cuh"
#include "qs_common.cuh"

namespace qs {
__global__ void lat_kernel(const float* buf, size_t n_rows, int rounds, int stride_rows, unsigned long long* out,
                           int cg) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  size_t row = (size_t)blockIdx.x * 977;
  for (int r = 0; r < rounds; ++r) {
    const unsigned long long t0 = gtimer();
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t rr = (row + (size_t)u * stride_rows) % n_rows;
      const float4* p = reinterpret_cast<const float4*>(buf + rr * 128) + lane;
      v[u] = cg ? __ldcg(p) : *p;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    row += (size_t)(acc != 12345.f) * 8 * stride_rows + 13;  // data dependence on this round
    if (lane == 0 && blockIdx.x == 0) out[r] = gtimer() - t0;
  }
  if (acc == 1.2345f) out[rounds] = 1;
}
}  // namespace qs

extern "C" int qs_debug_latency(const float* buf, size_t n_rows, int rounds, int stride_rows, int n_blocks,
                                uint64_t* out, int cg, void* stream) {
  qs::lat_kernel<<<n_blocks, 32, 0, (cudaStream_t)stream>>>(buf, n_rows, rounds, stride_rows,
                                                            reinterpret_cast<unsigned long long*>(out), cg);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
