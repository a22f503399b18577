// Microbenchmark (research tool, not part of the product library): issue rate of
// tcgen05.mma.kind::i8 with A in TMEM, 1-SM (M=128) vs 2-SM pair (M=256), vs N.
// Data is zero; only the time per instruction matters.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2410_11305_b200/csrc/ptx.cuh"

using namespace qs;

__device__ const uint8_t* g_src;
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int CG, int ST>
__global__ void __launch_bounds__(256, 1) mma_rate_kernel(int reps, unsigned long long* out, int* stop) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  constexpr int kBRows = CG == 2 ? N / 2 : N;  // each CTA of a pair holds half of B
  for (int i = tid; i < kBRows * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      tmem_alloc<512>(&tslot);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool leader = CG == 1 || cluster_rank() == 0;
  if (ST == 2 && warp == 4) {  // concurrent TMA traffic: 32 KB bulk copies global -> smem, back to back
    __shared__ uint64_t cbar;
    uint8_t* dst = sm + 64 * 1024;
    if (lane_id() == 0) {
      mbar_init(&cbar, 1);
      fence_mbar_init();
      volatile int* vs = stop;
      uint32_t ph = 0;
      int n = 0;
      const unsigned long long ts0 = gtimer();
      while (*vs == 0 && gtimer() - ts0 < 2000000000ull) {
        mbar_arrive_expect_tx(&cbar, 32768);
        bulk_g2s(dst, g_src + (size_t)((blockIdx.x * 7 + n) % 64) * 32768, 32768, &cbar);
        mbar_wait(&cbar, ph);
        ph ^= 1;
        ++n;
      }
      out[148 + blockIdx.x * 4] = n;
    }
  }
  if (ST == 1 && warp >= 4 && warp < 8) {  // concurrent A staging traffic: tcgen05.st 32x32b.x32 into cols [128, 256)
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i;
    volatile int* vs = stop;
    const unsigned long long ts0 = gtimer();
    int n = 0;
    while (*vs == 0 && gtimer() - ts0 < 2000000000ull) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st32(tmem + lane_base + 128 + c * 32, v);
      tmem_wait_st();
      ++n;
    }
    if ((tid & 31) == 0) out[148 + blockIdx.x * 4 + (warp & 3)] = n;
  }
  if (warp == 0 && leader) {
    const uint64_t bdesc = sdesc_sw128(smem_u32(sm));
    const uint32_t idesc = idesc_i8(CG == 2 ? 256 : 128, N);
    const unsigned long long t0 = gtimer();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (CG == 2) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(tmem + 256 + kk * 8), "l"(bdesc + (uint64_t)(kk * 2)), "r"(idesc), "r"(kk)
              : "memory");
        } else {
          mma_i8_ts_elect(tmem, tmem + 256 + kk * 8, bdesc + (uint64_t)(kk * 2), idesc, kk);
        }
      }
    }
    if (CG == 2) {
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar))
          : "memory");
    } else {
      mma_commit_elect(&bar);
    }
    mbar_wait(&bar, 0);
    const unsigned long long t1 = gtimer();
    if (tid == 0) {
      out[blockIdx.x] = t1 - t0;
      *reinterpret_cast<volatile int*>(stop) = 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      tmem_dealloc<512>(tmem);
  }
}

// ST=3: the kernel's A staging pattern: 4 warps tcgen05.st a 32-column A slot (ring of 2),
// wait::st + fence + mbarrier arrive; the MMA warp waits, issues 4 MMAs on that slot,
// commits to the slot's "empty" barrier.  Time per slot (4 MMAs) vs the free-running rate.
template <int N, int SL, int CH>
__global__ void __launch_bounds__(256, 1) turnaround_kernel(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[SL], empty[SL];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < N * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (tid == 0) {
    for (int i = 0; i < SL; ++i) { mbar_init(&full[i], 4); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint64_t bdesc = sdesc_sw128(smem_u32(sm));
    const uint32_t idesc = idesc_i8(128, N);
    const unsigned long long t0 = gtimer();
    for (int r = 0; r < reps; ++r) {
      const int b = r % SL;
      mbar_wait(&full[b], (r / SL) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8_ts_elect(tmem + c * 8, tmem + 128 + (b * CH + c) * 32 + kk * 8, bdesc + (uint64_t)(kk * 2), idesc, kk);
      mma_commit_elect(&empty[b]);
    }
    mbar_wait(&empty[(reps - 1) % SL], ((reps - 1) / SL) & 1);
    const unsigned long long t1 = gtimer();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
  } else if (warp >= 4) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i * lane;
    for (int r = 0; r < reps; ++r) {
      const int b = r % SL;
      if (r >= SL) mbar_wait(&empty[b], ((r / SL) & 1) ^ 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < CH; ++c) tmem_st32(tmem + lane_base + 128 + (b * CH + c) * 32, v);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int SL, int CH>
static int turn(int reps, unsigned long long* out) {
  const size_t smem = 64 * 1024;
  cudaFuncSetAttribute(turnaround_kernel<8, SL, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  turnaround_kernel<8, SL, CH><<<148, 256, smem>>>(reps, out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
extern "C" int mma_turnaround(int slots, int chunks, int reps, unsigned long long* out) {
  if (slots == 2 && chunks == 1) return turn<2, 1>(reps, out);
  if (slots == 4 && chunks == 1) return turn<4, 1>(reps, out);
  if (slots == 8 && chunks == 1) return turn<8, 1>(reps, out);
  if (slots == 2 && chunks == 4) return turn<2, 4>(reps, out);
  if (slots == 3 && chunks == 4) return turn<3, 4>(reps, out);
  return -1;
}

template <int N, int CG, int ST>
static int run(int reps, unsigned long long* out, int grid, int* stop) {
  const size_t smem = 64 * 1024 + 32 * 1024 + 2048;
  cudaFuncSetAttribute(mma_rate_kernel<N, CG, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, mma_rate_kernel<N, CG, ST>, reps, out, stop);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : (int)e;
}

extern "C" int mma_set_src(const void* p) { return cudaMemcpyToSymbol(g_src, &p, sizeof(p)) == cudaSuccess ? 0 : 1; }

extern "C" int mma_rate(int n, int cg, int reps, unsigned long long* out, int grid, int st, int* stop) {
#define CASE(NN)                                                                        \
  if (n == NN) {                                                                        \
    if (st == 2) return run<NN, 1, 2>(reps, out, grid, stop);                               \
    if (st) return cg == 2 ? run<NN, 2, 1>(reps, out, grid, stop) : run<NN, 1, 1>(reps, out, grid, stop); \
    return cg == 2 ? run<NN, 2, 0>(reps, out, grid, stop) : run<NN, 1, 0>(reps, out, grid, stop); \
  }
  CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(192) CASE(256)
  return -1;
}
