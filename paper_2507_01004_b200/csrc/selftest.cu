// Diagnostic entry point: one tcgen05 MMA tile through the same descriptor /
// SW128 layout code the GLA kernels use, so a layout or encoding mistake shows
// up as a wrong 128x128 product instead of a wrong attention output.
#include "tc.cuh"
#include "zgla_internal.h"
#include "fast_common.cuh"

namespace zgla {

// A operand is M x K, B operand is K x N (math view).  Storage:
//   A K-major : a_src[M][K]      A MN-major : a_src[K][M]
//   B K-major : b_src[N][K]      B MN-major : b_src[K][N]
__global__ void __launch_bounds__(128) selftest_mma_kernel(const __nv_bfloat16* __restrict__ a_src,
                                                           const __nv_bfloat16* __restrict__ b_src,
                                                           float* __restrict__ d_out, int M, int N, int K,
                                                           int a_mn, int b_mn, int lane_off) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by offsetting the __shared__ array itself so the compiler keeps the shared address space (LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x;

  // storage shapes
  const int a_rows = a_mn ? K : M, a_cols = a_mn ? M : K;
  const int b_rows = b_mn ? K : N, b_cols = b_mn ? N : K;
  uint8_t* sa = smem;
  uint8_t* sb = smem + a_rows * a_cols * 2;  // multiples of 1024 for our shapes
  auto fill = [&](const __nv_bfloat16* src, int rows, int cols, uint8_t* dst) {
    const int chunks_per_row = cols / 8;
    for (int i = tid; i < rows * chunks_per_row; i += blockDim.x) {
      int r = i / chunks_per_row, c = i % chunks_per_row;
      int panel = c / 8, cc = c % 8;
      uint4 val = *reinterpret_cast<const uint4*>(src + r * cols + c * 8);
      *reinterpret_cast<uint4*>(dst + panel * rows * 128 + sw128(r, cc)) = val;
    }
  };
  fill(a_src, a_rows, a_cols, sa);
  fill(b_src, b_rows, b_cols, sb);
  fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) {
    tmem_alloc(&tmem_base_sh, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  const uint32_t d_tmem = tbase + (static_cast<uint32_t>(lane_off) << 16);

  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(M, N, a_mn, b_mn);
    for (int kk = 0; kk < K / 16; ++kk) {
      uint64_t ad, bd;
      if (a_mn) ad = sdesc(smem_u32(sa) + kk * 16 * 128, a_rows * 128, 1024);
      else ad = sdesc(smem_u32(sa) + (kk / 4) * a_rows * 128 + (kk % 4) * 32, 16, 1024);
      if (b_mn) bd = sdesc(smem_u32(sb) + kk * 16 * 128, b_rows * 128, 1024);
      else bd = sdesc(smem_u32(sb) + (kk / 4) * b_rows * 128 + (kk % 4) * 32, 16, 1024);
      mma_bf16_ss(d_tmem, ad, bd, idesc, kk > 0);
    }
    if (M == 64 && lane_off == 16) {
      // a second M=64 tile at lane offset 0 in the SAME columns: it must not disturb lanes
      // 16..31 of each quarter (the kernels pack two M=64 accumulators this way)
      for (int kk = 0; kk < K / 16; ++kk) {
        uint64_t ad, bd;
        if (a_mn) ad = sdesc(smem_u32(sa) + kk * 16 * 128, a_rows * 128, 1024);
        else ad = sdesc(smem_u32(sa) + (kk / 4) * a_rows * 128 + (kk % 4) * 32, 16, 1024);
        if (b_mn) bd = sdesc(smem_u32(sb) + kk * 16 * 128, b_rows * 128, 1024);
        else bd = sdesc(smem_u32(sb) + (kk / 4) * b_rows * 128 + (kk % 4) * 32, 16, 1024);
        mma_bf16_ss(tbase, ad, bd, idesc, 0u);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = tid / 32, lane = tid % 32;
  // row m of D lives in TMEM lane m (M=128) or lane (m%16)+32*(m/16) (+lane_off) (M=64)
  int row;
  if (M == 128) row = warp * 32 + lane;
  else row = (lane >= lane_off && lane < lane_off + 16) ? warp * 16 + (lane - lane_off) : -1;
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(taddr(tbase, warp * 32, c0), v);
    if (row >= 0)
      for (int j = 0; j < 32; ++j) d_out[row * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tbase, 256);
}

}  // namespace zgla

extern "C" int zgla_selftest_mma(const void* a, const void* b, float* d, int M, int N, int K, int a_mn, int b_mn,
                                 int lane_off, void* stream) {
  using namespace zgla;
  if (!((M == 64 || M == 128) && N % 16 == 0 && N <= 256 && K % 64 == 0 && (M == 64 || lane_off == 0)))
    return ZGLA_ERR_DIMS;
  size_t smem = 1024 + (size_t)M * K * 2 + (size_t)N * K * 2;
  cudaFuncSetAttribute(selftest_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  selftest_mma_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)a, (const __nv_bfloat16*)b, d, M, N, K, a_mn, b_mn, lane_off);
  return zgla_check_launch();
}

// ---------------------------------------------------------------------------
// Diagnostic: TMA streaming rate.  Every CTA streams `tiles_per_cta` tiles of
// [64 rows x 128 bf16] (2 boxes of 64x64, 16 KiB) x `boxes_per_stage/2` tensors
// through `ns` shared-memory stages; one consumer thread waits and releases.
namespace zgla {
__global__ void __launch_bounds__(64) selftest_stream_kernel(const __grid_constant__ CUtensorMap tm, int rows_total,
                                                             int tiles_per_cta, int ns, int tensors, int prefetch) {
  extern __shared__ uint8_t smem_raw[];
  // align by offsetting the __shared__ array itself so the compiler keeps the shared address space (LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stage_bytes = tensors * 16384;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ns * stage_bytes);
  uint64_t* empty = full + 8;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int base_row = blockIdx.x * tiles_per_cta * 64;
  if (tid == 0) {
    for (int i = 0; i < tiles_per_cta + prefetch; ++i) {
      if (prefetch && i < tiles_per_cta)
        for (int t = 0; t < tensors; ++t) {
          const int r = t * (rows_total / tensors) + base_row + i * 64;
          tma_prefetch_2d(&tm, 0, r);
          tma_prefetch_2d(&tm, 64, r);
        }
      const int j = i - prefetch;
      if (j < 0) continue;
      const int st = j % ns, ph = (j / ns) & 1;
      mbar_wait(&empty[st], ph ^ 1);
      mbar_arrive_expect_tx(&full[st], stage_bytes);
      for (int t = 0; t < tensors; ++t) {
        const int r = t * (rows_total / tensors) + base_row + j * 64;
        tma_load_2d(smem + st * stage_bytes + t * 16384, &tm, &full[st], 0, r);
        tma_load_2d(smem + st * stage_bytes + t * 16384 + 8192, &tm, &full[st], 64, r);
      }
    }
  } else if (tid == 32) {
    for (int j = 0; j < tiles_per_cta; ++j) {
      const int st = j % ns, ph = (j / ns) & 1;
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
}
}  // namespace zgla

extern "C" int zgla_selftest_stream(const void* src, long long rows, int tiles_per_cta, int ns, int tensors,
                                    int prefetch, int ctas, void* stream) {
  using namespace zgla;
  if (ns < 1 || ns > 8 || tensors < 1) return ZGLA_ERR_CONFIG;
  CUtensorMap m;
  if (int rc = fast::make_map(&m, src, true, (unsigned long long)rows, 128, 64, 64, true)) return rc;
  size_t smem = 1024 + (size_t)ns * tensors * 16384 + 256;
  if (smem > 227 * 1024) return ZGLA_ERR_CONFIG;
  cudaFuncSetAttribute(selftest_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  selftest_stream_kernel<<<ctas, 64, smem, (cudaStream_t)stream>>>(m, (int)rows, tiles_per_cta, ns, tensors,
                                                                    prefetch);
  return zgla_check_launch();
}

// ---------------------------------------------------------------------------
// Diagnostic: TMEM load/store throughput.  nwarps warps each issue `iters` x
// tcgen05.ld.32x32b.x32 (mode 0), ld pairs before one wait (mode 1) or
// tcgen05.st.32x32b.x32 (mode 2); clock64 delta of warp 0 is written to out[0].
namespace zgla {
__global__ void selftest_tmem_kernel(int iters, int mode, long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((32u * (warp & 3)) << 16) + 128u * (warp >> 2);
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < iters; ++i) {
      float v[32];
      tmem_ld32(base + 32 * (i & 3), v);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j];
    }
  } else if (mode == 1) {
    for (int i = 0; i < iters; i += 2) {
      uint32_t a[32], b[32];
      tmem_ld32_nw(base + 32 * (i & 3), a);
      tmem_ld32_nw(base + 32 * ((i + 1) & 3), b);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += __uint_as_float(a[j]) + __uint_as_float(b[j]);
    }
  } else {
    float v[32];
    for (int j = 0; j < 32; ++j) v[j] = (float)j;
    for (int i = 0; i < iters; ++i) tmem_st32(base + 32 * (i & 3), v);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}
}  // namespace zgla

extern "C" int zgla_selftest_tmem(int nwarps, int iters, int mode, long long* out, float* sink, void* stream) {
  using namespace zgla;
  if (nwarps < 1 || nwarps > 16) return ZGLA_ERR_CONFIG;
  selftest_tmem_kernel<<<1, 32 * nwarps, 0, (cudaStream_t)stream>>>(iters, mode, out, sink);
  return zgla_check_launch();
}

// ---- injected latency (diagnostics): one 32-thread CTA that spins on %globaltimer for `ns` nanoseconds.
// scripts/overlap_probe.py puts it where a peer's All-Scan chain would sit on one GPU, to measure how much
// of a chain's latency the head-group overlap schedule (ZecoRank overlap_groups) hides.
__global__ void __launch_bounds__(32) selftest_spin_kernel(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  } while ((long long)(t - t0) < ns);
}
extern "C" int zgla_selftest_spin(long long ns, void* stream) {
  selftest_spin_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ns);
  return zgla_check_launch();
}

// ---------------------------------------------------------------------------
// Diagnostic: tcgen05 MMA issue rate.  Every CTA (one per SM) issues `iters` groups of 8 SS MMAs of shape
// M x N x 16 (bf16, operands in SW128 shared memory, contents irrelevant) into one TMEM accumulator,
// commits each group to an mbarrier and waits for the last; out[blockIdx.x] = SM cycles per MMA.
namespace zgla {
template <bool TS>
__global__ void __launch_bounds__(128) selftest_mma_rate_kernel(int M, int N, int a_mn, int b_mn, int iters,
                                                                long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x;
  for (int i = tid; i < 131072 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) {
    tmem_alloc(&tmem_base_sh, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(M, N, a_mn != 0, b_mn != 0);
    const uint32_t sa = smem_u32(smem), sb = sa + 65536;  // MN-major panels 16 KiB apart
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      ad[kk] = a_mn ? sdesc(sa + kk * 2048, 16384, 1024) : sdesc(sa + kk * 32, 16, 1024);
      bd[kk] = b_mn ? sdesc(sb + kk * 2048, 16384, 1024) : sdesc(sb + kk * 32, 16, 1024);
    }
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if constexpr (TS)
          mma_bf16_ts(tbase, tbase + 256 + (kk & 3) * 8, bd[kk & 3], idesc, 1u);
        else
          mma_bf16_ss(tbase, ad[kk & 3], bd[kk & 3], idesc, 1u);
      }
      mma_commit(&bar);
    }
    mbar_wait(&bar, (iters - 1) & 1);
    const long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0) * 1000 / (8ll * iters);  // milli-cycles per MMA
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tbase, 512);
}
}  // namespace zgla

extern "C" int zgla_selftest_mma_rate(int M, int N, int a_mn, int b_mn, int iters, int ctas, long long* out,
                                      void* stream) {
  using namespace zgla;
  if (!((M == 64 || M == 128) && N % 16 == 0 && N >= 16 && N <= 256 && iters > 0 && ctas > 0)) return ZGLA_ERR_DIMS;
  const size_t smem = 1024 + 131072;
  auto kern = a_mn == 2 ? selftest_mma_rate_kernel<true> : selftest_mma_rate_kernel<false>;  // 2: A from TMEM
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<ctas, 128, smem, (cudaStream_t)stream>>>(M, N, a_mn == 2 ? 0 : a_mn, b_mn, iters, out);
  return zgla_check_launch();
}
