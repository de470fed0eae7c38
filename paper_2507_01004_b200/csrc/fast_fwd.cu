// Fused tcgen05 ZeCO GLA: segment-state kernels, segment scans and the forward
// output kernel (bf16 q/k/v/o, fp32 g and states, D = 128, 64-token tiles).
//
//   seg_state_kernel<FWD>  (K1)  dS_s  = sum_t e^{G_end - G_t} k_t^T v_t      reverse tile walk
//   seg_state_kernel<BWD>  (K4)  dD_s  = sum_t e^{G_t - G_start} q_t^T dO_t   forward tile walk
//       one TMEM accumulator per CTA; every coefficient is <= 1, so the whole
//       segment is ONE uninterrupted tcgen05 accumulation (no TMEM round trips)
//   seg_scan_kernel<0> / <1> (K2/K5): elementwise scans over segments
//   fwd_out_kernel (K3): per 64-token tile
//       A   = Qh Kh^T               (M=64,  N=64,  K=128)  scores, masked in registers
//       O   = Qh (e^{r} S)         (M=64,  N=128, K=128)  inter-chunk term
//       O  += mask(A) V             (M=64,  N=128, K=64)   intra-chunk term
//       KV  = Kh^T V                (M=128, N=128, K=64)   state contribution
//       S   = e^{gam} S + e^{gam-r} KV   (fp32 state resident in TMEM, updated by 8 warps)
//   with Qh = Q e^{logb - r}, Kh = K e^{r - logb}, r = logb at the middle row of
//   the tile (in-chunk reference point: |exponent| <= |gamma|/2).
//   The incoming state of every segment already contains the cross-rank
//   correction e^{G_t} S_prev (fused, no extra pass over HBM).
#include <mutex>
#include <unordered_map>
#include <vector>
#include "fast_common.cuh"

#ifndef ZGLA_ABL_NOSCAN
#define ZGLA_ABL_NOSCAN 0  // timing ablation only (wrong results): skip the segment scans K2 / K5
#endif
namespace zgla {
namespace fast {

// ============================================================== K1 / K4
constexpr int KS_NS = 3;
constexpr int KS_STAGE = 2 * TILE_BF16 + TILE_F32;  // a, b, g = 64 KiB
constexpr int KS_THREADS = 320;                     // 8 prep warps (2 groups), TMA warp, MMA warp
constexpr int KS_OFF_BAR = KS_NS * KS_STAGE;
constexpr size_t KS_SMEM = 1024 + KS_NS * KS_STAGE + 4096;

// PAIR (d = 64): the CTA's 128 channels are two heads, 2*hh (channels 0-63) and 2*hh+1 (64-127); the state
// accumulator keeps its cross-head blocks, which no consumer reads (see fwd_out_kernel)
template <int DIR, bool DENSE, bool PAIR = false>  // 0: forward local state (a=k, b=v, reverse walk); 1: backward (a=q, b=dO)
__global__ void __launch_bounds__(KS_THREADS, 1)
    seg_state_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                     const __grid_constant__ CUtensorMap tm_g, long long L, int in3d, int nseg, int ntiles,
                     float* __restrict__ out_state, float* __restrict__ out_gam, int* __restrict__ flags,
                     int* dom_sink) {
  extern __shared__ uint8_t smem_raw[];
  // align by offsetting the __shared__ array itself so the compiler keeps the shared address space (LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + KS_OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + KS_NS;
  uint64_t* prep = bars + 2 * KS_NS;
  uint64_t* gready = bars + 3 * KS_NS;  // [4] tile gammas published by one prep group for the other
  uint64_t* done = gready + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* xg = reinterpret_cast<float*>(smem + KS_OFF_BAR + 256);  // [4][D]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hh = blockIdx.x / nseg, s = blockIdx.x % nseg;
  int t0, t1;
  seg_range(s, nseg, ntiles, t0, t1);
  const int nt = t1 - t0;
  int bad = 0;  // DIR 0: a tile of this segment left the exponent domain

  if (tid == 0) {
    for (int i = 0; i < KS_NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&prep[i], 128);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&gready[i], 128);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 9) {
    tmem_alloc(tmem_slot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_a);
      tma_prefetch_desc(&tm_b);
      tma_prefetch_desc(&tm_g);
      // L2 reuse by the consumer kernel: it walks the segment in the opposite direction, so the tiles read
      // LAST here are read FIRST there.  The first part of this walk is loaded evict-first so that the
      // tail of the walk is what stays resident.
      const uint64_t pol_first = l2_policy_evict_first(), pol_keep = l2_policy_evict_normal();
      const int keep_from = nt - (nt * ZGLA_L2_KEEP_PCT) / 100;
      for (int j = 0; j < nt; ++j) {
        const int st = j % KS_NS, ph = (j / KS_NS) & 1;
        const int tile = DIR == 0 ? t1 - 1 - j : t0 + j;
        const uint64_t pol = j >= keep_from ? pol_keep : pol_first;
        uint8_t* sa = smem + st * KS_STAGE;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], KS_STAGE);
        const int r = tile * T;
        if constexpr (PAIR) {  // one 64-channel panel per head; gates as two [64][64] fp32 blocks
          tile_load<false>(sa, &tm_a, &full[st], 0, r, 2 * hh, L, 1, pol);
          tile_load<false>(sa + PANEL, &tm_a, &full[st], 0, r, 2 * hh + 1, L, 1, pol);
          tile_load<false>(sa + TILE_BF16, &tm_b, &full[st], 0, r, 2 * hh, L, 1, pol);
          tile_load<false>(sa + TILE_BF16 + PANEL, &tm_b, &full[st], 0, r, 2 * hh + 1, L, 1, pol);
          tile_load<false>(sa + 2 * TILE_BF16, &tm_g, &full[st], 0, r, 2 * hh, L, 1, pol);
          tile_load<false>(sa + 2 * TILE_BF16 + TILE_F32 / 2, &tm_g, &full[st], 0, r, 2 * hh + 1, L, 1, pol);
        } else {
          tile_load<DENSE>(sa, &tm_a, &full[st], 0, r, hh, L, in3d, pol);
          tile_load<DENSE>(sa + PANEL, &tm_a, &full[st], 64, r, hh, L, in3d, pol);
          tile_load<DENSE>(sa + TILE_BF16, &tm_b, &full[st], 0, r, hh, L, in3d, pol);
          tile_load<DENSE>(sa + TILE_BF16 + PANEL, &tm_b, &full[st], 64, r, hh, L, in3d, pol);
          tile_load<DENSE>(sa + 2 * TILE_BF16, &tm_g, &full[st], 0, r, hh, L, in3d, pol);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, 128, true, true);
      for (int i = 0; i < nt; ++i) {
        const int st = i % KS_NS, ph = (i / KS_NS) & 1;
        const uint32_t sa = smem_u32(smem + st * KS_STAGE);
        mbar_wait(&prep[st], ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint64_t ad = sdesc(sa + kk * 2048, PANEL, 1024);
          const uint64_t bd = sdesc(sa + TILE_BF16 + kk * 2048, PANEL, 1024);
          mma_bf16_ss(tbase, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&empty[st]);
      }
      mma_commit(done);
    }
  } else {
    // prep: thread per channel c; two groups of 4 warps take alternate tiles.  The coefficient of
    // tile i needs the sum of the gates of all tiles processed before it (acc_i); each group
    // publishes its tile gamma early so the other group can advance its running sum.
    const int c = tid & 127, grp = tid >> 7;
    const uint32_t coff = (c >> 6) * PANEL + (c & 7) * 2, cchk = (c & 63) >> 3;
    constexpr float LOG2E = 1.4426950408889634f;
    float acc = 0.f;       // sum of gammas of tiles processed before the current one
    float last_tot = 0.f;  // acc + gamma after my last tile
    for (int i = grp; i < nt; i += 2) {
      const int st = i % KS_NS, ph = (i / KS_NS) & 1;
      uint8_t* sa = smem + st * KS_STAGE;
      const float* gs = reinterpret_cast<const float*>(sa + 2 * TILE_BF16);
      mbar_wait(&full[st], ph);
      float lb[64];
      if constexpr (PAIR) {
        const float* gh = gs + (c >> 6) * (T * 64) + (c & 63);
#pragma unroll
        for (int r = 0; r < 64; ++r) lb[r] = gh[r * 64];
      } else {
#pragma unroll
        for (int r = 0; r < 64; ++r) lb[r] = gs[r * D + c];
      }
      if (DIR == 0) {  // the reference's SeqShard check (glasp/gla.py:106-107): every gate finite and < 0
        float mx = lb[0];
#pragma unroll
        for (int r = 1; r < 64; ++r) mx = fmaxf(mx, lb[r]);
        if (!(mx < 0.f)) bad = 1;
      }
#pragma unroll
      for (int r = 1; r < 64; ++r) lb[r] += lb[r - 1];
      const float gam = lb[63];
      if (DIR == 0 && !(gam >= -2.f * DOMAIN_EXP)) bad = 1;  // also catches NaN / -inf
      xg[(i & 3) * D + c] = gam;
      mbar_arrive(&gready[i & 3]);
      if (i >= 1) {  // gamma of tile i-1 (other group)
        mbar_wait(&gready[(i - 1) & 3], ((i - 1) >> 2) & 1);
        acc += xg[((i - 1) & 3) * D + c];
      }
#pragma unroll
      for (int r0 = 0; r0 < 64; r0 += 16) {  // batches: all loads, then all stores (smem may alias)
        __nv_bfloat16 x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = *reinterpret_cast<const __nv_bfloat16*>(sa + coff + sw128(r0 + r, cchk));
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const float e = DIR == 0 ? (acc + gam - lb[r0 + r]) : (acc + lb[r0 + r]);
          x[r] = __float2bfloat16_rn(__bfloat162float(x[r]) * fast_exp2(e * LOG2E));
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) *reinterpret_cast<__nv_bfloat16*>(sa + coff + sw128(r0 + r, cchk)) = x[r];
      }
      fence_proxy_async();
      mbar_arrive(&prep[st]);
      last_tot = acc + gam;
      acc += gam;  // own tile; the other group's next gamma is added at the next iteration
    }
    // epilogue (group 0): accumulator -> global (rows = d_k channels on TMEM lanes)
    if (grp == 0) {
      mbar_wait(done, 0);
      tc_fence_after();
      // workspace states are column-major ([v][c]) so lanes (= channels c) store contiguously
      float* dst = out_state + (long long)(hh * nseg + s) * D * D + c;
#pragma unroll
      for (int chn = 0; chn < D / 32; ++chn) {
        float v[32];
        tmem_ld32(taddr(tbase, warp * 32, chn * 32), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[(chn * 32 + j) * D] = v[j];
      }
    }
    if (nt > 0 && grp == ((nt - 1) & 1)) out_gam[(long long)(hh * nseg + s) * D + c] = last_tot;
  }
  tc_fence_before();
  // one domain flag word per CTA, written every call: no reset pass is needed before the kernel
  bad = __syncthreads_or(bad);
  if (DIR == 0 && flags != nullptr && threadIdx.x == 0) flags[blockIdx.x] = bad;
  // lazy host-visible report (zgla_zeco_watch_domain): host-mapped word, written only when a tile is bad
  if (DIR == 0 && dom_sink != nullptr && threadIdx.x == 0 && bad) *reinterpret_cast<volatile int*>(dom_sink) = 1;
  if (warp == 9) tmem_dealloc(tbase, 128);
}

// ============================================================== K2 / K5
// forward: Sin[s] = sum_{s'<s} e^{gam(s'+1..s-1)} dS[s'];  S_local = inclusive;  cumG / G_tot
// backward: Dend[s] = sum_{s'>s} e^{gam(s+1..s'-1)} dD[s'];  ds_local0 = inclusive of all;  cumGr
// One thread per four state elements walks the segments in order; the loads of a batch of SCAN_B segments
// are issued before the dependent multiply-adds, so the walk costs ~nseg/SCAN_B memory latencies
// instead of nseg.
#ifndef ZGLA_SCAN_B
#define ZGLA_SCAN_B 8
#endif
constexpr int SCAN_B = ZGLA_SCAN_B;

__device__ __forceinline__ float4 f4_fma_exp(float4 g, float4 r, float4 x) {
  return make_float4(expf(g.x) * r.x + x.x, expf(g.y) * r.y + x.y, expf(g.z) * r.z + x.z, expf(g.w) * r.w + x.w);
}
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// DIR 0 (K2): Sin / cumG / S_local / G_tot;  DIR 1 (K5): Dend / cumGr / ds_local0 (segments walked
// from the last).  Four adjacent channels per thread: 16-byte loads and stores.
// pair != 0: d = 64 head pairs; the API outputs take the two diagonal 64 x 64 blocks (heads 2*hh, 2*hh+1)
template <int DIR>
__global__ void seg_scan_kernel(int h, int nseg, int dr, const float* __restrict__ dS, const float* __restrict__ gam,
                                float* __restrict__ Sin, float* __restrict__ cumG, float* __restrict__ s_local,
                                float* __restrict__ g_tot, const float* __restrict__ pf0, const float* __restrict__ pf1,
                                int pair) {
  pdl_wait();
  pdl_trigger();
  const long long idx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (idx >= (long long)h * D * D) return;
  const int hh = (int)(idx / (D * D)), e = (int)(idx % (D * D)), c = e % D, vv = e / D;
  const long long base = (long long)hh * nseg * D * D + e;
  const float* gm = gam + (long long)hh * nseg * D + c;
  float4 run = make_float4(0.f, 0.f, 0.f, 0.f), cm = run;
  for (int b0 = 0; b0 < nseg; b0 += SCAN_B) {
    float4 x[SCAN_B], gg[SCAN_B];
#pragma unroll
    for (int j = 0; j < SCAN_B; ++j) {
      const int s = DIR == 0 ? b0 + j : nseg - 1 - b0 - j;
      const bool ok = b0 + j < nseg;
      x[j] = ok ? __ldcs(reinterpret_cast<const float4*>(dS + base + (long long)s * D * D)) : make_float4(0, 0, 0, 0);
      // K5: warm L2 with the forward segment states the backward output kernel's prologue reads next
      if (DIR == 1 && pf0 != nullptr && ok && (threadIdx.x & 7) == 0) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pf0 + base + (long long)s * D * D));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pf1 + base + (long long)s * D * D));
      }
      gg[j] = ok ? __ldg(reinterpret_cast<const float4*>(gm + s * D)) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < SCAN_B; ++j) {
      if (b0 + j < nseg) {
        const int s = DIR == 0 ? b0 + j : nseg - 1 - b0 - j;
        *reinterpret_cast<float4*>(Sin + base + (long long)s * D * D) = run;
        run = f4_fma_exp(gg[j], run, x[j]);
        if (vv == 0) *reinterpret_cast<float4*>(cumG + (long long)(hh * nseg + s) * D + c) = cm;
        cm = f4_add(cm, gg[j]);
      }
    }
  }
  const float rv[4] = {run.x, run.y, run.z, run.w}, cv[4] = {cm.x, cm.y, cm.z, cm.w};
  if (pair) {  // four channels of one head (c % 4 == 0 never straddles the 64-channel halves)
    const int e = c >> 6, head = 2 * hh + e;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cc = (c & 63) + u;
      if (s_local && (vv >> 6) == e) s_local[((long long)head * 64 + cc) * 64 + (vv & 63)] = rv[u];
      if (DIR == 0 && vv == 0 && g_tot) g_tot[head * 64 + cc] = cv[u];
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (s_local && c + u < dr && vv < dr) s_local[((long long)hh * dr + c + u) * dr + vv] = rv[u];
    if (DIR == 0 && vv == 0 && g_tot && c + u < dr) g_tot[hh * dr + c + u] = cv[u];
  }
}

// ============================================================== K3: forward outputs
constexpr int FO_NS = 3;
constexpr int FO_STAGE = 3 * TILE_BF16;  // q, k, v = 48 KiB (g goes straight to the prep warps' registers)
constexpr int FO_THREADS = 448;  // 4 state warps, 8 prep warps (2 groups, alternate tiles), TMA, MMA
constexpr int FO_OFF_SP = FO_NS * FO_STAGE;         // S' (bf16 [D][D], 2 panels)
constexpr int FO_OFF_AM = FO_OFF_SP + STATE_BF16;   // masked scores (bf16 [64][64], 1 panel)
constexpr int FO_OFF_OST = FO_OFF_AM + T * T * 2;   // O staging for the TMA store (2 x [64][128] bf16, 2 panels each)
constexpr int FO_OFF_VEC = FO_OFF_OST + (ZGLA_O_TMA ? 2 * TILE_BF16 : 0);  // gamma / r per stage
constexpr int FO_OFF_X = FO_OFF_VEC + FO_NS * 2 * D * 4;
constexpr int FO_OFF_BAR = FO_OFF_X + 2 * 64 * 8;
constexpr size_t FO_SMEM = 1024 + FO_OFF_BAR + 256;
// TMEM columns
constexpr uint32_t COL_KV = 0, COL_O = 128, COL_A = 256, COL_S = 320;

// PAIR (d = 64, heads 2*hh and 2*hh+1 on channels 0-63 / 64-127): the scores, the intra term and the
// inter term are per head (K = 64 halves into separate accumulators / output column halves); the fp32
// state keeps its cross-head blocks, which only the (cheap, full-width) state MMA writes and nobody reads.
// The second masked-score operand lives in the off-diagonal (unused) half of the S' buffer.
template <bool DENSE, bool PAIR = false>
__global__ void __launch_bounds__(FO_THREADS, 1)
    fwd_out_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_g,
                   const __grid_constant__ CUtensorMap tm_sp, const __grid_constant__ CUtensorMap tm_o,
                   const float* __restrict__ g, long long gts,
                   long long ghs, long long L, int in3d, int dr, int nseg, int ntiles,
                   const float* __restrict__ Sin,
                   const float* __restrict__ cumG, const float* __restrict__ s_prev,
                   __nv_bfloat16* __restrict__ out, long long ots, long long ohs,
                   __nv_bfloat16* __restrict__ sp_save, unsigned long long* trace, int trace_cta, int early) {
  extern __shared__ uint8_t smem_raw[];
  // align by offsetting the __shared__ array itself so the compiler keeps the shared address space (LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sp_buf = smem + FO_OFF_SP;
  uint8_t* am_buf = smem + FO_OFF_AM;
  uint8_t* ostage = smem + FO_OFF_OST;
  float* vgam = reinterpret_cast<float*>(smem + FO_OFF_VEC);  // [NS][D]
  float* vr = vgam + FO_NS * D;                               // [NS][D]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FO_OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + FO_NS;
  uint64_t* prep = bars + 2 * FO_NS;
  uint64_t* a_full = bars + 3 * FO_NS;
  uint64_t* a_done = a_full + 1;
  uint64_t* kv_full = a_full + 2;
  uint64_t* kv_empty = a_full + 3;
  uint64_t* s_ready = a_full + 4;
  uint64_t* o_full = a_full + 5;
  uint64_t* o_empty = a_full + 6;  // [2]: O is double buffered in the two lane halves
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hh = blockIdx.x / nseg, s = blockIdx.x % nseg;
  int t0, t1;
  seg_range(s, nseg, ntiles, t0, t1);
  const int nt = t1 - t0;
  unsigned long long* tr = (trace != nullptr && (int)blockIdx.x == trace_cta) ? trace : nullptr;
  if (trace != nullptr && threadIdx.x == 0) cta_trace_begin(trace);
  constexpr int DW = PAIR ? 64 : D;  // channels per head in memory
  if constexpr (DENSE) {  // compile-time strides for the dense layout
    gts = DW, ots = DW;
    ghs = L * DW, ohs = L * DW;
    dr = DW;
  }
  uint8_t* am1_buf = sp_buf + T * 128;  // PAIR: rows 64-127 of S' panel 0 (the cross-head block)

  if (tid == 0) {
    for (int i = 0; i < FO_NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&prep[i], 128);
    }
    mbar_init(a_full, 1);
    mbar_init(a_done, 128);
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 128);
    mbar_init(s_ready, 128);
    mbar_init(o_full, 1);
    mbar_init(&o_empty[0], 128);
    mbar_init(&o_empty[1], 128);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // Only the state warps read the preceding scan's outputs (Sin, cumG): with an early launch the
  // loads of q / k / v / g and the per-tile prep run while that kernel is still finishing.
  pdl_trigger();
  if (!early || warp < 4) pdl_wait();  // early: the other warps stream inputs the preceding kernel did not write

  if (warp == 12) {
    // ---------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_g);
      const uint64_t pol = ZGLA_CONSUMER_EVICT_FIRST ? l2_policy_evict_first() : 0;  // 0: no cache hint
      for (int n = 0; n < nt; ++n) {
        const int st = n % FO_NS, ph = (n / FO_NS) & 1;
        uint8_t* sb = smem + st * FO_STAGE;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], FO_STAGE);
        const int r = (t0 + n) * T;
        if constexpr (PAIR) {
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            const CUtensorMap* mx = x == 0 ? &tm_q : x == 1 ? &tm_k : &tm_v;
            tile_load<false>(sb + x * TILE_BF16, mx, &full[st], 0, r, 2 * hh, L, 1, pol);
            tile_load<false>(sb + x * TILE_BF16 + PANEL, mx, &full[st], 0, r, 2 * hh + 1, L, 1, pol);
          }
        } else {
          tile_load<DENSE>(sb, &tm_q, &full[st], 0, r, hh, L, in3d, pol);
          tile_load<DENSE>(sb + PANEL, &tm_q, &full[st], 64, r, hh, L, in3d, pol);
          tile_load<DENSE>(sb + TILE_BF16, &tm_k, &full[st], 0, r, hh, L, in3d, pol);
          tile_load<DENSE>(sb + TILE_BF16 + PANEL, &tm_k, &full[st], 64, r, hh, L, in3d, pol);
          tile_load<DENSE>(sb + 2 * TILE_BF16, &tm_v, &full[st], 0, r, hh, L, in3d, pol);
          tile_load<DENSE>(sb + 2 * TILE_BF16 + PANEL, &tm_v, &full[st], 64, r, hh, L, in3d, pol);
        }
#if ZGLA_G_PREFETCH_FWD
        // warm L2 with the gate tile the prep warps read (pointer loads) a few tiles from now
        if (n + ZGLA_G_PREFETCH_FWD < nt) {
          const int rg = (t0 + n + ZGLA_G_PREFETCH_FWD) * T;
          if constexpr (PAIR) {
            tma_prefetch_3d(&tm_g, 0, rg, 2 * hh);
            tma_prefetch_3d(&tm_g, 0, rg, 2 * hh + 1);
          } else if (in3d) {
            tma_prefetch_3d(&tm_g, 0, rg, hh);
          } else {
            tma_prefetch_2d(&tm_g, 0, (int)(hh * L + rg));
          }
        }
#endif
        ZTRACE(tr, 0, n);
      }
    }
  } else if (warp == 13) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_sc = idesc_bf16(64, 64, false, false);
      constexpr uint32_t id_qs = idesc_bf16(64, 128, false, true);
      constexpr uint32_t id_kv = idesc_bf16(128, 128, true, true);
      constexpr uint32_t id_av = idesc_bf16(64, 128, false, true);
      constexpr uint32_t id_h64 = idesc_bf16(64, 64, false, true);  // PAIR: per-head inter / intra (N = 64)
      const uint32_t spa = smem_u32(sp_buf), ama = smem_u32(am_buf), am1a = smem_u32(am1_buf);
      const bool save_sp = sp_save != nullptr;
      if (save_sp) tma_prefetch_desc(&tm_sp);
      for (int n = 0; n < nt; ++n) {
        const int st = n % FO_NS, ph = (n / FO_NS) & 1;
        const uint32_t qa = smem_u32(smem + st * FO_STAGE);
        const uint32_t ka = qa + TILE_BF16, va = qa + 2 * TILE_BF16;
        mbar_wait(&prep[st], ph);
        mbar_wait(a_done, (n & 1) ^ 1);  // scores of tile n-1 consumed
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * PANEL + (kk & 3) * 32;
          if constexpr (PAIR)  // per-head scores: head 1's in the other lane half of the same columns
            mma_bf16_ss(tbase + ((kk >> 2) ? (16u << 16) : 0u) + COL_A, sdesc(qa + off, 16, 1024),
                        sdesc(ka + off, 16, 1024), id_sc, (kk & 3) > 0);
          else
            mma_bf16_ss(tbase + COL_A, sdesc(qa + off, 16, 1024), sdesc(ka + off, 16, 1024), id_sc, kk > 0);
        }
        mma_commit(a_full);
        ZTRACE(tr, 2, n);
        mbar_wait(s_ready, n & 1);
        if (save_sp) {  // chunk-start state for the backward: async bulk store straight from smem
          if constexpr (PAIR) {  // the two diagonal 64 x 64 blocks, stored per head
            tma_store_2d(&tm_sp, sp_buf, 0, ((2 * hh) * ntiles + t0 + n) * 64);
            tma_store_2d(&tm_sp, sp_buf + SPANEL + T * 128, 0, ((2 * hh + 1) * ntiles + t0 + n) * 64);
          } else if (dr == D) {
            const int rs = (hh * ntiles + t0 + n) * D;
            tma_store_2d(&tm_sp, sp_buf, 0, rs);
            tma_store_2d(&tm_sp, sp_buf + SPANEL, 64, rs);
          } else {  // d = 64: only the 64 x 64 block of real channels is nonzero
            tma_store_2d(&tm_sp, sp_buf, 0, (hh * ntiles + t0 + n) * 64);
          }
          tma_store_commit();
        }
        const uint32_t ob = n & 1;
        const uint32_t t_o = tbase + ((16u * ob) << 16) + COL_O;
        mbar_wait(&o_empty[ob], ((n >> 1) & 1) ^ 1);
        ZTRACE(tr, 11, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * PANEL + (kk & 3) * 32;
          if constexpr (PAIR)  // O[:, 64e:64e+64] = Qh_e S'_ee (K = the head's 64 channels)
            mma_bf16_ss(t_o + 64 * (kk >> 2), sdesc(qa + off, 16, 1024),
                        sdesc(spa + (kk >> 2) * SPANEL + kk * 2048, SPANEL, 1024), id_h64, (kk & 3) > 0);
          else
            mma_bf16_ss(t_o, sdesc(qa + off, 16, 1024), sdesc(spa + kk * 2048, SPANEL, 1024), id_qs, kk > 0);
        }
        mbar_wait(kv_empty, (n & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)
          mma_bf16_ss(tbase + COL_KV, sdesc(ka + kk * 2048, PANEL, 1024), sdesc(va + kk * 2048, PANEL, 1024),
                      id_kv, kk > 0);
        if (save_sp) tma_store_wait_read0();  // S' may be overwritten once kv_full fires
        mma_commit(kv_full);  // also orders the S' read of the inter-chunk MMA before the next S' write
        ZTRACE(tr, 3, n);
        mbar_wait(a_done, n & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          if constexpr (PAIR) {  // O[:, 64e:64e+64] += mask(A_e) V_e
            mma_bf16_ss(t_o, sdesc(ama + kk * 32, 16, 1024), sdesc(va + kk * 2048, PANEL, 1024), id_h64, 1);
            mma_bf16_ss(t_o + 64, sdesc(am1a + kk * 32, 16, 1024), sdesc(va + PANEL + kk * 2048, PANEL, 1024),
                        id_h64, 1);
          } else {
            mma_bf16_ss(t_o, sdesc(ama + kk * 32, 16, 1024), sdesc(va + kk * 2048, PANEL, 1024), id_av, 1);
          }
        }
        mma_commit(o_full);
        mma_commit(&empty[st]);
        ZTRACE(tr, 4, n);
      }
      if (save_sp) tma_store_wait0();
    }
  } else if (warp >= 4) {
    // ---------------- prep (2 groups of 4 warps, alternate tiles): one thread per channel c:
    //                  in-chunk log cumsum over the 64 rows, r = logb[31], gamma = logb[63], Qh / Kh in place
    const int t = tid - 128;
    const int c = t & 127, grp = t >> 7;
    const uint32_t coff = (c >> 6) * PANEL + (c & 7) * 2, cchk = (c & 63) >> 3;
    constexpr float LOG2E = 1.4426950408889634f;
    for (int n = grp; n < nt; n += 2) {
      const int st = n % FO_NS, ph = (n / FO_NS) & 1;
      uint8_t* sb = smem + st * FO_STAGE;
      float lb[64];
      const float* gp = PAIR ? g + (2 * hh + (c >> 6)) * ghs + (long long)(t0 + n) * T * gts + (c & 63)
                             : g + hh * ghs + (long long)(t0 + n) * T * gts + c;
      if constexpr (DENSE) {
#pragma unroll
        for (int r = 0; r < 64; ++r) lb[r] = __ldg(gp + r * DW);  // immediate offsets
      } else if (PAIR || c < dr) {
        const float* pr = gp;  // runtime stride: one pointer bump per row keeps the loads back to back
#pragma unroll
        for (int r = 0; r < 64; ++r, pr += gts) lb[r] = __ldg(pr);
      } else {
#pragma unroll
        for (int r = 0; r < 64; ++r) lb[r] = 0.f;  // zero-filled channel of a d = 64 head
      }
#pragma unroll
      for (int r = 1; r < 64; ++r) lb[r] += lb[r - 1];
      const float rr = lb[31];
      mbar_wait(&full[st], ph);
      if (t == 0 || t == 128) ZTRACE(tr, 12, n);
      vgam[st * D + c] = lb[63];
      vr[st * D + c] = rr;
#pragma unroll
      for (int r0 = 0; r0 < 64; r0 += 8) {  // batches: all loads, then all stores (smem may alias)
        __nv_bfloat16 xq[8], xk[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const uint32_t o = coff + sw128(r0 + r, cchk);
          xq[r] = *reinterpret_cast<const __nv_bfloat16*>(sb + o);
          xk[r] = *reinterpret_cast<const __nv_bfloat16*>(sb + TILE_BF16 + o);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float d = (lb[r0 + r] - rr) * LOG2E;
          xq[r] = __float2bfloat16_rn(__bfloat162float(xq[r]) * fast_exp2(d));
          xk[r] = __float2bfloat16_rn(__bfloat162float(xk[r]) * fast_exp2(-d));
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const uint32_t o = coff + sw128(r0 + r, cchk);
          *reinterpret_cast<__nv_bfloat16*>(sb + o) = xq[r];
          *reinterpret_cast<__nv_bfloat16*>(sb + TILE_BF16 + o) = xk[r];
        }
      }
      fence_proxy_async();
      mbar_arrive(&prep[st]);
      if (t == 0 || t == 128) ZTRACE(tr, 1, n);
    }
  } else {
    // ---------------- state / epilogue warps (4): thread owns row c of the fp32 state S (in TMEM)
    const int qd = warp;
    const int c = 32 * qd + lane;
    const uint32_t s_addr = taddr(tbase, 32 * qd, COL_S);
    // S' = scale * S for 32 columns [32*q, 32*q+32) -> smem B operand ([dk rows][dv], 2 SW128 panels)
    auto write_sp = [&](const float (&v)[32], int q, float scale) {
      if (PAIR && (q >> 1) != (c >> 6)) return;  // PAIR: only the head's diagonal block (the other is A_1)
      uint8_t* dst = sp_buf + (q >> 1) * SPANEL;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        uint4 w;
        w.x = pack_bf16(v[8 * m] * scale, v[8 * m + 1] * scale);
        w.y = pack_bf16(v[8 * m + 2] * scale, v[8 * m + 3] * scale);
        w.z = pack_bf16(v[8 * m + 4] * scale, v[8 * m + 5] * scale);
        w.w = pack_bf16(v[8 * m + 6] * scale, v[8 * m + 7] * scale);
        *reinterpret_cast<uint4*>(dst + sw128(c, 4 * (q & 1) + m)) = w;
      }
    };
    {
      const long long sidx = (long long)(hh * nseg + s) * D * D + c;  // column-major workspace state
      const float cg = s_prev ? expf(cumG[(hh * nseg + s) * D + c]) : 0.f;
      // API states are [head][dr][dr]; PAIR: row c of head 2*hh + c/64, applied to that head's 64 columns
      const float* pv = !s_prev ? nullptr
                        : PAIR ? s_prev + ((long long)(2 * hh + (c >> 6)) * 64 + (c & 63)) * 64 - 64 * (c >> 6)
                        : c < dr ? s_prev + ((long long)hh * dr + c) * dr : nullptr;
      // all loads first (two batches of 64 values, straight into TMEM); the bf16 copy S' needs the first
      // tile's reference point, so it is written from TMEM once the prep warps have published it
#pragma unroll 1
      for (int q2 = 0; q2 < 4; q2 += 2) {
        float v[2][32];
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const int col = 32 * (q2 + hq) + j;
            float4 a = make_float4(Sin[sidx + col * D], Sin[sidx + (col + 1) * D], Sin[sidx + (col + 2) * D],
                                   Sin[sidx + (col + 3) * D]);
            if (pv && (PAIR ? (col >> 6) == (c >> 6) : col < dr)) {
              const float4 b = *reinterpret_cast<const float4*>(pv + col);
              a.x += cg * b.x;
              a.y += cg * b.y;
              a.z += cg * b.z;
              a.w += cg * b.w;
            }
            v[hq][j] = a.x;
            v[hq][j + 1] = a.y;
            v[hq][j + 2] = a.z;
            v[hq][j + 3] = a.w;
          }
        }
        tmem_st32(s_addr + 32 * q2, v[0]);
        tmem_st32(s_addr + 32 * (q2 + 1), v[1]);
      }
      mbar_wait(&prep[0], 0);
      const float e0 = fast_exp(vr[c]);
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        float v[32];
        tmem_ld32(s_addr + 32 * q, v);
        write_sp(v, q, e0);
      }
    }
    fence_proxy_async();
    mbar_arrive(s_ready);

    for (int n = 0; n < nt; ++n) {
      const int st = n % FO_NS, ph = (n / FO_NS) & 1;
      mbar_wait(&prep[st], ph);
      const float gam_c = vgam[st * D + c], r_c = vr[st * D + c];
      // (a) causal mask of the scores -> bf16 K-major A operand (rows i = 16*qd + lane, lanes 0-15)
      mbar_wait(a_full, n & 1);
      tc_fence_after();
      if (tid == 0) ZTRACE(tr, 5, n);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float a[32];
        tmem_ld32(taddr(tbase, 32 * qd, COL_A + 32 * hf), a);
        if (PAIR || lane < 16) {  // PAIR: lanes 16-31 hold head 1's scores
          const int i = 16 * qd + (lane & 15);
          uint8_t* amb = (PAIR && lane >= 16) ? am1_buf : am_buf;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            uint4 w;
            const int j0 = 32 * hf + 8 * m;
            w.x = pack_bf16(j0 + 0 <= i ? a[8 * m + 0] : 0.f, j0 + 1 <= i ? a[8 * m + 1] : 0.f);
            w.y = pack_bf16(j0 + 2 <= i ? a[8 * m + 2] : 0.f, j0 + 3 <= i ? a[8 * m + 3] : 0.f);
            w.z = pack_bf16(j0 + 4 <= i ? a[8 * m + 4] : 0.f, j0 + 5 <= i ? a[8 * m + 5] : 0.f);
            w.w = pack_bf16(j0 + 6 <= i ? a[8 * m + 6] : 0.f, j0 + 7 <= i ? a[8 * m + 7] : 0.f);
            *reinterpret_cast<uint4*>(amb + sw128(i, 4 * hf + m)) = w;
          }
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(a_done);
      if (tid == 0) ZTRACE(tr, 6, n);
      // (b) state update S = e^{gam} S + e^{gam - r} (Kh^T V), and S'_{n+1} = e^{r_{n+1}} S
      const bool more = n + 1 < nt;
      float e1 = 0.f;
      if (more) {
        const int st1 = (n + 1) % FO_NS;
        mbar_wait(&prep[st1], ((n + 1) / FO_NS) & 1);
        e1 = fast_exp(vr[st1 * D + c]);
      }
      mbar_wait(kv_full, n & 1);
      tc_fence_after();
      if (tid == 0) ZTRACE(tr, 7, n);
      {
        const float eg = fast_exp(gam_c), egr = fast_exp(gam_c - r_c);
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          uint32_t kvr[32];
          float sv[32];
          tmem_ld32_nw(taddr(tbase, 32 * qd, COL_KV + 32 * q), kvr);
          tmem_ld32_nw(s_addr + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(sv));
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) sv[j] = eg * sv[j] + egr * __uint_as_float(kvr[j]);
          tmem_st32(s_addr + 32 * q, sv);
          if (more) write_sp(sv, q, e1);
        }
      }
      tc_fence_before();
      mbar_arrive(kv_empty);
      if (more) {
        fence_proxy_async();
        mbar_arrive(s_ready);
      }
      if (tid == 0) ZTRACE(tr, 8, n);
      // (c) epilogue: O tile (lane half n&1) -> global bf16
      mbar_wait(o_full, n & 1);
      tc_fence_after();
      if (tid == 0) ZTRACE(tr, 9, n);
      const int ob = n & 1;
      if constexpr (DENSE && ZGLA_O_TMA) {
        // rows -> swizzled staging tile (16-byte shared stores), then one bulk tensor store per 64 channels
        uint8_t* os = ostage + (n & 1) * TILE_BF16;
        if (tid == 0) tma_store_wait_read1();  // the store of tile n-2 has read this buffer
        named_bar(3, 128);
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          if (!PAIR && 32 * q >= dr) break;
          float o[32];
          tmem_ld32(taddr(tbase, 32 * qd, COL_O + 32 * q), o);
          if ((lane >> 4) == ob) {
            const int i = 16 * qd + (lane & 15);
            uint8_t* pan = os + (q >> 1) * PANEL;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              uint4 w;
              w.x = pack_bf16(o[8 * m + 0], o[8 * m + 1]);
              w.y = pack_bf16(o[8 * m + 2], o[8 * m + 3]);
              w.z = pack_bf16(o[8 * m + 4], o[8 * m + 5]);
              w.w = pack_bf16(o[8 * m + 6], o[8 * m + 7]);
              *reinterpret_cast<uint4*>(pan + sw128(i, 4 * (q & 1) + m)) = w;
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&o_empty[ob]);
        fence_proxy_async();
        named_bar(3, 128);
        if (tid == 0) {
          if constexpr (PAIR) {  // staging panel e -> head 2*hh + e ([h * L rows][64] map)
            tma_store_2d(&tm_o, os, 0, (int)(2 * hh * L + (long long)(t0 + n) * T));
            tma_store_2d(&tm_o, os + PANEL, 0, (int)((2 * hh + 1) * L + (long long)(t0 + n) * T));
          } else {
            const int row = (int)(hh * L + (long long)(t0 + n) * T);
            tma_store_2d(&tm_o, os, 0, row);
            if (dr == D) tma_store_2d(&tm_o, os + PANEL, 64, row);
          }
          tma_store_commit();
        }
      } else {  // strided / d = 64 outputs: 16-byte row pieces straight from the lane half that holds them
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          float o[32];
          tmem_ld32(taddr(tbase, 32 * qd, COL_O + 32 * q), o);
          if ((lane >> 4) == ob && (PAIR || 32 * q < dr)) {
            const int i = 16 * qd + (lane & 15);
            uint4* dst = reinterpret_cast<uint4*>(
                PAIR ? out + (2 * hh + (q >> 1)) * ohs + ((long long)(t0 + n) * T + i) * ots + 32 * (q & 1)
                     : out + hh * ohs + ((long long)(t0 + n) * T + i) * ots + 32 * q);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              uint4 w;
              w.x = pack_bf16(o[8 * m + 0], o[8 * m + 1]);
              w.y = pack_bf16(o[8 * m + 2], o[8 * m + 3]);
              w.z = pack_bf16(o[8 * m + 4], o[8 * m + 5]);
              w.w = pack_bf16(o[8 * m + 6], o[8 * m + 7]);
              dst[m] = w;
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&o_empty[ob]);
      }
      if (tid == 0) ZTRACE(tr, 10, n);
    }
    if (DENSE && ZGLA_O_TMA && tid == 0) tma_store_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (trace != nullptr && threadIdx.x == 0) cta_trace_end(trace);
  if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace fast

// ============================================================== host entry points
using namespace fast;

bool fast_supported(const zgla_shape* s) {
  return s && s->dtype == ZGLA_BF16 && s->key_dim == s->value_dim && (s->key_dim == D || s->key_dim == 64) &&
         s->seq_len % T == 0 &&
         s->heads * s->seq_len < (1ll << 31) && encode_fn() != nullptr;
}

long long fast_ws_bytes(const zgla_shape* s, int num_sms) { return ws_bytes(make_plan(s, num_sms)); }
int* domain_sink_of(const void* ws);

int launch_seg_state(int dir, const Plan& pl, const TRef& a, const TRef& b, const TRef& g, float* out_state,
                     float* out_gam, int* flags, cudaStream_t st, int* dom_sink = nullptr) {
  CUtensorMap ma, mb, mg;
  if (pl.pair) {
    const int heads = 2 * pl.h;
    if (int rc = map_act_pair(&ma, a, pl.L, heads)) return rc;
    if (int rc = map_act_pair(&mb, b, pl.L, heads)) return rc;
    if (int rc = map_gate_pair(&mg, g, pl.L, heads)) return rc;
    auto kern = dir == 0 ? seg_state_kernel<0, false, true> : seg_state_kernel<1, false, true>;
    set_smem_once((const void*)kern, (int)KS_SMEM);
    if (cudaError_t e = launch_k(kern, pl.h * pl.nseg, KS_THREADS, KS_SMEM, st, ma, mb, mg, pl.L, 1, pl.nseg,
                                  pl.ntiles, out_state, out_gam, flags, dom_sink))
      return cuda_fail(e, "seg_state_kernel (pairs)");
    return zgla_check_launch();
  }
  const bool dn = is_dense(a, pl.L) && is_dense(b, pl.L) && is_dense(g, pl.L);  // all TMA-read
  if (int rc = map_act(&ma, a, pl.L, pl.h, dn)) return rc;
  if (int rc = map_act(&mb, b, pl.L, pl.h, dn)) return rc;
  if (int rc = map_gate(&mg, g, pl.L, pl.h, dn)) return rc;
  auto kern = dir == 0 ? seg_state_kernel<0, true> : seg_state_kernel<1, true>;
  set_smem_once((const void*)kern, (int)KS_SMEM);
  if (cudaError_t e = launch_k(kern, pl.h * pl.nseg, KS_THREADS, KS_SMEM, st, ma, mb, mg, pl.L, dn ? 0 : 1, pl.nseg,
                                pl.ntiles, out_state, out_gam, flags, dom_sink))
    return cuda_fail(e, "seg_state_kernel");
  return zgla_check_launch();
}

int fast_fwd_local(const zgla_shape* s, int num_sms, const TRef& k, const TRef& v, const TRef& g, void* ws,
                   void* s_local, void* g_tot, cudaStream_t st) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, ws);
  if (int rc = launch_seg_state(0, pl, k, v, g, w.dS, w.gam, w.flags, st, domain_sink_of(ws))) return rc;
  const long long n = (long long)pl.h * D * D;
  if (ZGLA_ABL_NOSCAN) return zgla_check_launch();  // timing ablation only
  if (cudaError_t e = launch_k(seg_scan_kernel<0>, (unsigned)((n / 4 + 127) / 128), 128, 0, st, pl.h, pl.nseg, k.dr,
                                (const float*)w.dS, (const float*)w.gam, w.Sin, w.cumG, (float*)s_local, (float*)g_tot,
                                (const float*)nullptr, (const float*)nullptr, pl.pair))
    return cuda_fail(e, "seg_scan_kernel<0>");
  return zgla_check_launch();
}

int fast_fwd_output(const zgla_shape* s, int num_sms, const TRef& q, const TRef& k, const TRef& v, const TRef& g,
                    void* ws, const void* s_prev, const TRef& o, cudaStream_t st, bool save_states) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, ws);
  CUtensorMap mq, mk, mv, mg, msp;
  const int early = pdl_enabled() && early_inputs();
  if (pl.pair) {
    const int heads = 2 * pl.h;
    if (int rc = sp_map_pair(&msp, w.Sp, pl)) return rc;
    if (int rc = map_act_pair(&mq, q, pl.L, heads)) return rc;
    if (int rc = map_act_pair(&mk, k, pl.L, heads)) return rc;
    if (int rc = map_act_pair(&mv, v, pl.L, heads)) return rc;
    if (int rc = map_gate_pair(&mg, g, pl.L, heads)) return rc;
    const bool dn = is_dense64(g, pl.L) && is_dense64(o, pl.L) && ZGLA_O_TMA;
    CUtensorMap mo = mq;
    if (dn)
      if (int rc = make_map(&mo, o.p, true, (unsigned long long)heads * pl.L, 64, 64, T, true)) return rc;
    auto kern = dn ? fwd_out_kernel<true, true> : fwd_out_kernel<false, true>;
    set_smem_once((const void*)kern, (int)FO_SMEM);
    if (cudaError_t e = launch_kp(pdl_enabled(), kern, pl.h * pl.nseg, FO_THREADS, FO_SMEM, st, mq, mk, mv, mg, msp,
                                  mo, (const float*)g.p, g.ts, g.hs, pl.L, 1, 64, pl.nseg, pl.ntiles,
                                  (const float*)w.Sin, (const float*)w.cumG, (const float*)s_prev, (__nv_bfloat16*)o.p,
                                  o.ts, o.hs, save_states ? w.Sp : nullptr, g_trace_buf, g_trace_cta, early))
      return cuda_fail(e, "fwd_out_kernel (pairs)");
    return zgla_check_launch();
  }
  // maps: 2-D iff the TMA-read inputs are dense; kernel variant: compile-time strides iff the
  // pointer-addressed tensors (g, o) are dense
  const bool din = is_dense(q, pl.L) && is_dense(k, pl.L) && is_dense(v, pl.L);
  const bool dn = is_dense(g, pl.L) && is_dense(o, pl.L);
  if (int rc = sp_map(&msp, w.Sp, pl, q.dr)) return rc;
  if (int rc = map_act(&mq, q, pl.L, pl.h, din)) return rc;
  if (int rc = map_act(&mk, k, pl.L, pl.h, din)) return rc;
  if (int rc = map_act(&mv, v, pl.L, pl.h, din)) return rc;
  if (int rc = map_gate(&mg, g, pl.L, pl.h, din && is_dense(g, pl.L))) return rc;
  CUtensorMap mo = mq;  // the strided variant stores O through pointers
  if (dn && ZGLA_O_TMA)
    if (int rc = map_act(&mo, o, pl.L, pl.h, true)) return rc;
  auto kern = dn ? fwd_out_kernel<true> : fwd_out_kernel<false>;
  set_smem_once((const void*)kern, (int)FO_SMEM);
  if (cudaError_t e = launch_kp(pdl_enabled(), kern, pl.h * pl.nseg, FO_THREADS, FO_SMEM, st, mq, mk, mv, mg, msp,
                                mo, (const float*)g.p, g.ts, g.hs, pl.L, din ? 0 : 1, q.dr, pl.nseg, pl.ntiles,
                                (const float*)w.Sin, (const float*)w.cumG, (const float*)s_prev, (__nv_bfloat16*)o.p,
                                o.ts, o.hs, save_states ? w.Sp : nullptr,
                                g_trace_buf, g_trace_cta, early))
    return cuda_fail(e, "fwd_out_kernel");
  return zgla_check_launch();
}

int fast_bwd_local(const zgla_shape* s, int num_sms, const TRef& q, const TRef& g, const TRef& d_out, void* ws,
                   void* ds0, cudaStream_t st) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, ws);
  if (int rc = launch_seg_state(1, pl, q, d_out, g, w.dD, w.gam, nullptr, st)) return rc;
  const long long n = (long long)pl.h * D * D;
  if (ZGLA_ABL_NOSCAN) return zgla_check_launch();  // timing ablation only
  if (cudaError_t e = launch_k(seg_scan_kernel<1>, (unsigned)((n / 4 + 127) / 128), 128, 0, st, pl.h, pl.nseg, q.dr,
                                (const float*)w.dD, (const float*)w.gam, w.Dend, w.cumGr, (float*)ds0, (float*)nullptr,
                                (const float*)w.Sin, (const float*)w.dS, pl.pair))
    return cuda_fail(e, "seg_scan_kernel<1>");
  return zgla_check_launch();
}

}  // namespace zgla

namespace zgla {
// ---- lazy domain reports: workspace -> host-mapped flag word (zgla_zeco_watch_domain)
// Words come from slabs of host-mapped memory allocated once and never freed: a cudaHostAlloc /
// cudaFreeHost per shard would cost milliseconds and synchronise the device (cudaFreeHost does) every
// time a short-lived shard (one per layer call) comes and goes.  A released word is reused only after
// kQuarantine later releases, so a segment pass still in flight cannot mark its next owner.
namespace {
std::mutex g_dom_mu;
std::unordered_map<const void*, std::pair<int*, int*>> g_dom;  // ws -> (host, device) pointers
constexpr int kSlab = 4096, kQuarantine = 1024;
std::vector<std::pair<int*, int*>> g_dom_free;                  // never used
std::vector<std::pair<int*, int*>> g_dom_released;              // FIFO of released words
size_t g_dom_released_head = 0;
int take_word(std::pair<int*, int*>* out) {
  if (g_dom_released.size() - g_dom_released_head > (size_t)kQuarantine) {
    *out = g_dom_released[g_dom_released_head++];
    if (g_dom_released_head > 4096) {  // compact the consumed prefix now and then
      g_dom_released.erase(g_dom_released.begin(), g_dom_released.begin() + (long)g_dom_released_head);
      g_dom_released_head = 0;
    }
    return ZGLA_OK;
  }
  if (g_dom_free.empty()) {
    int* h = nullptr;
    int* d = nullptr;
    if (cudaError_t e = cudaHostAlloc(&h, kSlab * sizeof(int), cudaHostAllocMapped)) return cuda_fail(e, "cudaHostAlloc");
    if (cudaError_t e = cudaHostGetDevicePointer(&d, h, 0)) return cuda_fail(e, "cudaHostGetDevicePointer");
    for (int i = kSlab - 1; i >= 0; --i) g_dom_free.emplace_back(h + i, d + i);
  }
  *out = g_dom_free.back();
  g_dom_free.pop_back();
  return ZGLA_OK;
}
}  // namespace
int* domain_sink_of(const void* ws) {
  std::lock_guard<std::mutex> lock(g_dom_mu);
  auto it = g_dom.find(ws);
  return it == g_dom.end() ? nullptr : it->second.second;
}
int watch_domain(const void* ws, int** host_flag) {
  std::lock_guard<std::mutex> lock(g_dom_mu);
  auto it = g_dom.find(ws);
  if (it == g_dom.end()) {
    std::pair<int*, int*> w;
    if (int rc = take_word(&w)) return rc;
    *w.first = 0;
    it = g_dom.emplace(ws, w).first;
  }
  if (host_flag) *host_flag = it->second.first;
  return ZGLA_OK;
}
int unwatch_domain(const void* ws) {
  std::lock_guard<std::mutex> lock(g_dom_mu);
  auto it = g_dom.find(ws);
  if (it != g_dom.end()) {
    g_dom_released.push_back(it->second);
    g_dom.erase(it);
  }
  return ZGLA_OK;
}

int fast_domain_flag(const zgla_shape* s, int num_sms, const void* ws, int* host_flag, cudaStream_t st) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, const_cast<void*>(ws));
  std::vector<int> f((size_t)pl.h * pl.nseg);  // one word per forward segment-pass CTA
  if (cudaError_t e = cudaMemcpyAsync(f.data(), w.flags, f.size() * sizeof(int), cudaMemcpyDeviceToHost, st))
    return cuda_fail(e, "zgla_zeco_domain_check");
  if (cudaError_t e = cudaStreamSynchronize(st)) return cuda_fail(e, "zgla_zeco_domain_check");
  int any = 0;
  for (int x : f) any |= x;
  *host_flag = any;
  return ZGLA_OK;
}
}  // namespace zgla
