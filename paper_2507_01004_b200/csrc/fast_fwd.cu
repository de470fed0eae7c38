// Fused tcgen05 ZeCO GLA: segment-state kernels, segment scans and the forward
// output kernel (bf16 q/k/v/o, fp32 g and states, D = 128, 64-token tiles).
//
//   seg_state_kernel<FWD>  (K1)  dS_s  = sum_t e^{G_end - G_t} k_t^T v_t      reverse tile walk
//   seg_state_kernel<BWD>  (K4)  dD_s  = sum_t e^{G_t - G_start} q_t^T dO_t   forward tile walk
//       one TMEM accumulator per CTA; every coefficient is <= 1, so the whole
//       segment is ONE uninterrupted tcgen05 accumulation (no TMEM round trips)
//   fwd_scan_kernel / bwd_scan_kernel (K2/K5): elementwise scans over segments
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
#include "fast_common.cuh"

namespace zgla {
namespace fast {

// ============================================================== K1 / K4
constexpr int KS_NS = 3;
constexpr int KS_STAGE = 2 * TILE_BF16 + TILE_F32;  // a, b, g = 64 KiB
constexpr int KS_THREADS = 192;                     // 4 prep warps, TMA warp, MMA warp
constexpr size_t KS_SMEM = 1024 + KS_NS * KS_STAGE + 2048;

template <int DIR>  // 0: forward local state (a=k, b=v, reverse walk); 1: backward (a=q, b=dO, forward walk)
__global__ void __launch_bounds__(KS_THREADS, 1)
    seg_state_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                     const __grid_constant__ CUtensorMap tm_g, long long L, int nseg, int ntiles,
                     float* __restrict__ out_state, float* __restrict__ out_gam) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + KS_NS * KS_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + KS_NS;
  uint64_t* prep = bars + 2 * KS_NS;
  uint64_t* done = bars + 3 * KS_NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * KS_NS + 1);
  float2* xa = reinterpret_cast<float2*>(smem + KS_NS * KS_STAGE + 256);
  float2* xb = xa + 64;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hh = blockIdx.x / nseg, s = blockIdx.x % nseg;
  int t0, t1;
  seg_range(s, nseg, ntiles, t0, t1);
  const int nt = t1 - t0;
  const int row0 = (int)(hh * L);

  if (tid == 0) {
    for (int i = 0; i < KS_NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&prep[i], 128);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 5) {
    tmem_alloc(tmem_slot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_a);
      tma_prefetch_desc(&tm_b);
      tma_prefetch_desc(&tm_g);
      for (int i = 0; i < nt; ++i) {
        const int st = i % KS_NS, ph = (i / KS_NS) & 1;
        const int tile = DIR == 0 ? t1 - 1 - i : t0 + i;
        uint8_t* sa = smem + st * KS_STAGE;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], KS_STAGE);
        const int r = row0 + tile * T;
        tma_load_2d(sa, &tm_a, &full[st], 0, r);
        tma_load_2d(sa + PANEL, &tm_a, &full[st], 64, r);
        tma_load_2d(sa + TILE_BF16, &tm_b, &full[st], 0, r);
        tma_load_2d(sa + TILE_BF16 + PANEL, &tm_b, &full[st], 64, r);
        tma_load_2d(sa + 2 * TILE_BF16, &tm_g, &full[st], 0, r);
      }
    }
  } else if (warp == 5) {
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
    // prep warps: 128 threads = 64 channel pairs x 2 row halves
    const int cp = tid & 63, rh = tid >> 6;
    float acc0 = 0.f, acc1 = 0.f;  // running sum of gates of already-processed tiles (suffix / prefix)
    for (int i = 0; i < nt; ++i) {
      const int st = i % KS_NS, ph = (i / KS_NS) & 1;
      uint8_t* sa = smem + st * KS_STAGE;
      const float* gs = reinterpret_cast<const float*>(sa + 2 * TILE_BF16);
      mbar_wait(&full[st], ph);
      float lb0[32], lb1[32];
      float run0 = 0.f, run1 = 0.f;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const float2 gv = *reinterpret_cast<const float2*>(gs + (32 * rh + r) * D + 2 * cp);
        run0 += gv.x;
        run1 += gv.y;
        lb0[r] = run0;
        lb1[r] = run1;
      }
      if (rh == 0) xa[cp] = make_float2(run0, run1);
      named_bar(1, 128);
      float off0 = 0.f, off1 = 0.f;
      if (rh == 1) {
        const float2 o = xa[cp];
        off0 = o.x;
        off1 = o.y;
        xb[cp] = make_float2(o.x + run0, o.y + run1);
      }
      named_bar(1, 128);
      const float2 tot = xb[cp];  // gamma of the tile
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const float l0 = lb0[r] + off0, l1 = lb1[r] + off1;
        float w0, w1;
        if (DIR == 0) {
          w0 = fast_exp(acc0 + tot.x - l0);
          w1 = fast_exp(acc1 + tot.y - l1);
        } else {
          w0 = fast_exp(acc0 + l0);
          w1 = fast_exp(acc1 + l1);
        }
        uint32_t* p = reinterpret_cast<uint32_t*>(sa + pair_off(32 * rh + r, cp, PANEL));
        const float2 a = unpack_bf16(*p);
        *p = pack_bf16(a.x * w0, a.y * w1);
      }
      acc0 += tot.x;
      acc1 += tot.y;
      fence_proxy_async();
      mbar_arrive(&prep[st]);
    }
    // epilogue: accumulator -> global (rows = d_k channels on TMEM lanes)
    mbar_wait(done, 0);
    tc_fence_after();
    const int c = warp * 32 + lane;
    float* dst = out_state + ((long long)(hh * nseg + s) * D + c) * D;
#pragma unroll
    for (int ch = 0; ch < D / 32; ++ch) {
      float v[32];
      tmem_ld32(taddr(tbase, warp * 32, ch * 32), v);
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dst + ch * 32 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
    if (rh == 0) {
      float* gdst = out_gam + (long long)(hh * nseg + s) * D;
      gdst[2 * cp] = acc0;
      gdst[2 * cp + 1] = acc1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tbase, 128);
}

// ============================================================== K2 / K5
// forward: Sin[s] = sum_{s'<s} e^{gam(s'+1..s-1)} dS[s'];  S_local = inclusive;  cumG / G_tot
__global__ void fwd_scan_kernel(int h, int nseg, const float* __restrict__ dS, const float* __restrict__ gam,
                                float* __restrict__ Sin, float* __restrict__ cumG, float* __restrict__ s_local,
                                float* __restrict__ g_tot) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)h * D * D) return;
  const int hh = (int)(idx / (D * D)), e = (int)(idx % (D * D)), c = e / D;
  float run = 0.f;
  for (int s = 0; s < nseg; ++s) {
    const long long o = ((long long)(hh * nseg + s)) * D * D + e;
    Sin[o] = run;
    run = expf(gam[(hh * nseg + s) * D + c]) * run + dS[o];
  }
  if (s_local) s_local[idx] = run;
  if ((e % D) == 0) {
    float cm = 0.f;
    for (int s = 0; s < nseg; ++s) {
      cumG[(hh * nseg + s) * D + c] = cm;
      cm += gam[(hh * nseg + s) * D + c];
    }
    if (g_tot) g_tot[hh * D + c] = cm;
  }
}

// backward: Dend[s] = sum_{s'>s} e^{gam(s+1..s'-1)} dD[s'];  ds_local0 = Dend[-1] inclusive of all; cumGr
__global__ void bwd_scan_kernel(int h, int nseg, const float* __restrict__ dD, const float* __restrict__ gam,
                                float* __restrict__ Dend, float* __restrict__ cumGr, float* __restrict__ ds0) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)h * D * D) return;
  const int hh = (int)(idx / (D * D)), e = (int)(idx % (D * D)), c = e / D;
  float run = 0.f;
  for (int s = nseg - 1; s >= 0; --s) {
    const long long o = ((long long)(hh * nseg + s)) * D * D + e;
    Dend[o] = run;
    run = expf(gam[(hh * nseg + s) * D + c]) * run + dD[o];
  }
  if (ds0) ds0[idx] = run;
  if ((e % D) == 0) {
    float cm = 0.f;
    for (int s = nseg - 1; s >= 0; --s) {
      cumGr[(hh * nseg + s) * D + c] = cm;
      cm += gam[(hh * nseg + s) * D + c];
    }
  }
}

// ============================================================== K3: forward outputs
constexpr int FO_NS = 2;
constexpr int FO_STAGE = 3 * TILE_BF16 + TILE_F32;  // q, k, v, g = 80 KiB
constexpr int FO_THREADS = 448;                     // 8 state warps, 4 prep warps, TMA warp, MMA warp
constexpr int FO_OFF_SP = FO_NS * FO_STAGE;         // S' (bf16 [D][D], 2 panels)
constexpr int FO_OFF_AM = FO_OFF_SP + STATE_BF16;   // masked scores (bf16 [64][64], 1 panel)
constexpr int FO_OFF_VEC = FO_OFF_AM + T * T * 2;   // gamma / r per stage
constexpr int FO_OFF_X = FO_OFF_VEC + FO_NS * 2 * D * 4;
constexpr int FO_OFF_BAR = FO_OFF_X + 2 * 64 * 8;
constexpr size_t FO_SMEM = 1024 + FO_OFF_BAR + 256;
// TMEM columns
constexpr uint32_t COL_KV = 0, COL_O = 128, COL_A = 256, COL_S = 320;

__global__ void __launch_bounds__(FO_THREADS, 1)
    fwd_out_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_g, long long L,
                   int nseg, int ntiles, const float* __restrict__ Sin, const float* __restrict__ cumG,
                   const float* __restrict__ s_prev, __nv_bfloat16* __restrict__ out,
                   __nv_bfloat16* __restrict__ sp_save) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sp_buf = smem + FO_OFF_SP;
  uint8_t* am_buf = smem + FO_OFF_AM;
  float* vgam = reinterpret_cast<float*>(smem + FO_OFF_VEC);  // [NS][D]
  float* vr = vgam + FO_NS * D;                               // [NS][D]
  float2* xa = reinterpret_cast<float2*>(smem + FO_OFF_X);
  float2* xb = xa + 64;
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
  uint64_t* o_empty = a_full + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 7);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hh = blockIdx.x / nseg, s = blockIdx.x % nseg;
  int t0, t1;
  seg_range(s, nseg, ntiles, t0, t1);
  const int nt = t1 - t0;
  const int row0 = (int)(hh * L);

  if (tid == 0) {
    for (int i = 0; i < FO_NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&prep[i], 128);
    }
    mbar_init(a_full, 1);
    mbar_init(a_done, 256);
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 256);
    mbar_init(s_ready, 256);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 256);
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

  if (warp == 12) {
    // ---------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_g);
      for (int n = 0; n < nt; ++n) {
        const int st = n % FO_NS, ph = (n / FO_NS) & 1;
        uint8_t* sb = smem + st * FO_STAGE;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], FO_STAGE);
        const int r = row0 + (t0 + n) * T;
        tma_load_2d(sb, &tm_q, &full[st], 0, r);
        tma_load_2d(sb + PANEL, &tm_q, &full[st], 64, r);
        tma_load_2d(sb + TILE_BF16, &tm_k, &full[st], 0, r);
        tma_load_2d(sb + TILE_BF16 + PANEL, &tm_k, &full[st], 64, r);
        tma_load_2d(sb + 2 * TILE_BF16, &tm_v, &full[st], 0, r);
        tma_load_2d(sb + 2 * TILE_BF16 + PANEL, &tm_v, &full[st], 64, r);
        tma_load_2d(sb + 3 * TILE_BF16, &tm_g, &full[st], 0, r);
      }
    }
  } else if (warp == 13) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_sc = idesc_bf16(64, 64, false, false);
      constexpr uint32_t id_qs = idesc_bf16(64, 128, false, true);
      constexpr uint32_t id_kv = idesc_bf16(128, 128, true, true);
      constexpr uint32_t id_av = idesc_bf16(64, 128, false, true);
      const uint32_t spa = smem_u32(sp_buf), ama = smem_u32(am_buf);
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
          mma_bf16_ss(tbase + COL_A, sdesc(qa + off, 16, 1024), sdesc(ka + off, 16, 1024), id_sc, kk > 0);
        }
        mma_commit(a_full);
        mbar_wait(s_ready, n & 1);
        mbar_wait(o_empty, (n & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * PANEL + (kk & 3) * 32;
          mma_bf16_ss(tbase + COL_O, sdesc(qa + off, 16, 1024), sdesc(spa + kk * 2048, SPANEL, 1024), id_qs,
                      kk > 0);
        }
        mbar_wait(kv_empty, (n & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)
          mma_bf16_ss(tbase + COL_KV, sdesc(ka + kk * 2048, PANEL, 1024), sdesc(va + kk * 2048, PANEL, 1024),
                      id_kv, kk > 0);
        mma_commit(kv_full);  // also orders the S' read of the inter-chunk MMA before the next S' write
        mbar_wait(a_done, n & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)
          mma_bf16_ss(tbase + COL_O, sdesc(ama + kk * 32, 16, 1024), sdesc(va + kk * 2048, PANEL, 1024), id_av, 1);
        mma_commit(o_full);
        mma_commit(&empty[st]);
      }
    }
  } else if (warp >= 8) {
    // ---------------- prep: in-chunk log cumsum, reference point, Qh / Kh in place
    const int t = tid - 256;
    const int cp = t & 63, rh = t >> 6;
    for (int n = 0; n < nt; ++n) {
      const int st = n % FO_NS, ph = (n / FO_NS) & 1;
      uint8_t* sb = smem + st * FO_STAGE;
      const float* gs = reinterpret_cast<const float*>(sb + 3 * TILE_BF16);
      mbar_wait(&full[st], ph);
      float lb0[32], lb1[32];
      float run0 = 0.f, run1 = 0.f;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const float2 gv = *reinterpret_cast<const float2*>(gs + (32 * rh + r) * D + 2 * cp);
        run0 += gv.x;
        run1 += gv.y;
        lb0[r] = run0;
        lb1[r] = run1;
      }
      if (rh == 0) xa[cp] = make_float2(run0, run1);
      named_bar(1, 128);
      const float2 half = xa[cp];  // logb at row 31 = the reference point r
      float off0 = 0.f, off1 = 0.f;
      if (rh == 1) {
        off0 = half.x;
        off1 = half.y;
        xb[cp] = make_float2(half.x + run0, half.y + run1);
      }
      named_bar(1, 128);
      if (rh == 0) {
        const float2 gam = xb[cp];
        vgam[st * D + 2 * cp] = gam.x;
        vgam[st * D + 2 * cp + 1] = gam.y;
        vr[st * D + 2 * cp] = half.x;
        vr[st * D + 2 * cp + 1] = half.y;
      }
      constexpr float LOG2E = 1.4426950408889634f;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const float d0 = (lb0[r] + off0 - half.x) * LOG2E, d1 = (lb1[r] + off1 - half.y) * LOG2E;
        const float e0 = fast_exp2(d0), e1 = fast_exp2(d1);
        const float i0 = fast_exp2(-d0), i1 = fast_exp2(-d1);
        const uint32_t o = pair_off(32 * rh + r, cp, PANEL);
        uint32_t* pq = reinterpret_cast<uint32_t*>(sb + o);
        uint32_t* pk = reinterpret_cast<uint32_t*>(sb + TILE_BF16 + o);
        const float2 qv = unpack_bf16(*pq), kv = unpack_bf16(*pk);
        *pq = pack_bf16(qv.x * e0, qv.y * e1);
        *pk = pack_bf16(kv.x * i0, kv.y * i1);
      }
      fence_proxy_async();
      mbar_arrive(&prep[st]);
    }
  } else {
    // ---------------- state / epilogue warps (8): thread owns S[c][64*ch .. +64] (in TMEM), c = 32*qd + lane
    const int qd = warp & 3, ch = warp >> 2;
    const int c = 32 * qd + lane;
    const uint32_t s_addr = taddr(tbase, 32 * qd, COL_S + 64 * ch);
    // S' = scale * S for 32 columns -> smem B operand (and the backward's copy in global memory)
    auto write_sp = [&](const float (&v)[32], int hf, int tile_idx, float scale) {
      uint8_t* dst = sp_buf + ch * SPANEL;
      __nv_bfloat16* gdst =
          sp_save ? sp_save + ((long long)(hh * ntiles + t0 + tile_idx) * D + c) * D + 64 * ch + 32 * hf : nullptr;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        uint4 w;
        w.x = pack_bf16(v[8 * m] * scale, v[8 * m + 1] * scale);
        w.y = pack_bf16(v[8 * m + 2] * scale, v[8 * m + 3] * scale);
        w.z = pack_bf16(v[8 * m + 4] * scale, v[8 * m + 5] * scale);
        w.w = pack_bf16(v[8 * m + 6] * scale, v[8 * m + 7] * scale);
        *reinterpret_cast<uint4*>(dst + sw128(c, 4 * hf + m)) = w;
        if (gdst) reinterpret_cast<uint4*>(gdst)[m] = w;
      }
    };
    {
      const long long sidx = ((long long)(hh * nseg + s) * D + c) * D + 64 * ch;
      const float cg = s_prev ? expf(cumG[(hh * nseg + s) * D + c]) : 0.f;
      const float* pv = s_prev ? s_prev + ((long long)hh * D + c) * D + 64 * ch : nullptr;
      mbar_wait(&prep[0], 0);
      const float e0 = fast_exp(vr[c]);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 a = *reinterpret_cast<const float4*>(Sin + sidx + 32 * hf + j);
          if (pv) {
            const float4 b = *reinterpret_cast<const float4*>(pv + 32 * hf + j);
            a.x += cg * b.x;
            a.y += cg * b.y;
            a.z += cg * b.z;
            a.w += cg * b.w;
          }
          v[j] = a.x;
          v[j + 1] = a.y;
          v[j + 2] = a.z;
          v[j + 3] = a.w;
        }
        tmem_st32(s_addr + 32 * hf, v);
        write_sp(v, hf, 0, e0);
      }
    }
    fence_proxy_async();
    mbar_arrive(s_ready);

    for (int n = 0; n < nt; ++n) {
      const int st = n % FO_NS, ph = (n / FO_NS) & 1;
      mbar_wait(&prep[st], ph);
      const float gam_c = vgam[st * D + c], r_c = vr[st * D + c];
      // (a) causal mask of the scores -> bf16 K-major A operand
      mbar_wait(a_full, n & 1);
      tc_fence_after();
      {
        float a[32];
        tmem_ld32(taddr(tbase, 32 * qd, COL_A + 32 * ch), a);
        if (lane < 16) {
          const int i = 16 * qd + lane;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            uint4 w;
            const int j0 = 32 * ch + 8 * m;
            w.x = pack_bf16(j0 + 0 <= i ? a[8 * m + 0] : 0.f, j0 + 1 <= i ? a[8 * m + 1] : 0.f);
            w.y = pack_bf16(j0 + 2 <= i ? a[8 * m + 2] : 0.f, j0 + 3 <= i ? a[8 * m + 3] : 0.f);
            w.z = pack_bf16(j0 + 4 <= i ? a[8 * m + 4] : 0.f, j0 + 5 <= i ? a[8 * m + 5] : 0.f);
            w.w = pack_bf16(j0 + 6 <= i ? a[8 * m + 6] : 0.f, j0 + 7 <= i ? a[8 * m + 7] : 0.f);
            *reinterpret_cast<uint4*>(am_buf + sw128(i, 4 * ch + m)) = w;
          }
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(a_done);
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
      {
        const float eg = fast_exp(gam_c), egr = fast_exp(gam_c - r_c);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float kv[32], sv[32];
          tmem_ld32(taddr(tbase, 32 * qd, COL_KV + 64 * ch + 32 * hf), kv);
          tmem_ld32(s_addr + 32 * hf, sv);
#pragma unroll
          for (int j = 0; j < 32; ++j) sv[j] = eg * sv[j] + egr * kv[j];
          tmem_st32(s_addr + 32 * hf, sv);
          if (more) write_sp(sv, hf, n + 1, e1);
        }
      }
      tc_fence_before();
      mbar_arrive(kv_empty);
      if (more) {
        fence_proxy_async();
        mbar_arrive(s_ready);
      }
      // (c) epilogue: O tile -> global bf16
      mbar_wait(o_full, n & 1);
      tc_fence_after();
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float o[32];
        tmem_ld32(taddr(tbase, 32 * qd, COL_O + 64 * ch + 32 * hf), o);
        if (lane < 16) {
          const int i = 16 * qd + lane;
          uint4* dst = reinterpret_cast<uint4*>(out + ((long long)row0 + (t0 + n) * T + i) * D + 64 * ch + 32 * hf);
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
      mbar_arrive(o_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace fast

// ============================================================== host entry points
using namespace fast;

bool fast_supported(const zgla_shape* s) {
  return s && s->dtype == ZGLA_BF16 && s->key_dim == D && s->value_dim == D && s->seq_len % T == 0 &&
         s->heads * s->seq_len < (1ll << 31) && encode_fn() != nullptr;
}

long long fast_ws_bytes(const zgla_shape* s, int num_sms) { return ws_bytes(make_plan(s, num_sms)); }

static int map_bf16(CUtensorMap* m, const void* p, const Plan& pl) {
  return make_map(m, p, true, (unsigned long long)pl.h * pl.L, D, 64, T, true);
}
static int map_f32(CUtensorMap* m, const void* p, const Plan& pl) {
  return make_map(m, p, false, (unsigned long long)pl.h * pl.L, D, D, T, false);
}

int launch_seg_state(int dir, const Plan& pl, const void* a, const void* b, const void* g, float* out_state,
                     float* out_gam, cudaStream_t st) {
  CUtensorMap ma, mb, mg;
  if (int rc = map_bf16(&ma, a, pl)) return rc;
  if (int rc = map_bf16(&mb, b, pl)) return rc;
  if (int rc = map_f32(&mg, g, pl)) return rc;
  auto kern = dir == 0 ? seg_state_kernel<0> : seg_state_kernel<1>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KS_SMEM);
  kern<<<pl.h * pl.nseg, KS_THREADS, KS_SMEM, st>>>(ma, mb, mg, pl.L, pl.nseg, pl.ntiles, out_state, out_gam);
  return zgla_check_launch();
}

int fast_fwd_local(const zgla_shape* s, int num_sms, const void* k, const void* v, const void* g, void* ws,
                   void* s_local, void* g_tot, cudaStream_t st) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, ws);
  if (int rc = launch_seg_state(0, pl, k, v, g, w.dS, w.gam, st)) return rc;
  const long long n = (long long)pl.h * D * D;
  fwd_scan_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pl.h, pl.nseg, w.dS, w.gam, w.Sin, w.cumG,
                                                              (float*)s_local, (float*)g_tot);
  return zgla_check_launch();
}

int fast_fwd_output(const zgla_shape* s, int num_sms, const void* q, const void* k, const void* v, const void* g,
                    void* ws, const void* s_prev, void* o, cudaStream_t st) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, ws);
  CUtensorMap mq, mk, mv, mg;
  if (int rc = map_bf16(&mq, q, pl)) return rc;
  if (int rc = map_bf16(&mk, k, pl)) return rc;
  if (int rc = map_bf16(&mv, v, pl)) return rc;
  if (int rc = map_f32(&mg, g, pl)) return rc;
  cudaFuncSetAttribute(fwd_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FO_SMEM);
  fwd_out_kernel<<<pl.h * pl.nseg, FO_THREADS, FO_SMEM, st>>>(mq, mk, mv, mg, pl.L, pl.nseg, pl.ntiles, w.Sin,
                                                              w.cumG, (const float*)s_prev, (__nv_bfloat16*)o,
                                                              w.Sp);
  return zgla_check_launch();
}

int fast_bwd_local(const zgla_shape* s, int num_sms, const void* q, const void* g, const void* d_out, void* ws,
                   void* ds0, cudaStream_t st) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, ws);
  if (int rc = launch_seg_state(1, pl, q, d_out, g, w.dD, w.gam, st)) return rc;
  const long long n = (long long)pl.h * D * D;
  bwd_scan_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pl.h, pl.nseg, w.dD, w.gam, w.Dend, w.cumGr,
                                                              (float*)ds0);
  return zgla_check_launch();
}

}  // namespace zgla
