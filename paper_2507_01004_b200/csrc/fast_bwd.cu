// Fused tcgen05 ZeCO GLA backward (reference glasp/gla.py:359-444, paper Alg. 3),
// bf16 q/k/v/dO/dq/dk/dv, fp32 g/dg/states, D = 128, 64-token tiles.
//
// One CTA per (head, segment) walks its tiles RIGHT TO LEFT carrying the fp32
// state cotangent D in TMEM, seeded with the lifted segment-end cotangent
// D_end = Dend_loc + e^{G_L - G_end} ds_next  (fused bwd correction).  D is kept
// in the per-tile frame Dt_n = e^{-r_n} D_n, so the recurrence
//   Dt_n = e^{gam_n - r_n + r_{n+1}} Dt_{n+1} + Qh^T dO
// is one per-row rescale (which also yields D' for the MMAs) followed by a
// tcgen05 accumulation straight into TMEM (all factors <= 1).
// The forward chunk-start states come from the forward kernel (saved as
// S'_n = e^{r_n} S_n in bf16), so no forward recomputation walk is needed.
// Per tile (Qh = Q e^{logb-r}, Kh = K e^{r-logb}, D' = e^{gam-r} D_{n+1}):
//   A    = Qh Kh^T      dP = dO V^T                 (M=64, N=64)   masked in registers
//   Dt  += Qh^T dO                                   (M=128,N=128)  accumulated in place
//   dq^T = Kh^T dPm^T + S' dO^T                      (M=128,N=64)   dq = E (.) dq_raw
//   dk^T = Qh^T dPm   + D' V^T                       (M=128,N=64)   dk = dk_raw / E
//   dv^T = dO^T Am    + D'^T Kh^T                    (M=128,N=64)
// All gradient accumulators are TRANSPOSED (channels on TMEM lanes), so the
// epilogue thread of channel c owns a token column and computes
//   da_t = Qh (.) dq_raw - Kh (.) dk_raw  (= q.dq - k.dk)
//   dg_t = sum_{t' >= t in tile} da_t' + rho_{n+1},   rho_n = rho_{n+1} + sum_tile da
// sequentially, where rho at the segment end is rowsum(S_end (.) D_end): the
// suffix sum of da beyond a boundary equals that boundary rowsum, so dg needs
// no cross-segment pass (it includes the reference's tail term,
// glasp/gla.py:440-443, at the shard end).
#include "fast_common.cuh"

namespace zgla {
namespace fast {

#ifndef ZGLA_SP_WAIT
#define ZGLA_SP_WAIT 0
#endif
#ifndef ZGLA_RHO_RESEED
#define ZGLA_RHO_RESEED 8  // tiles between dg re-seeds from rowsum(S' (.) Dt) (0: never)
#endif
#ifndef ZGLA_ABL_PART2
#define ZGLA_ABL_PART2 0  // timing ablation only (wrong results): skip the D'-dependent dk / dv MMAs
#endif
constexpr int BO_NS = 2;
constexpr int BO_STAGE = 4 * TILE_BF16;  // q, k, v, dO
constexpr int BO_THREADS = 448;          // 8 state warps, 4 prep warps, TMA warp, MMA warp
constexpr int BO_OFF_SP = BO_NS * BO_STAGE;
constexpr int BO_OFF_DP = BO_OFF_SP + STATE_BF16;
constexpr int BO_OFF_AM = BO_OFF_DP + STATE_BF16;
constexpr int BO_OFF_DPM = BO_OFF_AM + T * T * 2;
constexpr int BO_OFF_VEC = BO_OFF_DPM + T * T * 2;
constexpr int BO_OFF_X = BO_OFF_VEC + BO_NS * 2 * D * 4;
constexpr int BO_OFF_BAR = BO_OFF_X + 4096;
constexpr size_t BO_SMEM = 1024 + BO_OFF_BAR + 256;
// TMEM columns.  Scores (lanes 0-15 of each quarter) and dP (lanes 16-31) share one M=64 column block;
// LB holds d = logb - r per (channel lane, token column), double buffered, written by the prep warps.
constexpr uint32_t BC_DQ = 0, BC_DK = 64, BC_DV = 128, BC_QDO = 192, BC_SC = 320, BC_LB = 384;
// PAIR (d = 64, heads 2*hh / 2*hh+1 on channels 0-63 / 64-127): every accumulator whose rows are channels
// is split per head into two M = 64 MMAs that fill the two lane halves of each TMEM lane quarter, so TMEM
// lane l = 32*qd + 16*e + x holds channel c = 64*e + 16*qd + x of head e (pair_channel).  Dt shrinks to
// 64 columns (its cross-head blocks are never formed), which frees BC_SC2 for the second head's scores.
// The second head's masked operands live in the unused off-diagonal blocks of the S' buffer.
constexpr uint32_t BC_SC2 = 256;
__device__ __forceinline__ int pair_channel(int lane_id) {  // TMEM lane (0..127) -> channel of the pair
  return 64 * ((lane_id & 31) >> 4) + 16 * (lane_id >> 5) + (lane_id & 15);
}

// dg re-seeding (section 4 of DESIGN.md): on tile m with (m + 1) % ZGLA_RHO_RESEED == 0 the seed of the next
// tile is rho_n = rowsum(S'_n (.) Dt_n); k-th such tile -> parity k & 1 of the sp_read barrier
__device__ __forceinline__ bool reseed_tile(int m, int nt) {
  return ZGLA_RHO_RESEED > 0 && m + 1 < nt && (m + 1) % (ZGLA_RHO_RESEED > 0 ? ZGLA_RHO_RESEED : 1) == 0;
}

template <bool DENSE, bool PAIR = false>
__global__ void __launch_bounds__(BO_THREADS, 1)
    bwd_out_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                   const __grid_constant__ CUtensorMap tm_sp, const __grid_constant__ CUtensorMap tm_g,
                   const __grid_constant__ CUtensorMap tm_dg, const float* __restrict__ g, long long gts, long long ghs, long long L, int in3d, int dr,
                   int nseg,
                   int ntiles, const float* __restrict__ Sin, const float* __restrict__ cumG,
                   const float* __restrict__ dS, const float* __restrict__ gamseg, const float* __restrict__ s_prev,
                   const float* __restrict__ Dend, const float* __restrict__ cumGr,
                   const float* __restrict__ ds_next, __nv_bfloat16* __restrict__ dq, __nv_bfloat16* __restrict__ dk,
                   __nv_bfloat16* __restrict__ dv, float* __restrict__ dg, Strides4 gs, unsigned long long* trace,
                   int trace_cta, int early) {
  extern __shared__ uint8_t smem_raw[];
  // align by offsetting the __shared__ array itself so the compiler keeps the shared address space (LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sp_buf = smem + BO_OFF_SP;
  uint8_t* dp_buf = smem + BO_OFF_DP;
  uint8_t* am_buf = smem + BO_OFF_AM;
  uint8_t* dpm_buf = smem + BO_OFF_DPM;
  float* vgam = reinterpret_cast<float*>(smem + BO_OFF_VEC);
  float* vr = vgam + BO_NS * D;
  float* xrho = reinterpret_cast<float*>(smem + BO_OFF_X + 1024);  // [2][D] row-sum partials
  float* xcarry = xrho + 3 * D;                                    // [2][D] per-half sums of da
  float* xr = xcarry + 2 * D;                                      // [D] rho at the current tile end
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BO_OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + BO_NS;
  uint64_t* prep = bars + 2 * BO_NS;
  uint64_t* sc_full = bars + 3 * BO_NS;
  uint64_t* sc_done = sc_full + 1;
  uint64_t* qdo_full = sc_full + 2;
  uint64_t* qdo_empty = sc_full + 3;
  uint64_t* dp_ready = sc_full + 4;
  uint64_t* grads_full = sc_full + 5;
  uint64_t* grads_empty = sc_full + 6;
  uint64_t* sp_full = sc_full + 7;
  uint64_t* sp_empty = sc_full + 8;
  uint64_t* lb_empty = sc_full + 9;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sc_full + 11);
  uint64_t* sp_read = sc_full + 12;  // dg re-seed tiles: the epilogue has read S' (the producer may reload it)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hh = blockIdx.x / nseg, s = blockIdx.x % nseg;
  int t0, t1;
  seg_range(s, nseg, ntiles, t0, t1);
  const int nt = t1 - t0;
  unsigned long long* tr = (trace != nullptr && (int)blockIdx.x == trace_cta) ? trace : nullptr;
  if (trace != nullptr && threadIdx.x == 0) cta_trace_begin(trace);
  constexpr int DW = PAIR ? 64 : D;  // channels per head in memory
  if constexpr (DENSE) {  // compile-time strides for the dense layout
    gts = DW, ghs = L * DW;
    gs = Strides4{DW, DW, DW, DW, L * DW, L * DW, L * DW, L * DW};
    dr = DW;
  }

  if (tid == 0) {
    for (int i = 0; i < BO_NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 256 + 1);  // the epilogue's reads of Qh / Kh + the MMA warp's last commit
      mbar_init(&prep[i], 128);
    }
    mbar_init(sc_full, 1);
    mbar_init(sc_done, 256);
    mbar_init(qdo_full, 1);
    mbar_init(qdo_empty, 256);
    mbar_init(dp_ready, 256);
    mbar_init(grads_full, 1);
    mbar_init(grads_empty, 256);
    mbar_init(sp_full, 1);
    mbar_init(sp_empty, 1);
    mbar_init(&lb_empty[0], 256);
    mbar_init(&lb_empty[1], 256);
    mbar_init(sp_read, 256);
    fence_barrier_init();
  }
  uint8_t* am1_buf = sp_buf + T * 128;  // PAIR: S' panel 0 rows 64-127
  uint8_t* dpm1_buf = sp_buf + SPANEL;   // PAIR: S' panel 1 rows 0-63
  if (!PAIR && dr < D) {  // d = 64: S' tiles fill only the top-left 64 x 64 block of this buffer
    for (int i = tid; i < STATE_BF16 / 16; i += BO_THREADS) reinterpret_cast<uint4*>(sp_buf)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // under a programmatic (PDL) launch every warp waits for the preceding grid before touching memory;
  // early inputs: only the epilogue warps, whose prologue reads the preceding scan's outputs (Dend, cumGr)
  pdl_trigger();
  // early inputs: no warp waits here; the TMA lane waits before its first S' load, the epilogue warps after
  // reading the forward's segment states (everything they read before it was written >= 2 grids back)
  if (!early) pdl_wait();

  if (warp == 12) {
    // ---------------- TMA producer (tiles right to left)
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_do);
      tma_prefetch_desc(&tm_sp);
      if (ZGLA_G_PREFETCH) tma_prefetch_desc(&tm_g);
      const uint64_t pol = ZGLA_CONSUMER_EVICT_FIRST ? l2_policy_evict_first() : 0;  // 0: no cache hint
      for (int m = 0; m < nt; ++m) {
        const int st = m % BO_NS, ph = (m / BO_NS) & 1;
        const int n = t1 - 1 - m;
        uint8_t* sb = smem + st * BO_STAGE;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], BO_STAGE);
        const int r = n * T;
        if constexpr (PAIR) {
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const CUtensorMap* mx = x == 0 ? &tm_q : x == 1 ? &tm_k : x == 2 ? &tm_v : &tm_do;
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
          tile_load<DENSE>(sb + 3 * TILE_BF16, &tm_do, &full[st], 0, r, hh, L, in3d, pol);
          tile_load<DENSE>(sb + 3 * TILE_BF16 + PANEL, &tm_do, &full[st], 64, r, hh, L, in3d, pol);
        }
        // S' comes from the forward output kernel, which has completed when this grid starts in the entry-point
        // order: every grid between the two (segment pass, segment scan, All-Scan chain) waits for its
        // predecessor before it lets its dependents launch.  ZGLA_SP_WAIT=1 keeps a wait for the preceding
        // grid before the first S' load anyway
        if (ZGLA_SP_WAIT && m == 0 && early) pdl_wait();
        mbar_wait(sp_empty, (m & 1) ^ 1);
        if (m > 0 && reseed_tile(m - 1, nt))  // the previous S' also fed the epilogue's dg re-seed
          mbar_wait(sp_read, ((m / (ZGLA_RHO_RESEED > 0 ? ZGLA_RHO_RESEED : 1)) - 1) & 1);
        if constexpr (PAIR) {  // the two per-head blocks onto the diagonal of the [c][v] buffer
          mbar_arrive_expect_tx(sp_full, 2 * T * 128);
          tma_load_2d(sp_buf, &tm_sp, sp_full, 0, ((2 * hh) * ntiles + n) * 64);
          tma_load_2d(sp_buf + SPANEL + T * 128, &tm_sp, sp_full, 0, ((2 * hh + 1) * ntiles + n) * 64);
        } else if (dr == D) {
          mbar_arrive_expect_tx(sp_full, STATE_BF16);
          const int rs = (hh * ntiles + n) * D;
          tma_load_2d(sp_buf, &tm_sp, sp_full, 0, rs);
          tma_load_2d(sp_buf + SPANEL, &tm_sp, sp_full, 64, rs);
        } else {  // d = 64: the real 64 x 64 block; the rest of the buffer stays zero (cleared at entry)
          mbar_arrive_expect_tx(sp_full, T * 128);
          tma_load_2d(sp_buf, &tm_sp, sp_full, 0, (hh * ntiles + n) * 64);
        }
#if ZGLA_G_PREFETCH
        // warm L2 with the gate tile the prep warps read (pointer loads) ZGLA_G_PREFETCH tiles from now
        if (n - ZGLA_G_PREFETCH >= t0) {
          const int rg = (n - ZGLA_G_PREFETCH) * T;
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
        ZTRACE(tr, 0, m);
      }
    }
  } else if (warp == 13) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_sc = idesc_bf16(64, 64, false, false);
      constexpr uint32_t id_qdo = idesc_bf16(128, 128, true, true);
      constexpr uint32_t id_mk = idesc_bf16(128, 64, true, false);
      constexpr uint32_t id_kk = idesc_bf16(128, 64, false, false);
      constexpr uint32_t id_mm = idesc_bf16(128, 64, true, true);
      // PAIR: per-head M = 64 shapes
      constexpr uint32_t id_mk64 = idesc_bf16(64, 64, true, false);
      constexpr uint32_t id_kk64 = idesc_bf16(64, 64, false, false);
      constexpr uint32_t id_mm64 = idesc_bf16(64, 64, true, true);
      const uint32_t spa = smem_u32(sp_buf), dpa = smem_u32(dp_buf);
      const uint32_t ama = smem_u32(am_buf), dpma = smem_u32(dpm_buf);
      const uint32_t am_e[2] = {ama, smem_u32(am1_buf)}, dpm_e[2] = {dpma, smem_u32(dpm1_buf)};
      for (int m = 0; m < nt; ++m) {
        const int st = m % BO_NS, ph = (m / BO_NS) & 1;
        const uint32_t qa = smem_u32(smem + st * BO_STAGE);
        const uint32_t ka = qa + TILE_BF16, va = qa + 2 * TILE_BF16, da = qa + 3 * TILE_BF16;
        mbar_wait(&prep[st], ph);
        tc_fence_after();
        if constexpr (PAIR) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {  // scores / dP of head e (K = its 64 channels) in lane half e
            const uint32_t lo = (16u * e) << 16;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t off = e * PANEL + kk * 32;
              mma_bf16_ss(tbase + lo + BC_SC, sdesc(qa + off, 16, 1024), sdesc(ka + off, 16, 1024), id_sc, kk > 0);
              mma_bf16_ss(tbase + lo + BC_SC2, sdesc(da + off, 16, 1024), sdesc(va + off, 16, 1024), id_sc, kk > 0);
            }
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {  // scores and dP, K = 128 channels
            const uint32_t off = (kk >> 2) * PANEL + (kk & 3) * 32;
            mma_bf16_ss(tbase + BC_SC, sdesc(qa + off, 16, 1024), sdesc(ka + off, 16, 1024), id_sc, kk > 0);
            mma_bf16_ss(tbase + (16u << 16) + BC_SC, sdesc(da + off, 16, 1024), sdesc(va + off, 16, 1024), id_sc,
                        kk > 0);
          }
        }
        mma_commit(sc_full);
        ZTRACE(tr, 2, m);
        mbar_wait(sc_done, m & 1);
        mbar_wait(grads_empty, (m & 1) ^ 1);
        mbar_wait(sp_full, m & 1);
        tc_fence_after();
        ZTRACE(tr, 3, m);
        if constexpr (PAIR) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t lo = (16u * e) << 16;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // dq^T_e = Kh_e^T dPm_e^T
              mma_bf16_ss(tbase + lo + BC_DQ, sdesc(ka + e * PANEL + kk * 2048, PANEL, 1024),
                          sdesc(dpm_e[e] + kk * 32, 16, 1024), id_mk64, kk > 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // dq^T_e += S'_ee dO_e^T (rows 64e.. of panel e)
              mma_bf16_ss(tbase + lo + BC_DQ, sdesc(spa + e * SPANEL + e * (T * 128) + kk * 32, 16, 1024),
                          sdesc(da + e * PANEL + kk * 32, 16, 1024), id_kk64, 1);
          }
          mma_commit(sp_empty);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t lo = (16u * e) << 16;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // dk^T_e = Qh_e^T dPm_e ; dv^T_e = dO_e^T Am_e
              mma_bf16_ss(tbase + lo + BC_DK, sdesc(qa + e * PANEL + kk * 2048, PANEL, 1024),
                          sdesc(dpm_e[e] + kk * 2048, PANEL, 1024), id_mm64, kk > 0);
              mma_bf16_ss(tbase + lo + BC_DV, sdesc(da + e * PANEL + kk * 2048, PANEL, 1024),
                          sdesc(am_e[e] + kk * 2048, PANEL, 1024), id_mm64, kk > 0);
            }
          }
          mbar_wait(dp_ready, m & 1);
          tc_fence_after();
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t lo = (16u * e) << 16;
            const uint32_t dpe = dpa + e * SPANEL + e * (T * 128);  // D'_ee: rows 64e.. of panel e
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // dk^T_e += D'_ee V_e^T ; dv^T_e += D'_ee^T Kh_e^T
              mma_bf16_ss(tbase + lo + BC_DK, sdesc(dpe + kk * 32, 16, 1024), sdesc(va + e * PANEL + kk * 32, 16, 1024),
                          id_kk64, 1);
              mma_bf16_ss(tbase + lo + BC_DV, sdesc(dpe + kk * 2048, SPANEL, 1024),
                          sdesc(ka + e * PANEL + kk * 32, 16, 1024), id_mk64, 1);
            }
          }
          mma_commit(grads_full);
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int kk = 0; kk < T / 16; ++kk)  // Dt_e += Qh_e^T dO_e
              mma_bf16_ss(tbase + ((16u * e) << 16) + BC_QDO, sdesc(qa + e * PANEL + kk * 2048, PANEL, 1024),
                          sdesc(da + e * PANEL + kk * 2048, PANEL, 1024), id_mm64, 1);
        } else {
#pragma unroll
          for (int kk = 0; kk < T / 16; ++kk)  // dq^T = Kh^T dPm^T
            mma_bf16_ss(tbase + BC_DQ, sdesc(ka + kk * 2048, PANEL, 1024), sdesc(dpma + kk * 32, 16, 1024), id_mk,
                        kk > 0);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)  // dq^T += S' dO^T
            mma_bf16_ss(tbase + BC_DQ, sdesc(spa + (kk >> 2) * SPANEL + (kk & 3) * 32, 16, 1024),
                        sdesc(da + (kk >> 2) * PANEL + (kk & 3) * 32, 16, 1024), id_kk, 1);
          mma_commit(sp_empty);
#pragma unroll
          for (int kk = 0; kk < T / 16; ++kk) {  // dk^T = Qh^T dPm ; dv^T = dO^T Am  (independent of D')
            mma_bf16_ss(tbase + BC_DK, sdesc(qa + kk * 2048, PANEL, 1024), sdesc(dpma + kk * 2048, PANEL, 1024), id_mm,
                        kk > 0);
            mma_bf16_ss(tbase + BC_DV, sdesc(da + kk * 2048, PANEL, 1024), sdesc(ama + kk * 2048, PANEL, 1024), id_mm,
                        kk > 0);
          }
          mbar_wait(dp_ready, m & 1);  // D' in smem and Dt rescaled in TMEM
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < (ZGLA_ABL_PART2 ? 0 : D / 16); ++kk) {  // dk^T += D' V^T ; dv^T += D'^T Kh^T
            const uint32_t boff = (kk >> 2) * PANEL + (kk & 3) * 32;
            mma_bf16_ss(tbase + BC_DK, sdesc(dpa + (kk >> 2) * SPANEL + (kk & 3) * 32, 16, 1024),
                        sdesc(va + boff, 16, 1024), id_kk, 1);
            mma_bf16_ss(tbase + BC_DV, sdesc(dpa + kk * 2048, SPANEL, 1024), sdesc(ka + boff, 16, 1024), id_mk, 1);
          }
          mma_commit(grads_full);
          // the state cotangent update is needed only by the next tile's rescale: issue it last
#pragma unroll
          for (int kk = 0; kk < T / 16; ++kk)  // Dt += Qh^T dO
            mma_bf16_ss(tbase + BC_QDO, sdesc(qa + kk * 2048, PANEL, 1024), sdesc(da + kk * 2048, PANEL, 1024),
                        id_qdo, 1);
        }
        mma_commit(qdo_full);
        mma_commit(&empty[st]);  // QDO reads q / dO of this stage
        ZTRACE(tr, 4, m);
      }
    }
  } else if (warp >= 8) {
    // ---------------- prep: one thread per channel c (warp w handles TMEM lane quarter w%4):
    //   logb over the 64 tile rows, r = logb[31], gamma = logb[63], Qh / Kh in place,
    //   d = logb - r -> TMEM (double buffered) for the epilogue
    const int c = PAIR ? pair_channel(tid - 256) : tid - 256;  // PAIR: the channel of TMEM lane tid - 256
    const int quarter = (tid - 256) >> 5;
    const uint32_t coff = (c >> 6) * PANEL + (c & 7) * 2, cchk = (c & 63) >> 3;
    constexpr float LOG2E = 1.4426950408889634f;
    for (int m = 0; m < nt; ++m) {
      const int st = m % BO_NS, ph = (m / BO_NS) & 1;
      const int n = t1 - 1 - m;
      uint8_t* sb = smem + st * BO_STAGE;
      float lb[64];
      const float* gp = PAIR ? g + (2 * hh + (c >> 6)) * ghs + (long long)n * T * gts + (c & 63)
                             : g + hh * ghs + (long long)n * T * gts + c;
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
      const float gam = (lb[63] - rr) + rr;  // (same rounding as the unscaled walk)
#pragma unroll
      for (int r = 0; r < 64; ++r) lb[r] = (lb[r] - rr) * LOG2E;  // log2-scaled d: TMEM holds it for the epilogue
      if (c == 0) ZTRACE(tr, 10, m);
      mbar_wait(&full[st], ph);
      if (c == 0) ZTRACE(tr, 11, m);
      vgam[st * D + c] = gam;
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
          const float d = lb[r0 + r];
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
      mbar_wait(&lb_empty[m & 1], ((m >> 1) & 1) ^ 1);
      tc_fence_after();
      {
        const uint32_t la = taddr(tbase, 32 * quarter, BC_LB + 64 * (m & 1));
        tmem_st32(la, *reinterpret_cast<const float(*)[32]>(&lb[0]));
        tmem_st32(la + 32, *reinterpret_cast<const float(*)[32]>(&lb[32]));
      }
      tc_fence_before();
      fence_proxy_async();
      mbar_arrive(&prep[st]);
      if (c == 0) ZTRACE(tr, 1, m);
    }
  } else {
    // ---------------- state / epilogue warps: thread (c, ch) owns Dt[c][64*ch .. +64] (TMEM) and,
    //                  in the epilogue, tokens [32*ch, 32*ch+32) of channel c
    const int qd = warp & 3, ch = warp >> 2;
    // PAIR: this thread's TMEM lane holds channel c (head e = c / 64) and columns [32*ch, 32*ch+32) of that
    // head's 64-column Dt block; otherwise channel 32*qd + lane and columns [64*ch, 64*ch+64)
    const int c = PAIR ? pair_channel(32 * qd + lane) : 32 * qd + lane;
    const int he = c >> 6;                                       // PAIR: head of the pair
    const int vcol0 = PAIR ? 64 * he + 32 * ch : 64 * ch;        // first state column (v) of this thread
    const uint32_t d_addr = taddr(tbase, 32 * qd, BC_QDO + (PAIR ? 32 * ch : 64 * ch));
    constexpr int NHF = PAIR ? 1 : 2;                            // 32-column halves held per thread
    {
      const long long sidx = (long long)(hh * nseg + s) * D * D + c;  // column-major workspace states
      const float cg = s_prev ? expf(cumG[(hh * nseg + s) * D + c]) : 0.f;
      const float eg = expf(gamseg[(hh * nseg + s) * D + c]);
      // API states are [h][dr][dr]; PAIR: head 2*hh + he, row c % 64
      const long long pidx = PAIR ? ((long long)(2 * hh + he) * 64 + (c & 63)) * 64 + 32 * ch
                                  : ((long long)hh * dr + c) * dr + 64 * ch;
      // (1) fp32 forward state at the segment end, e^{gam_s} S_in + dS_s: the forward's outputs (complete
      //     when this grid starts, see fwd/bwd launch order), so with early inputs this overlaps the
      //     preceding scan / All-Scan grid; explicit FMAs: the same rounding in every kernel variant
      float se[NHF][32];
#pragma unroll
      for (int hf = 0; hf < NHF; ++hf)
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const int jj = 32 * hf + j;
          const long long o = sidx + (long long)(vcol0 + jj) * D;
          float4 si = make_float4(Sin[o], Sin[o + D], Sin[o + 2 * D], Sin[o + 3 * D]);
          const float4 ds = make_float4(dS[o], dS[o + D], dS[o + 2 * D], dS[o + 3 * D]);
          const bool inb = PAIR || (c < dr && 64 * ch + jj < dr);
          if (s_prev && inb) {
            const float4 a = *reinterpret_cast<const float4*>(s_prev + pidx + jj);
            si.x = fmaf(cg, a.x, si.x); si.y = fmaf(cg, a.y, si.y);
            si.z = fmaf(cg, a.z, si.z); si.w = fmaf(cg, a.w, si.w);
          }
          se[hf][j] = fmaf(eg, si.x, ds.x);
          se[hf][j + 1] = fmaf(eg, si.y, ds.y);
          se[hf][j + 2] = fmaf(eg, si.z, ds.z);
          se[hf][j + 3] = fmaf(eg, si.w, ds.w);
        }
      if (early) pdl_wait();  // (2) the cotangent comes from the preceding scan / All-Scan grids
      const float cgr = ds_next ? expf(cumGr[(hh * nseg + s) * D + c]) : 0.f;
      float rho = 0.f;
#pragma unroll
      for (int hf = 0; hf < NHF; ++hf) {
        float dv32[32];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const int jj = 32 * hf + j;
          const long long o = sidx + (long long)(vcol0 + jj) * D;
          float4 dd = make_float4(Dend[o], Dend[o + D], Dend[o + 2 * D], Dend[o + 3 * D]);
          const bool inb = PAIR || (c < dr && 64 * ch + jj < dr);
          if (ds_next && inb) {
            const float4 a = *reinterpret_cast<const float4*>(ds_next + pidx + jj);
            dd.x = fmaf(cgr, a.x, dd.x); dd.y = fmaf(cgr, a.y, dd.y);
            dd.z = fmaf(cgr, a.z, dd.z); dd.w = fmaf(cgr, a.w, dd.w);
          }
          dv32[j] = dd.x; dv32[j + 1] = dd.y; dv32[j + 2] = dd.z; dv32[j + 3] = dd.w;
          rho = fmaf(se[hf][j], dd.x, rho);
          rho = fmaf(se[hf][j + 1], dd.y, rho);
          rho = fmaf(se[hf][j + 2], dd.z, rho);
          rho = fmaf(se[hf][j + 3], dd.w, rho);
        }
        tmem_st32(d_addr + 32 * hf, dv32);  // Dt at the segment end (frame r = 0)
      }
      xrho[ch * D + c] = rho;
    }
    tc_fence_before();
    named_bar(2, 256);
    if (tid == 0) ZTRACE(tr, 7, 0);
    if (ch == 0) xr[c] = xrho[c] + xrho[D + c];
    const uint32_t cbase = (c >> 6) * PANEL + (c & 7) * 2;
    const uint32_t cchunk = (c & 63) >> 3;
    float r_next = 0.f;  // reference point of the previously processed (later) tile
    for (int m = 0; m < nt; ++m) {
      const int st = m % BO_NS, ph = (m / BO_NS) & 1;
      const int n = t1 - 1 - m;
      // (a) masked scores (lanes 0-15) and dP (lanes 16-31) -> bf16 operands
      mbar_wait(sc_full, m & 1);
      tc_fence_after();
      if (tid == 0) ZTRACE(tr, 5, m);
#pragma unroll
      for (int pass = 0; pass < (PAIR ? 2 : 1); ++pass) {  // PAIR: scores (lane half = head), then dP
        float a[32];
        tmem_ld32(taddr(tbase, 32 * qd, (PAIR && pass ? BC_SC2 : BC_SC) + 32 * ch), a);
        const int i = 16 * qd + (lane & 15);
        uint8_t* dstbuf = PAIR ? (pass ? (lane < 16 ? dpm_buf : dpm1_buf) : (lane < 16 ? am_buf : am1_buf))
                               : (lane < 16 ? am_buf : dpm_buf);
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
          const int j0 = 32 * ch + 8 * mm;
          float x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = (j0 + u <= i) ? a[8 * mm + u] : 0.f;
          uint4 w;
          w.x = pack_bf16(x[0], x[1]);
          w.y = pack_bf16(x[2], x[3]);
          w.z = pack_bf16(x[4], x[5]);
          w.w = pack_bf16(x[6], x[7]);
          *reinterpret_cast<uint4*>(dstbuf + sw128(i, 4 * ch + mm)) = w;
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(sc_done);
      // (b) rescale Dt_{n+1} into this tile's frame: Dt <- f Dt, D' = f Dt (bf16 [c][v]),
      //     f = e^{gam_n - r_n + r_{n+1}}; the MMA then accumulates Qh^T dO into Dt
      mbar_wait(&prep[st], ph);
      const float gam_c = vgam[st * D + c], r_c = vr[st * D + c];
      if (m > 0) mbar_wait(qdo_full, (m - 1) & 1);
      tc_fence_after();
      if constexpr (DENSE && ZGLA_DG_TMA) {  // dp_buf staged the previous tile's dg: its bulk store has read it
        if (tid == 0) tma_store_wait_read0();
        named_bar(3, 256);
      }
      {
        const float f = fast_exp(gam_c - r_c + r_next);
        uint8_t* dst = dp_buf + (PAIR ? he : ch) * SPANEL;  // D' [c][v]: PAIR writes the head's diagonal block
#pragma unroll 1
        for (int hf = 0; hf < NHF; ++hf) {
          float x[32];
          tmem_ld32_nw(d_addr + 32 * hf, *reinterpret_cast<uint32_t(*)[32]>(x));
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) x[j] *= f;
          tmem_st32(d_addr + 32 * hf, x);
#pragma unroll
          for (int mm = 0; mm < 4; ++mm) {
            uint4 w;
            w.x = pack_bf16(x[8 * mm], x[8 * mm + 1]);
            w.y = pack_bf16(x[8 * mm + 2], x[8 * mm + 3]);
            w.z = pack_bf16(x[8 * mm + 4], x[8 * mm + 5]);
            w.w = pack_bf16(x[8 * mm + 6], x[8 * mm + 7]);
            *reinterpret_cast<uint4*>(dst + sw128(c, (PAIR ? 4 * ch : 4 * hf) + mm)) = w;
          }
        }
      }
      r_next = r_c;
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(dp_ready);
      if (tid == 0) ZTRACE(tr, 6, m);
      // (d) epilogue: thread owns channel c, tokens [32*ch, 32*ch+32): one TMEM pass stores dq/dk/dv and
      //     keeps da = Qh dq_raw - Kh dk_raw; dg_i = rho_{n+1} + sum_{i' >= i in tile} da_i'
      mbar_wait(grads_full, m & 1);
      tc_fence_after();
      if (tid == 0) ZTRACE(tr, 8, m);
      const bool reseed = reseed_tile(m, nt);
      if (reseed) {
        // the suffix sum of da beyond this tile's start from the state identity rho_n = rowsum(S_n (.) D_n) =
        // rowsum(S'_n (.) Dt_n) (both in this tile's frame; Dt_n after this tile's accumulation), so the bf16
        // error of da does not accumulate along long segments.  The producer holds the next S' load until
        // this read (sp_read).
        mbar_wait(sp_full, m & 1);
        mbar_wait(qdo_full, m & 1);
        tc_fence_after();
        const uint8_t* srow = sp_buf + (PAIR ? he : ch) * SPANEL;
        float part = 0.f;
#pragma unroll 1
        for (int hf = 0; hf < NHF; ++hf) {
          float x[32];
          tmem_ld32(d_addr + 32 * hf, x);
#pragma unroll
          for (int mm = 0; mm < 4; ++mm) {
            const uint4 w = *reinterpret_cast<const uint4*>(srow + sw128(c, (PAIR ? 4 * ch : 4 * hf) + mm));
            const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              part = fmaf(__uint_as_float(wv[u] << 16), x[8 * mm + 2 * u], part);
              part = fmaf(__uint_as_float(wv[u] & 0xffff0000u), x[8 * mm + 2 * u + 1], part);
            }
          }
        }
        mbar_arrive(sp_read);
        xrho[ch * D + c] = part;
      }
      const uint8_t* sb = smem + st * BO_STAGE;
      const uint32_t cols = 32 * ch;
      const uint32_t lbcol = BC_LB + 64 * (m & 1) + cols;
      const long long tok0 = (long long)n * T + cols;  // token index inside the head
      float da[32];
      float tsum = 0.f;
      const int oh = PAIR ? 2 * hh + he : hh, oc = PAIR ? (c & 63) : c;  // output head / channel
      __nv_bfloat16* pdq = dq + oh * gs.qh + tok0 * gs.qt + oc;
      __nv_bfloat16* pdk = dk + oh * gs.kh + tok0 * gs.kt + oc;
      __nv_bfloat16* pdv = dv + oh * gs.vh + tok0 * gs.vt + oc;
#pragma unroll
      for (int h8 = 0; h8 < 4; ++h8) {
        uint32_t gq[8], gk[8], gv8[8], dl[8];
        tmem_ld8_nw(taddr(tbase, 32 * qd, BC_DQ + cols + 8 * h8), gq);
        tmem_ld8_nw(taddr(tbase, 32 * qd, BC_DK + cols + 8 * h8), gk);
        tmem_ld8_nw(taddr(tbase, 32 * qd, BC_DV + cols + 8 * h8), gv8);
        tmem_ld8_nw(taddr(tbase, 32 * qd, lbcol + 8 * h8), dl);
        // shared-memory operands first: the global stores below go through generic pointers and
        // would otherwise serialise every later shared load behind them
        float qh[8], kh[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t o = cbase + sw128(cols + 8 * h8 + u, cchunk);
          qh[u] = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(sb + o));
          kh[u] = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(sb + TILE_BF16 + o));
        }
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = 8 * h8 + u;
          const float q_raw = __uint_as_float(gq[u]), k_raw = __uint_as_float(gk[u]);
          const float dlt = __uint_as_float(dl[u]);  // (logb - r) * log2(e), from the prep warps
          da[i] = __fsub_rn(__fmul_rn(qh[u], q_raw), __fmul_rn(kh[u], k_raw));  // no FMA contraction: identical in every variant
          tsum += da[i];
          if (DENSE || PAIR || c < dr) {  // channels of a d = 64 head beyond 64 are padding
            *pdq = __float2bfloat16_rn(q_raw * fast_exp2(dlt));
            *pdk = __float2bfloat16_rn(k_raw * fast_exp2(-dlt));
            *pdv = __float2bfloat16_rn(__uint_as_float(gv8[u]));
          }
          pdq += gs.qt, pdk += gs.kt, pdv += gs.vt;
        }
      }
      tc_fence_before();
      mbar_arrive(grads_empty);
      mbar_arrive(&lb_empty[m & 1]);
      mbar_arrive(&empty[st]);  // stage reads (Qh, Kh) done
      xcarry[ch * D + c] = tsum;
      named_bar(2, 256);
      const float rho_end = xr[c];
      const float t_upper = xcarry[D + c], t_lower = xcarry[c];
      float base = rho_end + (ch == 0 ? t_lower + t_upper : t_upper);
      if constexpr (DENSE && ZGLA_DG_TMA) {
        // dg rows -> the D' buffer (free from grads_full until the next tile's rescale) as fp32 [token][channel]
        // (PAIR: one [64][64] block per head), then one bulk tensor store per head: whole-wavefront STS instead
        // of 32 scalar global stores per thread
        float* stg = reinterpret_cast<float*>(dp_buf) + (PAIR ? he * (T * 64) + cols * 64 + oc : cols * D + c);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          stg[i * DW] = base;
          base -= da[i];
        }
        fence_proxy_async();
        if (tid == 0) ZTRACE(tr, 9, m);
        named_bar(2, 256);  // staging complete; everyone has read xr / xcarry of this tile
        if (tid == 0) {
          if constexpr (PAIR) {
            tma_store_2d(&tm_dg, dp_buf, 0, (int)((2 * hh) * L + (long long)n * T));
            tma_store_2d(&tm_dg, dp_buf + T * 64 * 4, 0, (int)((2 * hh + 1) * L + (long long)n * T));
          } else {
            tma_store_2d(&tm_dg, dp_buf, 0, (int)(hh * L + (long long)n * T));
          }
          tma_store_commit();
        }
      } else {
        float* pdg = dg + oh * gs.gh + tok0 * gs.gt + oc;
#pragma unroll
        for (int i = 0; i < 32; ++i, pdg += gs.gt) {
          if (DENSE || PAIR || c < dr) *pdg = base;
          base -= da[i];
        }
        if (tid == 0) ZTRACE(tr, 9, m);
        named_bar(2, 256);  // everyone has read xr / xcarry of this tile
      }
      if (ch == 0) xr[c] = reseed ? xrho[c] + xrho[D + c] : rho_end + t_lower + t_upper;  // rho at this tile's start
    }
    if (nt > 0) mbar_wait(qdo_full, (nt - 1) & 1);  // last Dt accumulation retired before dealloc
    if constexpr (DENSE && ZGLA_DG_TMA) {
      if (tid == 0) tma_store_wait0();  // the last dg store has left shared memory (and completed)
    }
  }
  tc_fence_before();
  __syncthreads();
  if (trace != nullptr && threadIdx.x == 0) cta_trace_end(trace);
  if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace fast

using namespace fast;

int fast_bwd_output(const zgla_shape* s, int num_sms, const TRef& q, const TRef& k, const TRef& v, const TRef& g,
                    const TRef& d_out, void* ws, const void* s_prev, const void* ds_next, const TRef& dq,
                    const TRef& dk, const TRef& dv, const TRef& dg, cudaStream_t st) {
  const Plan pl = make_plan(s, num_sms);
  Ws w = carve(pl, ws);
  CUtensorMap mq, mk, mv, mdo, msp, mg;
  const int early = pdl_enabled() && early_inputs();
  if (pl.pair) {
    const int heads = 2 * pl.h;
    if (int rc = map_act_pair(&mq, q, pl.L, heads)) return rc;
    if (int rc = map_act_pair(&mk, k, pl.L, heads)) return rc;
    if (int rc = map_act_pair(&mv, v, pl.L, heads)) return rc;
    if (int rc = map_act_pair(&mdo, d_out, pl.L, heads)) return rc;
    if (int rc = sp_map_pair(&msp, w.Sp, pl)) return rc;
    if (int rc = map_gate_pair(&mg, g, pl.L, heads)) return rc;
    const Strides4 gs{(int)dq.ts, (int)dk.ts, (int)dv.ts, (int)dg.ts, dq.hs, dk.hs, dv.hs, dg.hs};
    const bool dn = is_dense64(g, pl.L) && is_dense64(dq, pl.L) && is_dense64(dk, pl.L) && is_dense64(dv, pl.L) &&
                    is_dense64(dg, pl.L);
    auto kern = dn ? bwd_out_kernel<true, true> : bwd_out_kernel<false, true>;
    CUtensorMap mdg = mg;  // dense: fp32 [2h * L][64], one [64 tokens][64 channels] box per head
    if (dn && ZGLA_DG_TMA)
      if (int rc = make_map(&mdg, dg.p, false, (unsigned long long)heads * pl.L, 64, 64, T, false)) return rc;
    set_smem_once((const void*)kern, (int)BO_SMEM);
    if (cudaError_t e = launch_kp(pdl_enabled(), kern, pl.h * pl.nseg, BO_THREADS, BO_SMEM, st, mq, mk, mv, mdo, msp,
                                  mg, mdg, (const float*)g.p, g.ts, g.hs, pl.L, 1, 64, pl.nseg, pl.ntiles,
                                  (const float*)w.Sin, (const float*)w.cumG, (const float*)w.dS, (const float*)w.gam,
                                  (const float*)s_prev, (const float*)w.Dend, (const float*)w.cumGr,
                                  (const float*)ds_next, (__nv_bfloat16*)dq.p, (__nv_bfloat16*)dk.p,
                                  (__nv_bfloat16*)dv.p, (float*)dg.p, gs, g_trace_buf, g_trace_cta, early))
      return cuda_fail(e, "bwd_out_kernel (pairs)");
    return zgla_check_launch();
  }
  const bool din = is_dense(q, pl.L) && is_dense(k, pl.L) && is_dense(v, pl.L) && is_dense(d_out, pl.L);
  const bool dn = is_dense(g, pl.L) && is_dense(dq, pl.L) && is_dense(dk, pl.L) && is_dense(dv, pl.L) &&
                  is_dense(dg, pl.L);
  if (int rc = map_act(&mq, q, pl.L, pl.h, din)) return rc;
  if (int rc = map_act(&mk, k, pl.L, pl.h, din)) return rc;
  if (int rc = map_act(&mv, v, pl.L, pl.h, din)) return rc;
  if (int rc = map_act(&mdo, d_out, pl.L, pl.h, din)) return rc;
  if (int rc = sp_map(&msp, w.Sp, pl, q.dr)) return rc;
  if (int rc = map_gate(&mg, g, pl.L, pl.h, din && is_dense(g, pl.L))) return rc;
  const Strides4 gs{(int)dq.ts, (int)dk.ts, (int)dv.ts, (int)dg.ts, dq.hs, dk.hs, dv.hs, dg.hs};
  auto kern = dn ? bwd_out_kernel<true> : bwd_out_kernel<false>;
  CUtensorMap mdg = mg;  // dense: fp32 [h * L][128], one [64 tokens][128 channels] box per tile
  if (dn && ZGLA_DG_TMA)
    if (int rc = make_map(&mdg, dg.p, false, (unsigned long long)pl.h * pl.L, D, D, T, false)) return rc;
  set_smem_once((const void*)kern, (int)BO_SMEM);
  if (cudaError_t e = launch_kp(pdl_enabled(), kern, pl.h * pl.nseg, BO_THREADS, BO_SMEM, st, mq, mk, mv, mdo, msp, mg,
                                mdg, (const float*)g.p, g.ts, g.hs, pl.L, din ? 0 : 1, q.dr, pl.nseg, pl.ntiles,
                                (const float*)w.Sin, (const float*)w.cumG, (const float*)w.dS, (const float*)w.gam, (const float*)s_prev,
                                (const float*)w.Dend, (const float*)w.cumGr, (const float*)ds_next,
                                (__nv_bfloat16*)dq.p, (__nv_bfloat16*)dk.p, (__nv_bfloat16*)dv.p, (float*)dg.p, gs,
                                g_trace_buf, g_trace_cta, early))
    return cuda_fail(e, "bwd_out_kernel");
  return zgla_check_launch();
}

}  // namespace zgla
