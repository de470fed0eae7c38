// Shared pieces of the fused tcgen05 ZeCO kernels (bf16 storage, fp32 state).
//
// Geometry: head dim D = dk = dv = 128, tile T = 64 tokens.  Each head's shard
// of L tokens (NT = L/64 tiles) is cut into `nseg` contiguous SEGMENTS, one CTA
// each, so the grid is heads x nseg ~ one wave of 148 SMs.  The ZeCO identity
// (Appendix A) is applied *inside* the GPU as well: every
// segment first computes its local state contribution from zero, a small
// elementwise scan over segments gives each segment its incoming state, and
// the output kernel starts from that state.  Across GPUs the same identity is
// applied once more by All-Scan.
#pragma once
#include <cudaTypedefs.h>

#include <cstdlib>
#include <utility>

#include "tc.cuh"
#include "zgla_internal.h"

#ifndef ZGLA_L2_KEEP_PCT
#define ZGLA_L2_KEEP_PCT 20  // percent of a producer walk (K1 / K4) loaded with normal L2 priority (tuned: 0.3995 -> 0.3895 ms)
#endif
#ifndef ZGLA_G_PREFETCH
#define ZGLA_G_PREFETCH 1  // bwd: L2 prefetch of the gate tile this many tiles ahead (0: off); 1 tuned (2: worse)
#endif
#ifndef ZGLA_G_PREFETCH_FWD
#define ZGLA_G_PREFETCH_FWD 1  // fwd: L2 prefetch of the gate tile this many tiles ahead (0: off)
#endif
#ifndef ZGLA_O_TMA
#define ZGLA_O_TMA 1  // fwd: O through a swizzled staging tile and bulk tensor stores (dense outputs)
#endif
#ifndef ZGLA_DG_TMA
#define ZGLA_DG_TMA 1  // bwd: dg staged in the free D' buffer and written with bulk tensor stores (dense outputs)
#endif
#ifndef ZGLA_CONSUMER_EVICT_FIRST
#define ZGLA_CONSUMER_EVICT_FIRST 0  // consumer kernels (K3 / K6): 1 = evict-first hint, 0 = plain loads
#endif

namespace zgla {
namespace fast {

constexpr int D = 128;                 // head dim (dk = dv)
constexpr int T = 64;                  // tokens per tile
constexpr int PANEL = T * 128;         // one 64-column SW128 panel of a [64 x D] bf16 tile (8 KiB)
constexpr int TILE_BF16 = T * D * 2;   // 16 KiB
constexpr int TILE_F32 = T * D * 4;    // 32 KiB
constexpr int SPANEL = D * 128;        // one 64-column panel of a [D x D] bf16 state (16 KiB)
constexpr int STATE_BF16 = D * D * 2;  // 32 KiB

struct Plan {
  int h, nseg, ntiles;  // h: CTA heads (head PAIRS when pair != 0)
  long long L;
  int pair;  // d = 64 with an even head count: two heads per 128-channel CTA
};

__host__ __device__ inline void seg_range(int s, int nseg, int ntiles, int& t0, int& t1) {
  t0 = (int)((long long)s * ntiles / nseg);
  t1 = (int)((long long)(s + 1) * ntiles / nseg);
}

// workspace carve-up (fp32 unless noted), per shard
// Segment states are stored column-major per (head, segment): element (c, v) at v * D + c, so the
// thread-per-channel (TMEM lane) readers and writers touch 128 contiguous bytes per warp.
struct Ws {
  float* dS;      // [h][nseg][D][D]  fwd: segment-local final state from zero
  float* gam;     // [h][nseg][D]     segment total log decay
  float* Sin;     // [h][nseg][D][D]  fwd: rank-local state at segment start (exclusive scan)
  float* cumG;    // [h][nseg][D]     sum of gam over earlier segments
  float* dD;      // [h][nseg][D][D]  bwd: state cotangent at segment start from the segment's tokens
  float* Dend;    // [h][nseg][D][D]  bwd: rank-local cotangent at segment end (later segments)
  float* cumGr;   // [h][nseg][D]     sum of gam over later segments
  __nv_bfloat16* Sp;  // [h][NT][D][D] bf16: scaled chunk-start states e^{r} S for the backward
  int* flags;         // [h * nseg]: per forward segment-pass CTA, a 64-token tile's log-decay left the
                      // fast path's exponent domain
};

// The fused kernels scale q / k by e^{+-(logb - r)} with r the tile's middle row, so a tile whose total
// log-decay is below -2 * DOMAIN_EXP overflows fp32 / bf16.  The forward segment pass flags it.
constexpr float DOMAIN_EXP = 80.f;

inline long long ws_bytes(const Plan& p) {
  const long long st = (long long)p.h * p.nseg * D * D * 4;
  const long long vec = (long long)p.h * p.nseg * D * 4;
  const long long sp = (long long)p.h * p.ntiles * STATE_BF16;
  return 4 * st + 3 * vec + sp + 4096 + (((long long)p.h * p.nseg * 4 + 255) & ~255ll);
}

inline Ws carve(const Plan& p, void* base) {
  const long long st = (long long)p.h * p.nseg * D * D;
  const long long vec = (long long)p.h * p.nseg * D;
  float* f = reinterpret_cast<float*>(base);
  Ws w;
  w.dS = f;
  w.Sin = w.dS + st;
  w.dD = w.Sin + st;
  w.Dend = w.dD + st;
  w.gam = w.Dend + st;
  w.cumG = w.gam + vec;
  w.cumGr = w.cumG + vec;
  uintptr_t sp = reinterpret_cast<uintptr_t>(w.cumGr + vec);
  sp = (sp + 1023) & ~uintptr_t(1023);
  w.Sp = reinterpret_cast<__nv_bfloat16*>(sp);
  w.flags = reinterpret_cast<int*>(sp + (uintptr_t)p.h * p.ntiles * STATE_BF16);
  return w;
}

inline bool pair_mode(const zgla_shape* s) {
  static const bool off = std::getenv("ZGLA_NO_PAIR") != nullptr;  // A/B: d = 64 heads zero-filled to 128
  return s->key_dim == 64 && s->heads % 2 == 0 && !off;
}

inline Plan make_plan(const zgla_shape* s, int num_sms) {
  Plan p;
  p.pair = pair_mode(s) ? 1 : 0;
  p.h = p.pair ? s->heads / 2 : s->heads;
  p.L = s->seq_len;
  p.ntiles = (int)(s->seq_len / T);
  int nseg = num_sms / (p.h > 0 ? p.h : 1);
  if (nseg < 1) nseg = 1;
  if (nseg > p.ntiles) nseg = p.ntiles;
  p.nseg = nseg;
  return p;
}

// ---- host: TMA descriptors via the driver entry point (no libcuda link dependency)
// The driver call needs a current context in the calling thread.  A thread that has not touched the runtime
// yet (e.g. torch's autograd worker running a backward first) has none, and the encode fails with
// CUDA_ERROR_INVALID_CONTEXT: bind the device's primary context once per thread (cudaFree(0)).
inline void bind_context_once() {
  static thread_local bool bound = false;
  if (!bound) {
    cudaFree(nullptr);
    bound = true;
  }
}
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  bind_context_once();
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 2-D map over a row-major [rows][cols] tensor
inline int make_map(CUtensorMap* m, const void* base, bool bf16, unsigned long long rows, unsigned cols,
                    unsigned box_cols, unsigned box_rows, bool swizzle128) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZGLA_ERR_CUDA;
  }
  const unsigned eb = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * eb};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d)", (int)r);
    set_error(buf);
    return ZGLA_ERR_CUDA;
  }
  return ZGLA_OK;
}

// a [heads][tokens][D] tensor with arbitrary token / head strides (elements; channels contiguous)
struct TRef {
  const void* p;
  long long ts;  // token stride
  long long hs;  // head stride
  int dr;        // channels actually stored (128, or 64: the kernels see 128 with the rest zero-filled)
};
// token / head strides of the four gradient outputs of the backward kernel (elements)
struct Strides4 {  // token strides fit in 32 bits (fewer live registers in the epilogue); head strides not
  int qt, kt, vt, gt;
  long long qh, kh, vh, gh;
};
inline TRef dense_ref(const void* p, long long L) { return TRef{p, D, L * D, D}; }
inline TRef as_ref(const zgla_tensor* t, long long L, int heads, int dr) {
  // a single head's head stride is irrelevant: normalise it so dense single-head views stay dense
  return TRef{t->data, t->token_stride ? t->token_stride : dr,
              (t->head_stride && heads > 1) ? t->head_stride : L * dr, dr};
}
// TMA needs 16-byte aligned bases and strides; channel rows are 16-byte vectors for the stores
inline bool ref_ok(const TRef& r, int esize) {
  return r.p && (reinterpret_cast<uintptr_t>(r.p) & 15) == 0 && (r.ts * esize) % 16 == 0 &&
         (r.hs * esize) % 16 == 0 && r.ts >= r.dr && r.ts < (1ll << 31) && r.hs >= 0;
}

// 3-D map (channels, tokens, heads) over a strided [heads][tokens][D] tensor; box = box_cols x box_rows x 1
inline int make_map3(CUtensorMap* m, const TRef& r, bool bf16, long long L, int heads, unsigned box_cols,
                     unsigned box_rows, bool swizzle128) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZGLA_ERR_CUDA;
  }
  const unsigned eb = bf16 ? 2 : 4;
  // channels beyond r.dr are outside the map: TMA zero-fills them (d = 64 heads run the d = 128 kernels)
  cuuint64_t dims[3] = {(cuuint64_t)r.dr, (cuuint64_t)L, (cuuint64_t)heads};
  cuuint64_t strides[2] = {(cuuint64_t)(r.ts * eb), (cuuint64_t)((r.hs ? r.hs : L * r.dr) * eb)};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult e = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                  const_cast<void*>(r.p), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (e != CUDA_SUCCESS) {
    char buf[128];
    std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)e);
    set_error(buf);
    return ZGLA_ERR_CUDA;
  }
  return ZGLA_OK;
}
// saved chunk-start states S' (bf16): [h * NT * 128 rows][128] in two 64-column boxes of 128 rows, or
// for d = 64 only the real 64 x 64 block per tile ([h * NT * 64 rows][64], one box)
inline int sp_map(CUtensorMap* m, void* sp, const Plan& pl, int dr) {
  if (dr == D) return make_map(m, sp, true, (unsigned long long)pl.h * pl.ntiles * D, D, 64, D, true);
  return make_map(m, sp, true, (unsigned long long)pl.h * pl.ntiles * 64, 64, 64, 64, true);
}
inline bool is_dense(const TRef& r, long long L) { return r.dr == D && r.ts == D && r.hs == L * D; }
inline bool is_dense64(const TRef& r, long long L) { return r.dr == 64 && r.ts == 64 && r.hs == L * 64; }
inline int map_act(CUtensorMap* m, const TRef& r, long long L, int heads, bool dense) {  // bf16 64x64 SW128
  if (dense) return make_map(m, r.p, true, (unsigned long long)heads * L, D, 64, T, true);
  return make_map3(m, r, true, L, heads, 64, T, true);
}
// PAIR: per-head 64 x 64 boxes over (channels, tokens, heads) maps
inline int map_act_pair(CUtensorMap* m, const TRef& r, long long L, int heads) {
  return make_map3(m, r, true, L, heads, 64, T, true);
}
inline int map_gate_pair(CUtensorMap* m, const TRef& r, long long L, int heads) {
  return make_map3(m, r, false, L, heads, 64, T, false);
}
inline int sp_map_pair(CUtensorMap* m, void* sp, const Plan& pl) {  // [2 h NT 64 rows][64], per-head blocks
  return make_map(m, sp, true, (unsigned long long)2 * pl.h * pl.ntiles * 64, 64, 64, 64, true);
}
inline int map_gate(CUtensorMap* m, const TRef& r, long long L, int heads, bool dense) {  // fp32 128x64 boxes
  if (dense) return make_map(m, r.p, false, (unsigned long long)heads * L, D, D, T, false);
  return make_map3(m, r, false, L, heads, D, T, false);
}

// tile load of (channel col, token t) of head hh: dense tensors use 2-D maps over [h * L] rows,
// strided ones 3-D maps (channels, tokens, heads)
// (the map's dimensionality is a launch argument: strided TMA inputs cost nothing measurable, unlike
// runtime strides in the pointer-addressed g loads and output stores, which select the kernel variant)
template <bool DENSE>
__device__ __forceinline__ void tile_load(void* dst, const CUtensorMap* m, uint64_t* bar, int col, int t, int hh,
                                          long long L, int in3d, uint64_t policy) {
  if (!in3d) {
    if (policy)
      tma_load_2d_hint(dst, m, bar, col, (int)(hh * L + t), policy);
    else
      tma_load_2d(dst, m, bar, col, (int)(hh * L + t));
  } else {
    if (policy)
      tma_load_3d_hint(dst, m, bar, col, t, hh, policy);
    else
      tma_load_3d(dst, m, bar, col, t, hh);
  }
}

// ---- optional pipeline tracing (diagnostics): CTA g_trace_cta records %globaltimer per (event, tile)
constexpr int TRACE_TILES = 512;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ZTRACE(buf, ev, n)                                                              \
  do {                                                                                  \
    if ((buf) != nullptr && (n) < TRACE_TILES) (buf)[(ev) * TRACE_TILES + (n)] = gtimer(); \
  } while (0)

// per-CTA lifetime (diagnostics): rows 26/27/28 of the trace buffer hold start, end and SM id by CTA
__device__ __forceinline__ void cta_trace_begin(unsigned long long* buf) {
  if (blockIdx.x < TRACE_TILES) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    buf[26 * TRACE_TILES + blockIdx.x] = gtimer();
    buf[28 * TRACE_TILES + blockIdx.x] = smid;
  }
}
__device__ __forceinline__ void cta_trace_end(unsigned long long* buf) {
  if (blockIdx.x < TRACE_TILES) buf[27 * TRACE_TILES + blockIdx.x] = gtimer();
}

// opt a kernel into large dynamic shared memory once per process (the attribute is sticky)
inline void set_smem_once(const void* fn, int bytes) {
  static const void* done[16] = {nullptr};
  for (auto& d : done) {
    if (d == fn) return;
    if (d == nullptr) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      d = fn;
      return;
    }
  }
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// ---- launches with programmatic dependent launch (PDL): a kernel's CTAs become resident as the
// previous kernel's CTAs retire and run their prologue (barrier init, TMEM alloc, descriptor
// prefetch) before griddepcontrol.wait releases them.  Every warp of every fused kernel waits before
// its first global access (unless early inputs are enabled), and a grid completes only after its own
// wait, so all memory of the kernels before it is visible.  On by default (ZGLA_PDL=0 turns it off):
// on the final kernels the CUDA-graph step is 0.3649-0.3660 -> 0.3630-0.3637 ms (round-1 kernels:
// 0.3945 -> 0.400, then it was opt-in).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ZGLA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... Exp, typename... Act>
inline cudaError_t launch_kp(bool pdl, void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}
// Early inputs (zgla_set_early_inputs): the output kernels' TMA and prep warps read q / k / v / g / dO
// before griddepcontrol.wait, so they stream under the preceding kernel (the segment scan, or the All-Scan
// chain when there are peers).  A caller contract: those tensors must be complete before the matching
// zgla_zeco_*_local call is enqueued (true for ZecoRank, the GLA layer and bench.py; not for a caller
// that writes q or dO in its own programmatic-launch kernel right before an output call).  Off by default.
int early_inputs();
template <typename... Exp, typename... Act>
inline cudaError_t launch_k(void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

// ---- device helpers
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// address of the bf16 pair (row, 2*cp .. 2*cp+1) inside a [rows x 128] SW128 tile (2 panels of
// `panel_bytes` each)
__device__ __forceinline__ uint32_t pair_off(int row, int cp, int panel_bytes) {
  return (cp >> 5) * panel_bytes + sw128(row, (cp & 31) >> 2) + (cp & 3) * 4;
}

}  // namespace fast
}  // namespace zgla
