// All-Scan (paper Alg. 2; reference glasp/collectives.py:70-140) as an in-kernel
// pipelined chain over peer memory.
//
// Every rank owns, per direction, an INBOX (one state, fp32 [h][dk][dv]), a
// FLAGS array and an ACK array ([K pipeline blocks][B CTAs] u32 each).  Rank
// p's kernel, for every pipeline block b (rows [b*dk/K, (b+1)*dk/K) of all
// heads) and for its slice of that block:
//   1. waits until FLAGS[b][cta] >= epoch (predecessor's data has landed),
//   2. computes  scanned = e^{G_p} (.) recv + local  (recv = inbox, 0 at the source),
//   3. stores scanned straight into the SUCCESSOR's inbox (NVLink P2P store
//      when the successor is another GPU) and, after a system-scope fence,
//      publishes FLAGS[b][cta] = epoch in the successor's memory,
//   4. acks consumption of its own inbox block to the predecessor.
// A producer only overwrites a successor inbox block once that block's ACK
// from the previous epoch has arrived, so back-to-back calls are safe.  Blocks
// pipeline exactly as in the reference: rank p forwards block b while block
// b+1 is still in flight, giving the (K+P-1) hop schedule of Eq. 13.
//
// The same device code runs the reference's list form (all P ranks resident on
// one GPU, zgla_allscan_local / zgla_allscan_bind_local) and the SPMD form
// (one process per GPU, peers mapped with CUDA IPC).  Results are elementwise
// and independent of K and of the CTA split, so they are bit-identical for
// every K (reference tests/test_collectives.py:88-103).
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "zgla_internal.h"

namespace zgla {
namespace allscan {

constexpr int kThreads = 256;
constexpr int kCtasPerRank = 8;

template <typename T>
struct Link {
  const T* local;
  const T* logdecay;
  const T* inbox;         // my incoming buffer (nullptr at the source)
  const unsigned* flags;  // my incoming flags
  unsigned* ack_to_pred;  // predecessor's ACK array (peer), nullptr at the source
  T* succ_inbox;          // successor's inbox (peer), nullptr at the sink
  unsigned* succ_flags;   // successor's flags (peer)
  const unsigned* my_ack; // ACKs written by my successor
  T* recv_out;
  T* scanned_out;
};

template <typename T>
struct V4 {
  T x, y, z, w;
};
__device__ __forceinline__ V4<float> ldcg4(const V4<float>* p) {
  const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
  return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ V4<double> ldcg4(const V4<double>* p) {
  const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ float scan_update(float gl, float r, float x) {
  return __fadd_rn(__fmul_rn(expf(gl), r), x);
}
__device__ __forceinline__ double scan_update(double gl, double r, double x) {
  return __dadd_rn(__dmul_rn(exp(gl), r), x);
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool SYS>
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  if (SYS) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <bool SYS>
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  if (SYS) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <bool SYS>
__device__ __forceinline__ void fence_acq_rel() {
  if (SYS) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// poll with relaxed loads; one acquire fence once the value is seen (bar.sync then publishes it to the CTA)
template <bool SYS>
__device__ __forceinline__ bool spin_until_geq(const unsigned* p, unsigned target) {
  long long t0 = clock64();
  while ((int)(ld_relaxed<SYS>(p) - target) < 0) {
    if (clock64() - t0 > (1ll << 34)) return false;  // ~8 s at 2 GHz: treat as deadlock
  }
  fence_acq_rel<SYS>();
  return true;
}

// one CTA's share of the chain for one rank
template <typename T, bool SYS>
__device__ void rank_body(const Link<T>& L, int h, int dk, int dv, int K, int cta, int nctas, unsigned epoch,
                          int* err) {
  const int rows = dk / K;
  const int blk_el = rows * dv;          // elements of one head inside one pipeline block
  const bool vec4 = (dv % 4) == 0;
  int per_cta = (blk_el + nctas - 1) / nctas;
  if (vec4) per_cta = (per_cta + 3) & ~3;
  const int lo = min(blk_el, cta * per_cta), hi = min(blk_el, lo + per_cta);
  __shared__ int ok;
  // back-pressure: my slice of the successor's inbox may only be overwritten once the successor has
  // consumed it in the previous epoch (one ACK per CTA slice, independent of the block count K)
  if (threadIdx.x == 0 && L.succ_inbox && !spin_until_geq<SYS>(L.my_ack + cta, epoch - 1)) {
    atomicExch(err, 1);
    printf("zgla all-scan: ack wait timed out (deadlock)\n");
    __trap();
  }
  for (int b = 0; b < K; ++b) {
    const int fidx = b * nctas + cta;
    if (threadIdx.x == 0) {
      bool good = true;
      if (L.inbox) good = spin_until_geq<SYS>(L.flags + fidx, epoch);
      ok = good;
      if (!good) {
        atomicExch(err, 1);
        printf("zgla all-scan: flag wait timed out (deadlock), block %d\n", b);
        __trap();
      }
    }
    __syncthreads();
    if (!ok) return;
    if (vec4) {
      // float4 path: all loads of a batch are issued before any use (latency-bound otherwise)
      const int lo4 = lo >> 2, n4 = (hi - lo) >> 2, blk4 = blk_el >> 2;
      const int total = h * n4;
      for (int u0 = threadIdx.x; u0 < total; u0 += 4 * blockDim.x) {
        V4<T> r[4], x[4];
        T gl[4];
        long long e4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int u = u0 + k * blockDim.x;
          const int hh = u / max(n4, 1), i4 = lo4 + u % max(n4, 1);
          e4[k] = ((long long)hh * dk * dv + (long long)b * blk_el) / 4 + i4;
          if (u < total) {
            const int c = b * rows + (i4 * 4) / dv;
            gl[k] = L.logdecay[hh * dk + c];
            x[k] = reinterpret_cast<const V4<T>*>(L.local)[e4[k]];
            r[k] = L.inbox ? ldcg4(reinterpret_cast<const V4<T>*>(L.inbox) + e4[k]) : V4<T>{0, 0, 0, 0};
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (u0 + k * blockDim.x >= total) break;
          V4<T> sc;
          sc.x = scan_update(gl[k], r[k].x, x[k].x);
          sc.y = scan_update(gl[k], r[k].y, x[k].y);
          sc.z = scan_update(gl[k], r[k].z, x[k].z);
          sc.w = scan_update(gl[k], r[k].w, x[k].w);
          if (L.recv_out) reinterpret_cast<V4<T>*>(L.recv_out)[e4[k]] = r[k];
          reinterpret_cast<V4<T>*>(L.scanned_out)[e4[k]] = sc;
          if (L.succ_inbox) reinterpret_cast<V4<T>*>(L.succ_inbox)[e4[k]] = sc;
        }
      }
      (void)blk4;
    } else {
      for (int hh = 0; hh < h; ++hh) {
        const long long base = (long long)hh * dk * dv + (long long)b * blk_el;
        for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
          const long long e = base + i;
          const int c = b * rows + i / dv;
          const T r = L.inbox ? ldcg(L.inbox + e) : T(0);
          // same rounding sequence as the reference update (gate * recv, then + local)
          const T s = scan_update(L.logdecay[hh * dk + c], r, L.local[e]);
          if (L.recv_out) L.recv_out[e] = r;
          L.scanned_out[e] = s;
          if (L.succ_inbox) L.succ_inbox[e] = s;
        }
      }
    }
    __syncthreads();
    // release at system scope is cumulative over the CTA's stores observed through bar.sync
    if (threadIdx.x == 0 && L.succ_inbox) st_release<SYS>(L.succ_flags + fidx, epoch);
  }
  if (threadIdx.x == 0 && L.ack_to_pred) st_release<SYS>(L.ack_to_pred + cta, epoch);
}

// list form: P ranks on one device, recv[p] doubles as rank p's inbox
template <typename T>
__global__ void __launch_bounds__(kThreads) local_chain_kernel(int P, int h, int dk, int dv, int K, int dir,
                                                               const T* local, const T* logdecay, T* recv,
                                                               T* scanned, unsigned* flags, int* err) {
  const int pos = blockIdx.x / kCtasPerRank, cta = blockIdx.x % kCtasPerRank;
  const int rank = dir == ZGLA_FWD ? pos : P - 1 - pos;
  const long long nel = (long long)h * dk * dv;
  const int succ = dir == ZGLA_FWD ? rank + 1 : rank - 1;
  const int fl = K * kCtasPerRank;
  Link<T> L;
  L.local = local + rank * nel;
  L.logdecay = logdecay + (long long)rank * h * dk;
  L.inbox = pos == 0 ? nullptr : recv + rank * nel;
  L.flags = flags + (long long)rank * fl;
  L.ack_to_pred = nullptr;
  L.succ_inbox = pos == P - 1 ? nullptr : recv + (long long)succ * nel;
  L.succ_flags = pos == P - 1 ? nullptr : flags + (long long)succ * fl;
  L.my_ack = nullptr;
  L.recv_out = pos == 0 ? recv + rank * nel : nullptr;  // source writes its zero recv
  L.scanned_out = scanned + rank * nel;
  if (L.succ_inbox) {
    // no ACK protocol needed: flags are cleared before every list-form call
    L.my_ack = flags + (long long)P * fl;  // all-zero dummy; epoch-1 == 0 passes
  }
  rank_body<T, false>(L, h, dk, dv, K, cta, kCtasPerRank, 1u, err);  // one device: gpu scope
}

// SPMD form: one rank per process
// The epoch lives in device memory (ctl[0]) so that a captured CUDA graph replays correctly: every
// CTA reads the completed-call count at entry (the previous call on this stream has finished), and the
// last CTA to leave publishes the new count (ctl[1] counts departures).
__global__ void __launch_bounds__(kThreads) rank_chain_kernel(Link<float> L, int h, int dk, int dv, int K,
                                                              unsigned* ctl, int* err) {
  const unsigned epoch = *reinterpret_cast<volatile unsigned*>(ctl) + 1;
  rank_body<float, true>(L, h, dk, dv, K, blockIdx.x, gridDim.x, epoch, err);  // peers: system scope
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctl + 1, 1u) == gridDim.x - 1) {
      ctl[1] = 0;
      *reinterpret_cast<volatile unsigned*>(ctl) = epoch;
    }
  }
}

// list-form workspace (flags + error word), grown on demand
struct Scratch {
  std::mutex mu;
  unsigned* flags = nullptr;
  size_t bytes = 0;
};
static Scratch g_scratch;

}  // namespace allscan
}  // namespace zgla

using namespace zgla;
using namespace zgla::allscan;

extern "C" int zgla_allscan_local(int P, int heads, int key_dim, int value_dim, int dtype, int num_blocks,
                                  int direction, const void* local_states, const void* log_decays, void* recv,
                                  void* scanned, void* stream) {
  if (P < 1 || heads < 1 || key_dim < 1 || value_dim < 1) return ZGLA_ERR_DIMS;
  if (num_blocks < 1 || key_dim % num_blocks) return ZGLA_ERR_CONFIG;
  if (direction != ZGLA_FWD && direction != ZGLA_BWD) return ZGLA_ERR_CONFIG;
  if (dtype != ZGLA_F32 && dtype != ZGLA_F64) return ZGLA_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t fl = (size_t)num_blocks * kCtasPerRank;
  const size_t need = ((size_t)(P + 1) * fl + 1) * sizeof(unsigned);
  std::lock_guard<std::mutex> lock(g_scratch.mu);
  if (g_scratch.bytes < need) {
    if (g_scratch.flags) cudaFree(g_scratch.flags);
    g_scratch.flags = nullptr;
    g_scratch.bytes = 0;
    if (cudaError_t e = cudaMalloc(&g_scratch.flags, need)) return cuda_fail(e, "zgla_allscan_local");
    g_scratch.bytes = need;
  }
  if (cudaError_t e = cudaMemsetAsync(g_scratch.flags, 0, need, st)) return cuda_fail(e, "zgla_allscan_local");
  int* err = reinterpret_cast<int*>(g_scratch.flags + (P + 1) * fl);
  if (dtype == ZGLA_F64)
    local_chain_kernel<double><<<P * kCtasPerRank, kThreads, 0, st>>>(
        P, heads, key_dim, value_dim, num_blocks, direction, (const double*)local_states, (const double*)log_decays,
        (double*)recv, (double*)scanned, g_scratch.flags, err);
  else
    local_chain_kernel<float><<<P * kCtasPerRank, kThreads, 0, st>>>(
        P, heads, key_dim, value_dim, num_blocks, direction, (const float*)local_states, (const float*)log_decays,
        (float*)recv, (float*)scanned, g_scratch.flags, err);
  return zgla_check_launch();
}

extern "C" int zgla_release_cached(void) {
  std::lock_guard<std::mutex> lock(g_scratch.mu);
  if (g_scratch.flags) {
    cudaError_t e = cudaFree(g_scratch.flags);
    g_scratch.flags = nullptr;
    g_scratch.bytes = 0;
    if (e != cudaSuccess) return cuda_fail(e, "zgla_release_cached");
  }
  return ZGLA_OK;
}

// ------------------------------------------------------------------ SPMD comm
struct zgla_allscan_comm {
  int rank, world, h, dk, dv, max_blocks;
  long long nel;
  size_t region_bytes;
  unsigned char* region;  // [dir][inbox | flags | ack]
  unsigned char* next_region;
  unsigned char* prev_region;
  bool next_ipc, prev_ipc;
  int* err;  // [0] deadlock flag; [2 + 2 d], [3 + 2 d]: per-direction device epoch and departure count
  long long bytes_sent;
};

static size_t dir_bytes(const zgla_allscan_comm* c) {
  const size_t fl = (size_t)c->max_blocks * kCtasPerRank * sizeof(unsigned);
  size_t inbox = (size_t)c->nel * sizeof(float);
  inbox = (inbox + 255) & ~size_t(255);
  return inbox + 2 * fl;
}
static float* inbox_of(const zgla_allscan_comm* c, unsigned char* region, int dir) {
  return reinterpret_cast<float*>(region + dir * dir_bytes(c));
}
static unsigned* flags_of(const zgla_allscan_comm* c, unsigned char* region, int dir) {
  size_t inbox = ((size_t)c->nel * sizeof(float) + 255) & ~size_t(255);
  return reinterpret_cast<unsigned*>(region + dir * dir_bytes(c) + inbox);
}
static unsigned* ack_of(const zgla_allscan_comm* c, unsigned char* region, int dir) {
  return flags_of(c, region, dir) + (size_t)c->max_blocks * kCtasPerRank;
}

extern "C" int zgla_allscan_create(int rank, int world, int heads, int key_dim, int value_dim, int max_blocks,
                                   zgla_allscan_comm** out) {
  if (!out || world < 1 || rank < 0 || rank >= world || heads < 1 || key_dim < 1 || value_dim < 1 ||
      max_blocks < 1)
    return ZGLA_ERR_DIMS;
  auto* c = new zgla_allscan_comm();
  c->rank = rank;
  c->world = world;
  c->h = heads;
  c->dk = key_dim;
  c->dv = value_dim;
  c->max_blocks = max_blocks;
  c->nel = (long long)heads * key_dim * value_dim;
  c->region_bytes = 2 * dir_bytes(c);
  c->bytes_sent = 0;
  c->next_region = c->prev_region = nullptr;
  c->next_ipc = c->prev_ipc = false;
  if (cudaError_t e = cudaMalloc(&c->region, c->region_bytes)) {
    delete c;
    return cuda_fail(e, "zgla_allscan_create");
  }
  cudaMemset(c->region, 0, c->region_bytes);
  if (cudaError_t e = cudaMalloc(&c->err, 8 * sizeof(int))) {
    cudaFree(c->region);
    delete c;
    return cuda_fail(e, "zgla_allscan_create");
  }
  cudaMemset(c->err, 0, 8 * sizeof(int));
  if (cudaError_t e = cudaDeviceSynchronize()) return cuda_fail(e, "zgla_allscan_create");
  *out = c;
  return ZGLA_OK;
}

extern "C" int zgla_allscan_export(zgla_allscan_comm* c, void* ipc_handle_out) {
  if (!c || !ipc_handle_out) return ZGLA_ERR_DIMS;
  cudaIpcMemHandle_t h;
  if (cudaError_t e = cudaIpcGetMemHandle(&h, c->region)) return cuda_fail(e, "zgla_allscan_export");
  std::memcpy(ipc_handle_out, &h, sizeof(h));
  return ZGLA_OK;
}

extern "C" int zgla_allscan_bind(zgla_allscan_comm* c, const void* next_handle, const void* prev_handle) {
  if (!c) return ZGLA_ERR_DIMS;
  if (next_handle && c->rank + 1 < c->world) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, next_handle, sizeof(h));
    void* p = nullptr;
    if (cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess))
      return cuda_fail(e, "zgla_allscan_bind(next)");
    c->next_region = (unsigned char*)p;
    c->next_ipc = true;
  }
  if (prev_handle && c->rank > 0) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, prev_handle, sizeof(h));
    void* p = nullptr;
    if (cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess))
      return cuda_fail(e, "zgla_allscan_bind(prev)");
    c->prev_region = (unsigned char*)p;
    c->prev_ipc = true;
  }
  return ZGLA_OK;
}

extern "C" int zgla_allscan_bind_local(zgla_allscan_comm* c, zgla_allscan_comm* next, zgla_allscan_comm* prev) {
  if (!c) return ZGLA_ERR_DIMS;
  c->next_region = next ? next->region : nullptr;
  c->prev_region = prev ? prev->region : nullptr;
  return ZGLA_OK;
}

extern "C" int zgla_allscan_run(zgla_allscan_comm* c, int num_blocks, int direction, const float* local_state,
                                const float* log_decay, float* recv, float* scanned, void* stream) {
  if (!c || !local_state || !log_decay || !scanned) return ZGLA_ERR_DIMS;
  if (num_blocks < 1 || num_blocks > c->max_blocks || c->dk % num_blocks) return ZGLA_ERR_CONFIG;
  if (direction != ZGLA_FWD && direction != ZGLA_BWD) return ZGLA_ERR_CONFIG;
  cudaStream_t st = (cudaStream_t)stream;
  const int d = direction;
  // chain order: FWD 0 -> P-1, BWD P-1 -> 0
  const bool is_source = d == ZGLA_FWD ? c->rank == 0 : c->rank == c->world - 1;
  const bool is_sink = d == ZGLA_FWD ? c->rank == c->world - 1 : c->rank == 0;
  unsigned char* succ = d == ZGLA_FWD ? c->next_region : c->prev_region;
  unsigned char* pred = d == ZGLA_FWD ? c->prev_region : c->next_region;
  if ((!is_sink && !succ) || (!is_source && !pred)) return ZGLA_ERR_STATE;  // not bound
  Link<float> L;
  L.local = local_state;
  L.logdecay = log_decay;
  L.inbox = is_source ? nullptr : inbox_of(c, c->region, d);
  L.flags = flags_of(c, c->region, d);
  L.ack_to_pred = is_source ? nullptr : ack_of(c, pred, d);
  L.succ_inbox = is_sink ? nullptr : inbox_of(c, succ, d);
  L.succ_flags = is_sink ? nullptr : flags_of(c, succ, d);
  L.my_ack = ack_of(c, c->region, d);
  // recv is written by the chain kernel itself (zeros at the source), before the inbox is acked: a
  // predecessor running ahead into the next epoch can never overwrite data not yet copied out
  L.recv_out = recv;
  L.scanned_out = scanned;
  if (c->world == 1) L.inbox = nullptr;
  unsigned* ctl = reinterpret_cast<unsigned*>(c->err) + 2 + 2 * d;
  rank_chain_kernel<<<kCtasPerRank, kThreads, 0, st>>>(L, c->h, c->dk, c->dv, num_blocks, ctl, c->err);
  if (int rc = zgla_check_launch()) return rc;
  if (!is_sink) c->bytes_sent += c->nel * (long long)sizeof(float);
  return zgla_check_launch();
}

extern "C" int zgla_allscan_info(const zgla_allscan_comm* c, int* rank, int* world, int* heads) {
  if (!c) return ZGLA_ERR_DIMS;
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (heads) *heads = c->h;
  return ZGLA_OK;
}

extern "C" long long zgla_allscan_bytes_sent(const zgla_allscan_comm* c) { return c ? c->bytes_sent : -1; }

extern "C" int zgla_allscan_destroy(zgla_allscan_comm* c) {
  if (!c) return ZGLA_OK;
  cudaDeviceSynchronize();
  if (c->next_ipc && c->next_region) cudaIpcCloseMemHandle(c->next_region);
  if (c->prev_ipc && c->prev_region) cudaIpcCloseMemHandle(c->prev_region);
  cudaFree(c->region);
  cudaFree(c->err);
  delete c;
  return ZGLA_OK;
}
