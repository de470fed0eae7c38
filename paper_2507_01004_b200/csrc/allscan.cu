// All-Scan (paper Alg. 2; reference glasp/collectives.py:70-140) as an in-kernel
// pipelined chain over peer memory, with a low-latency (LL) data+flag protocol.
//
// Every word that travels between two ranks is 16 bytes {data, flag, data, flag}:
// each 8-byte half is written atomically by one vector store, so a receiver that
// sees flag == epoch in both halves also sees the data next to it.  There is no
// separate flag store, no fence and no per-block barrier on the data path: every
// thread of rank p polls its own inbox words, computes
//     scanned = e^{G_p} (.) recv + local          (recv = 0 at the chain source)
// and stores the result (with the epoch in both flag slots) straight into the
// successor's inbox (an NVLink P2P store when the successor is another GPU).
// The reference's K pipeline blocks (rows [b*dk/K, (b+1)*dk/K) of every head) set
// the ORDER in which a CTA forwards its words, so block 0 of every CTA leaves
// first; with LL the pipeline is per word, which is the limit of Eq. 13's
// (K + P - 1) hop schedule as K grows.  Results are elementwise, so they are
// bit-identical for every K and every CTA split (tests/test_collectives.py:88-103).
//
// Inboxes are double-buffered by epoch parity, so a producer only has to know that
// its successor finished the call TWO epochs back before it overwrites a buffer:
// one ACK word per direction, published by the successor's last departing CTA, and
// checked once per CTA at entry (never on the critical path in steady state).
//
// A wait that does not complete within the communicator's timeout sets an error
// word in host-mapped memory and the kernel exits (no trap): the CUDA context
// stays usable and the next zgla_allscan_run / zgla_allscan_status returns
// ZGLA_ERR_DEADLOCK (-> DeadlockError, glasp/errors.py).
//
// The same device code runs the reference's list form (all P ranks resident on one
// GPU, zgla_allscan_local) and the SPMD form (one process per GPU, peers mapped with
// CUDA IPC, or in-process ranks bound with zgla_allscan_bind_local).
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "zgla_internal.h"

namespace zgla {
namespace allscan {

constexpr int kThreads = 128;       // light CTAs: they co-reside with the fused kernels (PDL overlap)
constexpr int kMaxCtas = 256;       // per rank (SPMD); the list form caps P x CTAs at kMaxListCtas
#ifndef ZGLA_AS_LIST_CAP
#define ZGLA_AS_LIST_CAP 1024
#endif
#ifndef ZGLA_AS_WPT
#define ZGLA_AS_WPT 4
#endif
constexpr int kMaxListCtas = ZGLA_AS_LIST_CAP;
constexpr int kWordsPerThread = ZGLA_AS_WPT;  // CTA count: ~this many 16-byte words per thread and call (list form;
                                    // the SPMD form uses half, it has a GPU to itself)
#ifndef ZGLA_AS_BATCH
#define ZGLA_AS_BATCH 1
#endif
// Words a thread has in flight per step.  Measured (virtual ranks, P = 8, 1 MiB, graph-timed): 1 word
// 14.0 us, 2: 16.3, 4: 18.4, 8: 24.4 -- every strong (volatile) store of a batch sits between a word's
// arrival and its departure, so small batches forward sooner; the loads of the next step are the cost.
constexpr int kBatchList = ZGLA_AS_BATCH;  // list form
constexpr int kBatchRank = ZGLA_AS_BATCH;  // SPMD form (<= 64 registers: a CTA fits beside a fused-kernel CTA)

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// LL word accesses: volatile (relaxed.sys / relaxed.gpu / weak stores measured the same)
__device__ __forceinline__ uint4 ld_volatile4(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile4(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// scanned = e^{G} * recv + local with the reference's rounding sequence (multiply, then add; no FMA)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
// EPW consecutive elements of word f (one vector store when EPW = 2)
template <typename T, int EPW>
__device__ __forceinline__ void store_el(T* p, int f, const T (&v)[EPW]) {
  if (p == nullptr) return;
  if constexpr (EPW == 2 && sizeof(T) == 4) {
    *reinterpret_cast<float2*>(p + 2 * f) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int k = 0; k < EPW; ++k) p[f * EPW + k] = v[k];
  }
}

// element <-> LL word.  fp32: EPW = 2 elements per word {d0, f, d1, f}, or 1 ({d0, f, 0, f}) when a
// head's block length is odd; fp64: EPW = 1, the two 32-bit halves of the value in the two data slots.
template <typename T, int EPW>
struct Word;
template <int EPW>
struct Word<float, EPW> {
  __device__ static uint4 pack(const float (&s)[EPW], unsigned f) {
    return make_uint4(__float_as_uint(s[0]), f, EPW == 2 ? __float_as_uint(s[EPW - 1]) : 0u, f);
  }
  __device__ static void unpack(uint4 w, float (&r)[EPW]) {
    r[0] = __uint_as_float(w.x);
    if (EPW == 2) r[EPW - 1] = __uint_as_float(w.z);
  }
};
template <>
struct Word<double, 1> {
  __device__ static uint4 pack(const double (&s)[1], unsigned f) {
    return make_uint4((unsigned)__double2loint(s[0]), f, (unsigned)__double2hiint(s[0]), f);
  }
  __device__ static void unpack(uint4 w, double (&r)[1]) { r[0] = __hiloint2double((int)w.z, (int)w.x); }
};

template <typename T>
struct Chain {
  const T* local;
  const T* logdecay;
  const uint4* inbox;  // my incoming words (this epoch's parity buffer); nullptr at the source
  uint4* succ_inbox;   // successor's incoming words (peer memory); nullptr at the sink
  T* recv_out;
  T* scanned_out;
};

// one CTA's share of one rank's chain; false if a wait timed out.  With LL words the pipeline is per
// word: a word leaves as soon as its predecessor word has arrived, which is the fine-grained limit of
// the reference's K-block pipelining (glasp/collectives.py:96-131), so K does not change the schedule
// (nor, the update being elementwise, a single bit of the result).  CTA `cta` owns the contiguous word
// range [lo, hi) in element order; a thread's kBatch words are all in flight at once.
template <typename T, int EPW, int kBatch>
__device__ bool chain_slice(const Chain<T>& A, int nwords, int dv, int cta, int nctas, unsigned epoch,
                            unsigned long long deadline, unsigned long long* tr = nullptr) {
  const int per = (nwords + nctas - 1) / nctas;
  const int lo = min(nwords, cta * per), hi = min(nwords, lo + per);
  for (int f0 = lo + threadIdx.x; f0 < hi; f0 += kBatch * blockDim.x) {
    uint4 w[kBatch];
    T x[kBatch][EPW], eg[kBatch][EPW];
    // everything that does not depend on the predecessor first: the inbox loads, the local state and
    // e^{G} (so that only one multiply-add and the stores sit between arrival and departure of a word)
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int f = f0 + j * blockDim.x;
      w[j] = make_uint4(0, epoch, 0, epoch);
      if (f < hi) {
        if (A.inbox) w[j] = ld_volatile4(A.inbox + f);
#pragma unroll
        for (int k = 0; k < EPW; ++k) {
          const int e = f * EPW + k;
          eg[j][k] = A.logdecay[e / dv];  // [h][dk] decay of state row (head, channel) = e / dv
          x[j][k] = A.local[e];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j)
#pragma unroll
      for (int k = 0; k < EPW; ++k) eg[j][k] = ex(eg[j][k]);
    if (A.inbox) {  // poll until every word of the batch carries this epoch in both halves
      unsigned spins = 0;
      for (;;) {
        bool pending = false;
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
          if (w[j].y != epoch || w[j].w != epoch) {
            pending = true;
            w[j] = ld_volatile4(A.inbox + f0 + j * blockDim.x);
          }
        }
        if (!pending) break;
        if ((++spins & 1023u) == 0 && gtimer() > deadline) return false;
      }
    }
    if (tr != nullptr && threadIdx.x == 0 && f0 == lo) tr[1] = gtimer();
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int f = f0 + j * (int)blockDim.x;
      if (f >= hi) break;
      T r[EPW], sc[EPW];
      if (A.inbox) {
        Word<T, EPW>::unpack(w[j], r);
      } else {
#pragma unroll
        for (int k = 0; k < EPW; ++k) r[k] = T(0);
      }
#pragma unroll
      for (int k = 0; k < EPW; ++k) sc[k] = add_rn(mul_rn(eg[j][k], r[k]), x[j][k]);  // reference rounding
      if (A.succ_inbox) st_volatile4(A.succ_inbox + f, Word<T, EPW>::pack(sc, epoch));
      store_el<T, EPW>(A.recv_out, f, r);
      store_el<T, EPW>(A.scanned_out, f, sc);
    }
    if (tr != nullptr && threadIdx.x == 0 && f0 == lo) tr[2] = gtimer();
  }
  return true;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// last CTA to leave publishes the completed-call count (and, in the SPMD form, the ACK to the
// predecessor: a release at system scope, cumulative over the inbox reads of every CTA observed through
// the bar.sync / departure-counter chain).  The data path itself needs no fence: LL words carry their flag.
__device__ __forceinline__ void depart(unsigned* ctl, unsigned epoch, unsigned* pred_ack) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctl + 1, 1u) == gridDim.x - 1) {
      __threadfence();
      ctl[1] = 0;
      if (pred_ack) st_release_sys(pred_ack, epoch);
      *reinterpret_cast<volatile unsigned*>(ctl) = epoch;
    }
  }
}

// list form: P ranks on one device, one kernel; rank r's inbox is inbox + r * nwords.  The epoch is a
// call counter kept in device memory; inbox words of earlier calls carry older epochs, so no reset
// pass is needed between calls.
template <typename T, int EPW>
__global__ void __launch_bounds__(kThreads) local_chain_kernel(int P, int h, int dk, int dv, int K, int dir,
                                                               int nctas, const T* local, const T* logdecay,
                                                               T* recv, T* scanned, uint4* inbox,
                                                               long long nwords, unsigned* ctl, int* err,
                                                               unsigned long long timeout_ns,
                                                               unsigned long long* trace) {
  unsigned long long* tr = trace ? trace + 4 * blockIdx.x : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();
  const unsigned epoch = *reinterpret_cast<volatile unsigned*>(ctl) + 1;
  const int pos = blockIdx.x / nctas, cta = blockIdx.x % nctas;
  const int rank = dir == ZGLA_FWD ? pos : P - 1 - pos;
  const int succ = dir == ZGLA_FWD ? rank + 1 : rank - 1;
  const long long nel = (long long)h * dk * dv;  // (< 2^31: states are at most a few MiB)
  Chain<T> A;
  A.local = local + rank * nel;
  A.logdecay = logdecay + (long long)rank * h * dk;
  A.inbox = pos == 0 ? nullptr : inbox + rank * nwords;
  A.succ_inbox = pos == P - 1 ? nullptr : inbox + (long long)succ * nwords;
  A.recv_out = recv + rank * nel;
  A.scanned_out = scanned + rank * nel;
  const unsigned long long deadline = gtimer() + timeout_ns;
  if (!chain_slice<T, EPW, kBatchList>(A, (int)(nel / EPW), dv, cta, nctas, epoch, deadline, tr))
    atomicExch(err, ZGLA_ERR_DEADLOCK);
  depart(ctl, epoch, nullptr);
  if (tr && threadIdx.x == 0) tr[3] = gtimer();
}

// SPMD form: one rank per process.  ctl = {completed calls, departures} of this direction in device
// memory (a captured CUDA graph replays correctly); my_ack is written by the successor.
__global__ void __launch_bounds__(kThreads, 8) rank_chain_kernel(Chain<float> A, int h, int dk, int dv, int K,
                                                                 int epw, const uint4* inbox2, uint4* succ_inbox2,
                                                                 long long nwords, unsigned* ctl,
                                                                 const unsigned* my_ack, unsigned* pred_ack,
                                                                 int* err, unsigned long long timeout_ns) {
  pdl_wait();  // the local state comes from the kernel before (programmatic launch)
  pdl_trigger();
  const unsigned epoch = *reinterpret_cast<volatile unsigned*>(ctl) + 1;
  const unsigned long long deadline = gtimer() + timeout_ns;
  const int par = epoch & 1;
  A.inbox = inbox2 ? inbox2 + par * nwords : nullptr;
  A.succ_inbox = succ_inbox2 ? succ_inbox2 + par * nwords : nullptr;
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 1;
    // the successor must have consumed the buffer of this parity (epoch - 2) before it is overwritten
    if (A.succ_inbox && epoch > 2) {
      unsigned spins = 0;
      while ((int)(ld_acquire_sys(my_ack) - (epoch - 2)) < 0) {
        if ((++spins & 255u) == 0 && gtimer() > deadline) {
          ok = 0;
          break;
        }
      }
    }
  }
  __syncthreads();
  bool good = ok != 0;
  if (good) {
    const int nw = (int)((long long)h * dk * dv / epw);
    good = epw == 2 ? chain_slice<float, 2, kBatchRank>(A, nw, dv, blockIdx.x, gridDim.x, epoch, deadline)
                    : chain_slice<float, 1, kBatchRank>(A, nw, dv, blockIdx.x, gridDim.x, epoch, deadline);
  }
  if (!good) atomicExch(err, ZGLA_ERR_DEADLOCK);
  depart(ctl, epoch, pred_ack);
}

inline int epw_for(int dv, bool f64) { return (f64 || dv % 2) ? 1 : 2; }  // a word never straddles a row
inline int ctas_for(long long nwords, int cap = kMaxCtas, int wpt = kWordsPerThread / 2) {
  long long n = (nwords + (long long)kThreads * wpt - 1) / ((long long)kThreads * wpt);
  return (int)std::max(1ll, std::min((long long)cap, n));
}
inline unsigned long long timeout_ns_default() {
  static const unsigned long long t = [] {
    const char* e = std::getenv("ZGLA_ALLSCAN_TIMEOUT_MS");
    const long long ms = e ? std::atoll(e) : 10000;
    return (unsigned long long)(ms > 0 ? ms : 10000) * 1000000ull;
  }();
  return t;
}

// host-mapped error word: the kernel reports a timed-out wait without trapping, the host reads it
// without a device synchronisation
struct MappedErr {
  int* host = nullptr;
  int* dev = nullptr;
  int alloc() {
    if (host) return ZGLA_OK;
    if (cudaError_t e = cudaHostAlloc(&host, 64, cudaHostAllocMapped)) return cuda_fail(e, "cudaHostAlloc");
    std::memset(host, 0, 64);
    if (cudaError_t e = cudaHostGetDevicePointer(&dev, host, 0)) return cuda_fail(e, "cudaHostGetDevicePointer");
    return ZGLA_OK;
  }
  void release() {
    if (host) cudaFreeHost(host);
    host = dev = nullptr;
  }
};

// list-form workspace (inboxes + control words), grown on demand
struct Scratch {
  std::mutex mu;
  unsigned char* base = nullptr;
  size_t bytes = 0;
  MappedErr err;
};
static Scratch g_scratch;

}  // namespace allscan
}  // namespace zgla

using namespace zgla;
using namespace zgla::allscan;

template <typename... Exp, typename... Act>
static cudaError_t launch_ex(bool pdl, void (*kern)(Exp...), int grid, int block, cudaStream_t st, Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

static bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("ZGLA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

extern "C" int zgla_allscan_local(int P, int heads, int key_dim, int value_dim, int dtype, int num_blocks,
                                  int direction, const void* local_states, const void* log_decays, void* recv,
                                  void* scanned, void* stream) {
  if (P < 1 || heads < 1 || key_dim < 1 || value_dim < 1) return ZGLA_ERR_DIMS;
  if (num_blocks < 1 || key_dim % num_blocks) return ZGLA_ERR_CONFIG;
  if (direction != ZGLA_FWD && direction != ZGLA_BWD) return ZGLA_ERR_CONFIG;
  if (dtype != ZGLA_F32 && dtype != ZGLA_F64) return ZGLA_ERR_UNSUPPORTED;
  if (!local_states || !log_decays || !recv || !scanned) return ZGLA_ERR_DIMS;
  cudaStream_t st = (cudaStream_t)stream;
  const bool f64 = dtype == ZGLA_F64;
  const int epw = epw_for(value_dim, f64);
  const long long nel = (long long)heads * key_dim * value_dim;
  const long long nwords = nel / epw;
  const int nctas = ctas_for(nwords, std::max(1, kMaxListCtas / P), kWordsPerThread);
  const size_t need = 256 + (size_t)P * nwords * sizeof(uint4);
  std::lock_guard<std::mutex> lock(g_scratch.mu);
  if (int rc = g_scratch.err.alloc()) return rc;
  if (*reinterpret_cast<volatile int*>(g_scratch.err.host)) {
    g_scratch.err.host[0] = 0;
    set_error("a previous zgla_allscan_local call timed out waiting for its predecessor");
    return ZGLA_ERR_DEADLOCK;
  }
  if (g_scratch.bytes < need) {
    if (g_scratch.base) {
      cudaStreamSynchronize(st);
      cudaFree(g_scratch.base);
    }
    g_scratch.base = nullptr;
    g_scratch.bytes = 0;
    if (cudaError_t e = cudaMalloc(&g_scratch.base, need)) return cuda_fail(e, "zgla_allscan_local");
    // zero flags never match an epoch (>= 1); the call counter starts at 0
    if (cudaError_t e = cudaMemsetAsync(g_scratch.base, 0, need, st)) return cuda_fail(e, "zgla_allscan_local");
    g_scratch.bytes = need;
  }
  unsigned* ctl = reinterpret_cast<unsigned*>(g_scratch.base);
  uint4* inbox = reinterpret_cast<uint4*>(g_scratch.base + 256);
  const unsigned long long to = timeout_ns_default();
  cudaError_t e;
  if (f64)
    e = launch_ex(false, local_chain_kernel<double, 1>, P * nctas, kThreads, st, P, heads, key_dim, value_dim,
                  num_blocks, direction, nctas, (const double*)local_states, (const double*)log_decays,
                  (double*)recv, (double*)scanned, inbox, nwords, ctl, g_scratch.err.dev, to, g_trace_buf);
  else if (epw == 2)
    e = launch_ex(false, local_chain_kernel<float, 2>, P * nctas, kThreads, st, P, heads, key_dim, value_dim,
                  num_blocks, direction, nctas, (const float*)local_states, (const float*)log_decays, (float*)recv,
                  (float*)scanned, inbox, nwords, ctl, g_scratch.err.dev, to, g_trace_buf);
  else
    e = launch_ex(false, local_chain_kernel<float, 1>, P * nctas, kThreads, st, P, heads, key_dim, value_dim,
                  num_blocks, direction, nctas, (const float*)local_states, (const float*)log_decays, (float*)recv,
                  (float*)scanned, inbox, nwords, ctl, g_scratch.err.dev, to, g_trace_buf);
  if (e != cudaSuccess) return cuda_fail(e, "local_chain_kernel");
  return zgla_check_launch();
}

extern "C" int zgla_release_cached(void) {
  std::lock_guard<std::mutex> lock(g_scratch.mu);
  if (g_scratch.base) {
    cudaError_t e = cudaFree(g_scratch.base);
    g_scratch.base = nullptr;
    g_scratch.bytes = 0;
    if (e != cudaSuccess) return cuda_fail(e, "zgla_release_cached");
  }
  return ZGLA_OK;
}

// ------------------------------------------------------------------ SPMD comm
// region layout, per direction d: [inbox parity 0 | inbox parity 1] (nwords uint4 each) then
// control words {ctl[0] epoch, ctl[1] departures, ack}
struct zgla_allscan_comm {
  int rank, world, h, dk, dv, max_blocks;
  long long nel, nwords;  // nwords: LL words per inbox buffer (worst case EPW = 1 when dv is odd)
  size_t region_bytes;
  unsigned char* region;
  unsigned char* next_region;
  unsigned char* prev_region;
  bool next_ipc, prev_ipc;
  MappedErr err;
  unsigned long long timeout_ns;
  long long bytes_sent;
  bool broken;
};

static size_t dir_bytes(const zgla_allscan_comm* c) { return 2 * (size_t)c->nwords * sizeof(uint4) + 256; }
static uint4* inbox_of(const zgla_allscan_comm* c, unsigned char* region, int dir) {
  return reinterpret_cast<uint4*>(region + dir * dir_bytes(c));
}
static unsigned* ctl_of(const zgla_allscan_comm* c, unsigned char* region, int dir) {
  return reinterpret_cast<unsigned*>(region + dir * dir_bytes(c) + 2 * (size_t)c->nwords * sizeof(uint4));
}
static unsigned* ack_of(const zgla_allscan_comm* c, unsigned char* region, int dir) { return ctl_of(c, region, dir) + 2; }

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
  c->nwords = value_dim % 2 == 0 ? c->nel / 2 : c->nel;
  c->region_bytes = 2 * dir_bytes(c);
  c->timeout_ns = timeout_ns_default();
  c->bytes_sent = 0;
  c->broken = false;
  c->next_region = c->prev_region = nullptr;
  c->next_ipc = c->prev_ipc = false;
  if (cudaError_t e = cudaMalloc(&c->region, c->region_bytes)) {
    delete c;
    return cuda_fail(e, "zgla_allscan_create");
  }
  if (int rc = c->err.alloc()) {
    cudaFree(c->region);
    delete c;
    return rc;
  }
  cudaMemset(c->region, 0, c->region_bytes);
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

extern "C" int zgla_allscan_status(zgla_allscan_comm* c, int sync) {
  if (!c) return ZGLA_ERR_DIMS;
  if (sync) {
    if (cudaError_t e = cudaDeviceSynchronize()) return cuda_fail(e, "zgla_allscan_status");
  }
  if (c->broken || *reinterpret_cast<volatile int*>(c->err.host)) {
    c->broken = true;
    set_error("All-Scan: a flag / ack wait timed out (a peer never arrived); the communicator is unusable");
    return ZGLA_ERR_DEADLOCK;
  }
  return ZGLA_OK;
}

extern "C" int zgla_allscan_run(zgla_allscan_comm* c, int num_blocks, int direction, const float* local_state,
                                const float* log_decay, float* recv, float* scanned, void* stream) {
  if (!c || !local_state || !log_decay || !scanned) return ZGLA_ERR_DIMS;
  if (num_blocks < 1 || num_blocks > c->dk || c->dk % num_blocks) return ZGLA_ERR_CONFIG;
  if (direction != ZGLA_FWD && direction != ZGLA_BWD) return ZGLA_ERR_CONFIG;
  if (int rc = zgla_allscan_status(c, 0)) return rc;  // an earlier call timed out
  cudaStream_t st = (cudaStream_t)stream;
  const int d = direction;
  // chain order: FWD 0 -> P-1, BWD P-1 -> 0
  const bool is_source = d == ZGLA_FWD ? c->rank == 0 : c->rank == c->world - 1;
  const bool is_sink = d == ZGLA_FWD ? c->rank == c->world - 1 : c->rank == 0;
  unsigned char* succ = d == ZGLA_FWD ? c->next_region : c->prev_region;
  unsigned char* pred = d == ZGLA_FWD ? c->prev_region : c->next_region;
  if ((!is_sink && !succ) || (!is_source && !pred)) {
    set_error("All-Scan communicator is not bound to its chain neighbours");
    return ZGLA_ERR_STATE;
  }
  const int epw = epw_for(c->dv, false);
  const long long nwords = c->nwords;  // buffer stride; a call uses nel / epw of them
  Chain<float> A;
  A.local = local_state;
  A.logdecay = log_decay;
  A.inbox = nullptr;
  A.succ_inbox = nullptr;
  A.recv_out = recv;
  A.scanned_out = scanned;
  const uint4* inbox2 = is_source || c->world == 1 ? nullptr : inbox_of(c, c->region, d);
  uint4* succ_inbox2 = is_sink ? nullptr : inbox_of(c, succ, d);
  unsigned* ctl = ctl_of(c, c->region, d);
  const unsigned* my_ack = ack_of(c, c->region, d);
  unsigned* pred_ack = is_source ? nullptr : ack_of(c, pred, d);
  const int nctas = ctas_for(c->nel / epw);
  if (cudaError_t e = launch_ex(pdl_on(), rank_chain_kernel, nctas, kThreads, st, A, c->h, c->dk, c->dv, num_blocks,
                                epw, inbox2, succ_inbox2, nwords, ctl, my_ack, pred_ack, c->err.dev, c->timeout_ns))
    return cuda_fail(e, "rank_chain_kernel");
  if (int rc = zgla_check_launch()) return rc;
  if (!is_sink) c->bytes_sent += c->nel * (long long)sizeof(float);
  return ZGLA_OK;
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
  // callers synchronise all ranks (device sync + barrier) before destroying, so no peer still writes
  // into this region or reads from a mapping closed here (distributed.AllScanP2P.close)
  cudaDeviceSynchronize();
  if (c->next_ipc && c->next_region) cudaIpcCloseMemHandle(c->next_region);
  if (c->prev_ipc && c->prev_region) cudaIpcCloseMemHandle(c->prev_region);
  cudaFree(c->region);
  c->err.release();
  delete c;
  return ZGLA_OK;
}
