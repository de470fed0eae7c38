// Host-buffer entry point: one ZeCO GLA layer forward + backward whose inputs and
// outputs live in (pinned) HOST memory -- the shape of the reference's own
// verify/bench flow (glasp/cli.py:241-361: run_forward then run_backward with a
// given dO, arrays in host memory).
//
// Heads are independent, so the call cuts the heads into `head_groups` groups
// and runs a three-stage pipeline over them on three streams:
//   h2d stream :  q,k,v,g,dO of group j  host -> device
//   compute    :  fwd_local -> All-Scan FWD -> fwd_output -> bwd_local ->
//                 All-Scan BWD -> bwd_output of group j   (the caller's stream)
//   d2h stream :  o,dq,dk,dv,dg of group j  device -> host
// so the PCIe transfers of both directions run concurrently with each other
// and with the kernels; the whole call costs about max(H2D, D2H) bytes over
// the link plus one group's latency, instead of H2D + compute + D2H.
// With a peer communicator (world > 1) every group runs its own All-Scan on
// the group's [hg, dk, dv] states; all ranks walk the groups in the same
// order, so the chain protocol's epochs line up.
#include <cuda.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "zgla_internal.h"

namespace zgla {
namespace hostpipe {

struct Ctx {
  int dev = -1;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;  // per group: H2D done, kernels done, D2H done; then start, done
  // geometry of the last call (ZGLA_HOST_OVERLAP chains only onto an identical previous call)
  int last_G = 0, last_heads = 0, last_dtype = -1;
  long long last_L = 0;
  const void* last_buf = nullptr;
};
static std::mutex g_mu;
static Ctx g_ctx[64];

static int get_ctx(Ctx** out, size_t nev) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_fail(e, "zgla_zeco_fwd_bwd_host");
  if (dev < 0 || dev >= 64) return ZGLA_ERR_CONFIG;
  Ctx& c = g_ctx[dev];
  if (c.dev < 0) {
    if (cudaError_t e = cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking)) return cuda_fail(e, "stream");
    if (cudaError_t e = cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking)) return cuda_fail(e, "stream");
    c.dev = dev;
  }
  while (c.ev.size() < nev) {
    cudaEvent_t e;
    if (cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) return cuda_fail(r, "event");
    c.ev.push_back(e);
  }
  *out = &c;
  return ZGLA_OK;
}

// the five transfers of one group and direction, in the order given by `ord`: runs of equal-sized
// transfers whose sources and destinations are both equally spaced (tensors allocated back to back, as
// the device layout places q k v dO and o dq dk dv) go out as ONE cudaMemcpy2DAsync (rows = tensors), the
// rest as one cudaMemcpyAsync each.  Each submitted copy costs ~50 us of duplex DMA efficiency on this link,
// so fewer, larger submissions win.
// true iff the byte ranges [a, a+1) and [b, b+1) lie in the same CUDA allocation (pinned host memory or device
// memory; unified addressing): a 2-D copy may only span rows of one allocation
static bool same_alloc(const void* a, const void* b) {
  using Fn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
  static Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuPointerGetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<Fn>(p)
               : nullptr;
  }();
  if (!fn) return false;
  CUdeviceptr sa = 0, sb = 0;
  if (fn(&sa, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, reinterpret_cast<CUdeviceptr>(a)) != CUDA_SUCCESS ||
      fn(&sb, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, reinterpret_cast<CUdeviceptr>(b)) != CUDA_SUCCESS)
    return false;
  return sa == sb;
}

static int copy5(void** dsts, void** srcs, size_t* sizes, const int* ord, cudaMemcpyKind kind, cudaStream_t st) {
  int i = 0;
  while (i < 5) {
    const int a = ord[i];
    int n = 1;
    long long dp = 0, sp = 0;
    if (i + 1 < 5) {
      const int b = ord[i + 1];
      dp = (long long)((char*)dsts[b] - (char*)dsts[a]);
      sp = (long long)((char*)srcs[b] - (char*)srcs[a]);
      if (sizes[b] == sizes[a] && dp >= (long long)sizes[a] && sp >= (long long)sizes[a]) {
        n = 2;
        while (i + n < 5) {
          const int c = ord[i + n], p = ord[i + n - 1];
          if (sizes[c] != sizes[a] || (char*)dsts[c] - (char*)dsts[p] != dp || (char*)srcs[c] - (char*)srcs[p] != sp)
            break;
          ++n;
        }
      }
    }
    if (sizes[a] == 0) {
      i += n;
      continue;
    }
    if (n > 1) {  // the rows must lie in one allocation on both sides (tensors carved from one arena)
      const int last = ord[i + n - 1];
      if (!same_alloc(srcs[a], (char*)srcs[last] + sizes[a] - 1) || !same_alloc(dsts[a], (char*)dsts[last] + sizes[a] - 1)) {
        for (int j = 0; j < n; ++j) {
          const int c = ord[i + j];
          if (cudaError_t e = cudaMemcpyAsync(dsts[c], srcs[c], sizes[c], kind, st)) return cuda_fail(e, "host copy");
        }
        i += n;
        continue;
      }
    }
    cudaError_t r = n > 1 ? cudaMemcpy2DAsync(dsts[a], (size_t)dp, srcs[a], (size_t)sp, sizes[a], (size_t)n, kind, st)
                          : cudaMemcpyAsync(dsts[a], srcs[a], sizes[a], kind, st);
    if (r != cudaSuccess) {  // e.g. a pitch beyond the device limit: one copy per tensor
      cudaGetLastError();
      for (int j = 0; j < n; ++j) {
        const int c = ord[i + j];
        if (cudaError_t e = cudaMemcpyAsync(dsts[c], srcs[c], sizes[c], kind, st)) return cuda_fail(e, "host copy");
      }
    }
    i += n;
  }
  return ZGLA_OK;
}

inline long long al256(long long x) { return (x + 255) & ~255ll; }
inline int esize(int dt) { return dt == ZGLA_BF16 ? 2 : dt == ZGLA_F32 ? 4 : 8; }
inline int asize(int dt) { return dt == ZGLA_F64 ? 8 : 4; }

// Head ranges of the groups.  Single-rank calls taper the pipeline: the first and the last group
// hold one head each (pipeline fill = one head's H2D, drain = one head's kernels + D2H) and the
// interior groups share the rest evenly.  With peers every group must match the communicator's
// head count, so the split is uniform.
static std::vector<int> group_bounds(int H, int G, bool tapered) {
  std::vector<int> b(G + 1);
  if (tapered && G >= 3 && H >= G + 1) {
    b[0] = 0;
    b[1] = 1;
    for (int j = 1; j < G - 1; ++j) b[j + 1] = 1 + (int)((long long)j * (H - 2) / (G - 2));
    b[G] = H;
  } else {
    for (int j = 0; j <= G; ++j) b[j] = (int)((long long)j * H / G);
  }
  return b;
}

// device scratch carve-up: 5 inputs, 5 outputs, ZeCO workspace of the largest group, 7 group states
struct Layout {
  long long in[5], out[5], ws, st[7], total;
};

static int layout(const zgla_shape* s, int num_sms, int groups, bool tapered, Layout* lo) {
  if (!s || s->heads < 1 || groups < 1 || groups > s->heads) return ZGLA_ERR_CONFIG;
  const std::vector<int> gb = group_bounds(s->heads, groups, tapered);
  const long long HL = (long long)s->heads * s->seq_len;
  const long long e = esize(s->dtype), a = asize(s->dtype);
  const long long in_bytes[5] = {HL * s->key_dim * e, HL * s->key_dim * e, HL * s->value_dim * e,
                                 HL * s->key_dim * a, HL * s->value_dim * e};  // q k v g dO
  const long long out_bytes[5] = {HL * s->value_dim * e, HL * s->key_dim * e, HL * s->key_dim * e,
                                  HL * s->value_dim * e, HL * s->key_dim * a};  // o dq dk dv dg
  long long off = 0;
  for (int i : {0, 1, 2, 4, 3}) lo->in[i] = off, off += al256(in_bytes[i]);  // q k v dO g: equal pitch for 2-D copies
  for (int i = 0; i < 5; ++i) lo->out[i] = off, off += al256(out_bytes[i]);
  long long ws = 0;
  int hmax = 0;
  for (int j = 0; j < groups; ++j) hmax = gb[j + 1] - gb[j] > hmax ? gb[j + 1] - gb[j] : hmax;
  for (int j = 0; j < groups; ++j) {
    const int hg = gb[j + 1] - gb[j];
    zgla_shape gs = *s;
    gs.heads = hg;
    const long long b = zgla_zeco_workspace_bytes(&gs, num_sms);
    if (b < 0) return ZGLA_ERR_DIMS;
    ws = b > ws ? b : ws;
  }
  lo->ws = off;
  off += al256(ws);
  const long long st = (long long)hmax * s->key_dim * s->value_dim * a;
  for (int i = 0; i < 7; ++i) lo->st[i] = off, off += al256(i == 1 ? (long long)hmax * s->key_dim * a : st);
  lo->total = off;
  return ZGLA_OK;
}

}  // namespace hostpipe
}  // namespace zgla

using namespace zgla;
using namespace zgla::hostpipe;

extern "C" long long zgla_zeco_fwd_bwd_host_bytes(const zgla_shape* s, int num_sms, int head_groups) {
  // the larger of the two splits, so one buffer serves single-rank and peer calls
  Layout a, b;
  if (layout(s, num_sms, head_groups, true, &a) || layout(s, num_sms, head_groups, false, &b)) return -1;
  return a.total > b.total ? a.total : b.total;
}

extern "C" int zgla_zeco_fwd_bwd_host(const zgla_shape* s, int num_sms, int head_groups, zgla_allscan_comm* comm,
                                      int num_blocks, const void* q, const void* k, const void* v, const void* g,
                                      const void* d_out, void* o, void* dq, void* dk, void* dv, void* dg,
                                      void* dev_buf, long long dev_buf_bytes, int flags, void* stream) {
  if (!s) return ZGLA_ERR_DIMS;
  int rank = 0, world = 1, comm_heads = 0;
  if (comm) {
    if (int rc = zgla_allscan_info(comm, &rank, &world, &comm_heads)) return rc;
    if (s->dtype == ZGLA_F64) return ZGLA_ERR_UNSUPPORTED;  // the peer chain carries fp32 states
    if (world > 1 && (head_groups < 1 || s->heads % head_groups || comm_heads != s->heads / head_groups)) {
      set_error("zgla_zeco_fwd_bwd_host: the communicator must be created for heads / head_groups heads");
      return ZGLA_ERR_CONFIG;
    }
  }
  const bool peers = comm && world > 1;
  Layout lo;
  if (int rc = layout(s, num_sms, head_groups, !peers, &lo)) return rc;
  const std::vector<int> gb = group_bounds(s->heads, head_groups, !peers);
  if (!q || !k || !v || !g || !d_out || !o || !dq || !dk || !dv || !dg || !dev_buf) return ZGLA_ERR_DIMS;
  if (dev_buf_bytes < lo.total) {
    set_error("zgla_zeco_fwd_bwd_host: device buffer smaller than zgla_zeco_fwd_bwd_host_bytes()");
    return ZGLA_ERR_DIMS;
  }
  const int G = head_groups;
  Ctx* cx = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (int rc = get_ctx(&cx, 3 * (size_t)G + 2)) return rc;
  }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char* base = reinterpret_cast<unsigned char*>(dev_buf);
  const long long L = s->seq_len, e = esize(s->dtype), a = asize(s->dtype);
  // per-head bytes of each tensor (inputs q k v g dO, outputs o dq dk dv dg)
  const long long ph_in[5] = {L * s->key_dim * e, L * s->key_dim * e, L * s->value_dim * e, L * s->key_dim * a,
                              L * s->value_dim * e};
  const long long ph_out[5] = {L * s->value_dim * e, L * s->key_dim * e, L * s->key_dim * e,
                               L * s->value_dim * e, L * s->key_dim * a};
  const void* hin[5] = {q, k, v, g, d_out};
  void* hout[5] = {o, dq, dk, dv, dg};
  cudaEvent_t* ev_in = &cx->ev[0];
  cudaEvent_t* ev_comp = &cx->ev[G];
  cudaEvent_t* ev_d2h = &cx->ev[2 * G];
  cudaEvent_t ev_start = cx->ev[3 * G], ev_done = cx->ev[3 * G + 1];
  // ZGLA_HOST_OVERLAP: chain onto the previous call with the same geometry and buffer through per-group
  // events only (group j's H2D waits for the previous call's group-j kernels, its kernels for the
  // previous call's group-j D2H), so this call's H2D runs under the previous call's D2H.  The caller's
  // stream is then NOT made to wait for the D2H: zgla_zeco_host_wait() does that.
  const bool chain = (flags & ZGLA_HOST_OVERLAP) && cx->last_G == G && cx->last_buf == dev_buf &&
                     cx->last_heads == s->heads && cx->last_L == s->seq_len && cx->last_dtype == s->dtype;
  // diagnostics: ZGLA_HOST_TRACE=1 prints the per-group timeline (synchronises; never in timed runs)
  static const bool trace = std::getenv("ZGLA_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  if (trace) {
    tev.resize(3 * G + 1);
    for (auto& x : tev) cudaEventCreate(&x);
    cudaEventRecord(tev[3 * G], st);
  }
  if (!chain) {
    // the device buffers may still be in use by earlier work on the caller's stream
    if (cudaError_t r = cudaEventRecord(ev_start, st)) return cuda_fail(r, "zgla_zeco_fwd_bwd_host");
    cudaStreamWaitEvent(cx->h2d, ev_start, 0);
    cudaStreamWaitEvent(cx->d2h, ev_start, 0);
  }
  for (int j = 0; j < G; ++j) {
    const int h0 = gb[j], h1 = gb[j + 1];
    const int hg = h1 - h0;
    if (chain) cudaStreamWaitEvent(cx->h2d, ev_comp[j], 0);  // previous call's kernels of group j
    {
      void* dsts[5];
      void* srcs[5];
      size_t sizes[5];
      for (int i = 0; i < 5; ++i) {
        dsts[i] = base + lo.in[i] + h0 * ph_in[i];
        srcs[i] = const_cast<unsigned char*>(reinterpret_cast<const unsigned char*>(hin[i])) + h0 * ph_in[i];
        sizes[i] = (size_t)(hg * ph_in[i]);
      }
      static const int ord_in[5] = {0, 1, 2, 4, 3};  // q k v dO g
      if (int rc = copy5(dsts, srcs, sizes, ord_in, cudaMemcpyHostToDevice, cx->h2d)) return rc;
    }
    cudaEventRecord(ev_in[j], cx->h2d);
    if (trace) cudaEventRecord(tev[3 * j], cx->h2d);
    cudaStreamWaitEvent(st, ev_in[j], 0);
    if (chain) cudaStreamWaitEvent(st, ev_d2h[j], 0);  // previous call's D2H of group j's outputs
    zgla_shape gs = *s;
    gs.heads = hg;
    void* in[5];
    void* out[5];
    for (int i = 0; i < 5; ++i) in[i] = base + lo.in[i] + h0 * ph_in[i];
    for (int i = 0; i < 5; ++i) out[i] = base + lo.out[i] + h0 * ph_out[i];
    void* ws = base + lo.ws;
    float* s_local = reinterpret_cast<float*>(base + lo.st[0]);
    float* g_tot = reinterpret_cast<float*>(base + lo.st[1]);
    float* recv_f = reinterpret_cast<float*>(base + lo.st[2]);
    float* scan_f = reinterpret_cast<float*>(base + lo.st[3]);
    float* ds0 = reinterpret_cast<float*>(base + lo.st[4]);
    float* recv_b = reinterpret_cast<float*>(base + lo.st[5]);
    float* scan_b = reinterpret_cast<float*>(base + lo.st[6]);
    if (int rc = zgla_zeco_fwd_local(&gs, num_sms, in[1], in[2], in[3], ws, s_local, g_tot, st)) return rc;
    const void* prev = nullptr;
    if (peers) {
      if (int rc = zgla_allscan_run(comm, num_blocks, ZGLA_FWD, s_local, g_tot, recv_f, scan_f, st)) return rc;
      prev = rank > 0 ? recv_f : nullptr;
    }
    if (int rc = zgla_zeco_fwd_output(&gs, num_sms, in[0], in[1], in[2], in[3], ws, prev, out[0], st)) return rc;
    if (int rc = zgla_zeco_bwd_local(&gs, num_sms, in[0], in[3], in[4], ws, ds0, st)) return rc;
    const void* ds_next = nullptr;
    if (peers) {
      if (int rc = zgla_allscan_run(comm, num_blocks, ZGLA_BWD, ds0, g_tot, recv_b, scan_b, st)) return rc;
      ds_next = rank < world - 1 ? recv_b : nullptr;
    }
    if (int rc = zgla_zeco_bwd_output(&gs, num_sms, in[0], in[1], in[2], in[3], in[4], ws, prev, ds_next, out[1],
                                      out[2], out[3], out[4], st))
      return rc;
    cudaEventRecord(ev_comp[j], st);
    if (trace) cudaEventRecord(tev[3 * j + 1], st);
    cudaStreamWaitEvent(cx->d2h, ev_comp[j], 0);
    {
      void* dsts[5];
      void* srcs[5];
      size_t sizes[5];
      for (int i = 0; i < 5; ++i) {
        dsts[i] = reinterpret_cast<unsigned char*>(hout[i]) + h0 * ph_out[i];
        srcs[i] = base + lo.out[i] + h0 * ph_out[i];
        sizes[i] = (size_t)(hg * ph_out[i]);
      }
      static const int ord_out[5] = {0, 1, 2, 3, 4};  // o dq dk dv dg
      if (int rc = copy5(dsts, srcs, sizes, ord_out, cudaMemcpyDeviceToHost, cx->d2h)) return rc;
    }
    cudaEventRecord(ev_d2h[j], cx->d2h);
    if (trace) cudaEventRecord(tev[3 * j + 2], cx->d2h);
  }
  cudaEventRecord(ev_done, cx->d2h);
  const bool overlap = (flags & ZGLA_HOST_OVERLAP) != 0;
  if (!overlap) cudaStreamWaitEvent(st, ev_done, 0);  // completion of the caller's stream => outputs written
  cx->last_G = G;
  cx->last_buf = dev_buf;
  cx->last_heads = s->heads;
  cx->last_L = s->seq_len;
  cx->last_dtype = s->dtype;
  if (trace) {
    cudaDeviceSynchronize();
    for (int j = 0; j < G; ++j) {
      float t0, t1, t2;
      cudaEventElapsedTime(&t0, tev[3 * G], tev[3 * j]);
      cudaEventElapsedTime(&t1, tev[3 * G], tev[3 * j + 1]);
      cudaEventElapsedTime(&t2, tev[3 * G], tev[3 * j + 2]);
      std::fprintf(stderr, "zgla host trace group %d: h2d %.3f compute %.3f d2h %.3f ms\n", j, t0, t1, t2);
    }
    for (auto& x : tev) cudaEventDestroy(x);
  }
  return zgla_check_launch();
}

extern "C" int zgla_zeco_host_wait(void* stream) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_fail(e, "zgla_zeco_host_wait");
  std::lock_guard<std::mutex> lock(g_mu);
  Ctx& c = g_ctx[dev];
  if (c.dev < 0 || c.ev.empty() || c.last_G <= 0) return ZGLA_OK;
  if (cudaError_t e = cudaStreamWaitEvent((cudaStream_t)stream, c.ev[3 * c.last_G + 1], 0))
    return cuda_fail(e, "zgla_zeco_host_wait");
  return ZGLA_OK;
}
