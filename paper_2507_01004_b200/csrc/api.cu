// C ABI: library bookkeeping and the ZeCO per-rank entry points
// (dispatch between the fused tcgen05 path and the generic validation path).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "fast_common.cuh"
#include "zgla_internal.h"

namespace zgla {

unsigned long long* g_trace_buf = nullptr;
int g_trace_cta = 0;

// early inputs of the fused output kernels (fast_common.cuh): process-wide caller contract, off by default
static std::atomic<int> g_early_inputs{-1};
namespace fast {
int early_inputs() {
  int v = g_early_inputs.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("ZGLA_EARLY_INPUTS");
    v = (e && e[0] == '1') ? 1 : 0;
    g_early_inputs.store(v, std::memory_order_relaxed);
  }
  return v;
}
}  // namespace fast

static thread_local char g_err[512] = "";

void set_error(const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
}

int cuda_fail(cudaError_t e, const char* where) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
  return ZGLA_ERR_CUDA;
}

// provided by generic.cu
int generic_zeco_fwd_local(const zgla_shape*, const void*, const void*, const void*, void*, void*, void*,
                           cudaStream_t);
int generic_zeco_fwd_output(const zgla_shape*, const void*, const void*, const void*, const void*, void*,
                            const void*, void*, cudaStream_t);
int generic_zeco_bwd_local(const zgla_shape*, const void*, const void*, const void*, void*, void*, cudaStream_t);
int generic_zeco_bwd_output(const zgla_shape*, const void*, const void*, const void*, const void*, const void*,
                            void*, const void*, const void*, void*, void*, void*, void*, cudaStream_t);
long long generic_ws_bytes(const zgla_shape*);

// provided by fast_fwd.cu / fast_bwd.cu (strided tensors)
namespace fast {
struct TRef;
}
bool fast_supported(const zgla_shape* s);
int fast_domain_flag(const zgla_shape* s, int num_sms, const void* ws, int* host_flag, cudaStream_t st);
long long fast_ws_bytes(const zgla_shape* s, int num_sms);
int fast_fwd_local(const zgla_shape*, int, const fast::TRef&, const fast::TRef&, const fast::TRef&, void*, void*,
                   void*, cudaStream_t);
int fast_fwd_output(const zgla_shape*, int, const fast::TRef&, const fast::TRef&, const fast::TRef&,
                    const fast::TRef&, void*, const void*, const fast::TRef&, cudaStream_t, bool save_states = true);
int fast_bwd_local(const zgla_shape*, int, const fast::TRef&, const fast::TRef&, const fast::TRef&, void*, void*,
                   cudaStream_t);
int fast_bwd_output(const zgla_shape*, int, const fast::TRef&, const fast::TRef&, const fast::TRef&,
                    const fast::TRef&, const fast::TRef&, void*, const void*, const void*, const fast::TRef&,
                    const fast::TRef&, const fast::TRef&, const fast::TRef&, cudaStream_t);

}  // namespace zgla

using namespace zgla;

extern "C" int zgla_check_launch_impl(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, where);
  return ZGLA_OK;
}

extern "C" int zgla_set_trace(void* dev_buf, int cta) {
  g_trace_buf = reinterpret_cast<unsigned long long*>(dev_buf);
  g_trace_cta = cta;
  return ZGLA_OK;
}

extern "C" const char* zgla_version(void) { return "zeco-gla-b200 0.1.0 (sm_100a)"; }
extern "C" const char* zgla_last_error(void) { return g_err; }

static int validate_zeco(const zgla_shape* s, int num_sms) {
  if (!s || s->heads < 1 || s->key_dim < 1 || s->value_dim < 1 || s->seq_len < 1 || s->chunk_len < 1)
    return ZGLA_ERR_DIMS;
  if (s->seq_len % s->chunk_len) return ZGLA_ERR_DIMS;
  if (s->dtype < ZGLA_BF16 || s->dtype > ZGLA_F64) return ZGLA_ERR_CONFIG;
  if (num_sms < 1) return ZGLA_ERR_CONFIG;
  return ZGLA_OK;
}

extern "C" int zgla_fast_path(const zgla_shape* s) { return (s && fast_supported(s)) ? 1 : 0; }

extern "C" long long zgla_zeco_workspace_bytes(const zgla_shape* s, int num_sms) {
  if (validate_zeco(s, num_sms)) return -1;
  return fast_supported(s) ? fast_ws_bytes(s, num_sms) : generic_ws_bytes(s);
}

// ---- ZeCO entry points: strided (zgla_tensor) forms; the pointer forms below are dense wrappers
static bool dense(const zgla_tensor* t, const zgla_shape* s, int width) {
  return (t->token_stride == 0 || t->token_stride == width) &&
         (t->head_stride == 0 || s->heads == 1 || t->head_stride == s->seq_len * width);
}
// fast path: every tensor 16-byte aligned with aligned strides; SIMT path: dense tensors only
static int check_refs(const zgla_shape* s, std::initializer_list<const zgla_tensor*> ts, bool fast_path) {
  for (const zgla_tensor* t : ts) {
    if (!t || !t->data) return ZGLA_ERR_DIMS;
    if (fast_path) {
      if (!fast::ref_ok(fast::as_ref(t, s->seq_len, s->heads, s->key_dim), 2)) {
        set_error("strided tensor: base and strides must be 16-byte aligned, token stride >= channels");
        return ZGLA_ERR_LAYOUT;
      }
    } else if (!dense(t, s, s->key_dim) && !dense(t, s, s->value_dim)) {
      set_error("the SIMT (non-bf16 / non-128) path needs dense [heads][tokens][channels] tensors");
      return ZGLA_ERR_LAYOUT;
    }
  }
  return ZGLA_OK;
}

extern "C" int zgla_zeco_fwd_local_v(const zgla_shape* s, int num_sms, const zgla_tensor* k, const zgla_tensor* v,
                                     const zgla_tensor* g, void* ws, void* s_local, void* g_tot, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  const bool fp = fast_supported(s);
  if (int rc = check_refs(s, {k, v, g}, fp)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long L = s->seq_len;
  if (fp)
    return fast_fwd_local(s, num_sms, fast::as_ref(k, L, s->heads, s->key_dim), fast::as_ref(v, L, s->heads, s->key_dim), fast::as_ref(g, L, s->heads, s->key_dim), ws, s_local, g_tot,
                          st);
  return generic_zeco_fwd_local(s, k->data, v->data, g->data, ws, s_local, g_tot, st);
}

extern "C" int zgla_zeco_fwd_output_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* k,
                                      const zgla_tensor* v, const zgla_tensor* g, void* ws, const void* s_prev,
                                      const zgla_tensor* o, void* stream) {
  return zgla_zeco_fwd_output_ex_v(s, num_sms, q, k, v, g, ws, s_prev, o, 0, stream);
}

extern "C" int zgla_zeco_fwd_output_ex_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* k,
                                         const zgla_tensor* v, const zgla_tensor* g, void* ws, const void* s_prev,
                                         const zgla_tensor* o, int flags, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  if (flags & ~ZGLA_FWD_NO_SAVE) return ZGLA_ERR_CONFIG;
  const bool fp = fast_supported(s);
  if (int rc = check_refs(s, {q, k, v, g, o}, fp)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long L = s->seq_len;
  if (fp)
    return fast_fwd_output(s, num_sms, fast::as_ref(q, L, s->heads, s->key_dim), fast::as_ref(k, L, s->heads, s->key_dim), fast::as_ref(v, L, s->heads, s->key_dim),
                           fast::as_ref(g, L, s->heads, s->key_dim), ws, s_prev, fast::as_ref(o, L, s->heads, s->key_dim), st,
                           (flags & ZGLA_FWD_NO_SAVE) == 0);
  return generic_zeco_fwd_output(s, q->data, k->data, v->data, g->data, ws, s_prev, o->data, st);
}

extern "C" int zgla_zeco_bwd_local_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* g,
                                     const zgla_tensor* d_out, void* ws, void* ds_local0, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  const bool fp = fast_supported(s);
  if (int rc = check_refs(s, {q, g, d_out}, fp)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long L = s->seq_len;
  if (fp)
    return fast_bwd_local(s, num_sms, fast::as_ref(q, L, s->heads, s->key_dim), fast::as_ref(g, L, s->heads, s->key_dim), fast::as_ref(d_out, L, s->heads, s->key_dim), ws, ds_local0,
                          st);
  return generic_zeco_bwd_local(s, q->data, g->data, d_out->data, ws, ds_local0, st);
}

extern "C" int zgla_zeco_bwd_output_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* k,
                                      const zgla_tensor* v, const zgla_tensor* g, const zgla_tensor* d_out, void* ws,
                                      const void* s_prev, const void* ds_next, const zgla_tensor* dq,
                                      const zgla_tensor* dk, const zgla_tensor* dv, const zgla_tensor* dg,
                                      void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  const bool fp = fast_supported(s);
  if (int rc = check_refs(s, {q, k, v, g, d_out, dq, dk, dv, dg}, fp)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long L = s->seq_len;
  if (fp)
    return fast_bwd_output(s, num_sms, fast::as_ref(q, L, s->heads, s->key_dim), fast::as_ref(k, L, s->heads, s->key_dim), fast::as_ref(v, L, s->heads, s->key_dim),
                           fast::as_ref(g, L, s->heads, s->key_dim), fast::as_ref(d_out, L, s->heads, s->key_dim), ws, s_prev, ds_next, fast::as_ref(dq, L, s->heads, s->key_dim),
                           fast::as_ref(dk, L, s->heads, s->key_dim), fast::as_ref(dv, L, s->heads, s->key_dim), fast::as_ref(dg, L, s->heads, s->key_dim), st);
  return generic_zeco_bwd_output(s, q->data, k->data, v->data, g->data, d_out->data, ws, s_prev, ds_next, dq->data,
                                 dk->data, dv->data, dg->data, st);
}

static zgla_tensor dn(const void* p) { return zgla_tensor{const_cast<void*>(p), 0, 0}; }

extern "C" int zgla_zeco_fwd_local(const zgla_shape* s, int num_sms, const void* k, const void* v, const void* g,
                                   void* ws, void* s_local, void* g_tot, void* stream) {
  const zgla_tensor tk = dn(k), tv = dn(v), tg = dn(g);
  return zgla_zeco_fwd_local_v(s, num_sms, &tk, &tv, &tg, ws, s_local, g_tot, stream);
}

extern "C" int zgla_zeco_fwd_output(const zgla_shape* s, int num_sms, const void* q, const void* k, const void* v,
                                    const void* g, void* ws, const void* s_prev, void* o, void* stream) {
  const zgla_tensor tq = dn(q), tk = dn(k), tv = dn(v), tg = dn(g), to = dn(o);
  return zgla_zeco_fwd_output_v(s, num_sms, &tq, &tk, &tv, &tg, ws, s_prev, &to, stream);
}

extern "C" int zgla_zeco_bwd_local(const zgla_shape* s, int num_sms, const void* q, const void* g,
                                   const void* d_out, void* ws, void* ds_local0, void* stream) {
  const zgla_tensor tq = dn(q), tg = dn(g), td = dn(d_out);
  return zgla_zeco_bwd_local_v(s, num_sms, &tq, &tg, &td, ws, ds_local0, stream);
}

extern "C" int zgla_zeco_bwd_output(const zgla_shape* s, int num_sms, const void* q, const void* k, const void* v,
                                    const void* g, const void* d_out, void* ws, const void* s_prev,
                                    const void* ds_next, void* dq, void* dk, void* dv, void* dg, void* stream) {
  const zgla_tensor tq = dn(q), tk = dn(k), tv = dn(v), tg = dn(g), td = dn(d_out);
  const zgla_tensor a = dn(dq), b = dn(dk), c = dn(dv), e = dn(dg);
  return zgla_zeco_bwd_output_v(s, num_sms, &tq, &tk, &tv, &tg, &td, ws, s_prev, ds_next, &a, &b, &c, &e, stream);
}

namespace zgla {
int watch_domain(const void* ws, int** host_flag);
int unwatch_domain(const void* ws);
}
extern "C" int zgla_zeco_watch_domain(void* ws, int** host_flag) {
  if (!ws || !host_flag) return ZGLA_ERR_DIMS;
  return zgla::watch_domain(ws, host_flag);
}
extern "C" int zgla_zeco_unwatch_domain(void* ws) { return zgla::unwatch_domain(ws); }

extern "C" int zgla_zeco_domain_check(const zgla_shape* s, int num_sms, const void* ws, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  if (!fast_supported(s)) return ZGLA_OK;  // the SIMT paths use the exact token recurrence: any gate
  int flag = 0;
  if (int rc = fast_domain_flag(s, num_sms, ws, &flag, (cudaStream_t)stream)) return rc;
  if (flag) {
    set_error("a log-decay entry is >= 0 or not finite (glasp/gla.py:106-107), or a 64-token tile's summed "
              "log-decay is below -160 (outside the fused bf16 path's exponent domain: use the fp32 mode)");
    return ZGLA_ERR_DOMAIN;
  }
  return ZGLA_OK;
}

extern "C" int zgla_set_early_inputs(int on) {
  const int old = zgla::fast::early_inputs();
  zgla::g_early_inputs.store(on ? 1 : 0, std::memory_order_relaxed);
  return old;
}
