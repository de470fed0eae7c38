// C ABI: library bookkeeping and the ZeCO per-rank entry points
// (dispatch between the fused tcgen05 path and the generic validation path).
#include <cstdio>
#include <cstring>
#include <mutex>

#include "zgla_internal.h"

namespace zgla {

unsigned long long* g_trace_buf = nullptr;
int g_trace_cta = 0;

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

// provided by fast_fwd.cu / fast_bwd.cu
bool fast_supported(const zgla_shape* s);
long long fast_ws_bytes(const zgla_shape* s, int num_sms);
int fast_fwd_local(const zgla_shape*, int, const void*, const void*, const void*, void*, void*, void*, cudaStream_t);
int fast_fwd_output(const zgla_shape*, int, const void*, const void*, const void*, const void*, void*, const void*,
                    void*, cudaStream_t);
int fast_bwd_local(const zgla_shape*, int, const void*, const void*, const void*, void*, void*, cudaStream_t);
int fast_bwd_output(const zgla_shape*, int, const void*, const void*, const void*, const void*, const void*, void*,
                    const void*, const void*, void*, void*, void*, void*, cudaStream_t);

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

extern "C" int zgla_zeco_fwd_local(const zgla_shape* s, int num_sms, const void* k, const void* v, const void* g,
                                   void* ws, void* s_local, void* g_tot, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (fast_supported(s)) return fast_fwd_local(s, num_sms, k, v, g, ws, s_local, g_tot, st);
  return generic_zeco_fwd_local(s, k, v, g, ws, s_local, g_tot, st);
}

extern "C" int zgla_zeco_fwd_output(const zgla_shape* s, int num_sms, const void* q, const void* k, const void* v,
                                    const void* g, void* ws, const void* s_prev, void* o, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (fast_supported(s)) return fast_fwd_output(s, num_sms, q, k, v, g, ws, s_prev, o, st);
  return generic_zeco_fwd_output(s, q, k, v, g, ws, s_prev, o, st);
}

extern "C" int zgla_zeco_bwd_local(const zgla_shape* s, int num_sms, const void* q, const void* g,
                                   const void* d_out, void* ws, void* ds_local0, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (fast_supported(s)) return fast_bwd_local(s, num_sms, q, g, d_out, ws, ds_local0, st);
  return generic_zeco_bwd_local(s, q, g, d_out, ws, ds_local0, st);
}

extern "C" int zgla_zeco_bwd_output(const zgla_shape* s, int num_sms, const void* q, const void* k, const void* v,
                                    const void* g, const void* d_out, void* ws, const void* s_prev,
                                    const void* ds_next, void* dq, void* dk, void* dv, void* dg, void* stream) {
  if (int rc = validate_zeco(s, num_sms)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (fast_supported(s))
    return fast_bwd_output(s, num_sms, q, k, v, g, d_out, ws, s_prev, ds_next, dq, dk, dv, dg, st);
  return generic_zeco_bwd_output(s, q, k, v, g, d_out, ws, s_prev, ds_next, dq, dk, dv, dg, st);
}
