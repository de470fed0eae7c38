// Token-by-token GLA recurrence: the exactness oracle of the reference's API
// (glasp/gla.py:210-230 recurrent_forward) and the loss it differentiates
// numerically (glasp/gla.py:447-480 finite_diff_grad).  Deliberately
// independent of every chunkwise kernel (generic.cu, fast_*.cu): no chunk
// factorisation, no segment scan -- one state update per token,
//
//     S_t = e^{g_t} (.) S_{t-1} + k_t^T v_t,     o_t = q_t S_t,
//
// with the reference's rounding sequence for the update (the decay product and
// the outer product rounded separately, then added; no FMA contraction).
//
// recurrent_kernel: one CTA per (head, slab of J value columns); thread
// (c, jj) owns state element S[c][j] in a register; o_t[j] is reduced over c
// in a fixed sequential order from a double-buffered shared product tile (one
// barrier per token).  Boundary states are written after every C tokens.
//
// fd_loss_kernel: one CTA per perturbation (tensor element, +step / -step).
// The CTA runs the whole recurrence (all heads) with the state in shared
// memory and returns sum(probe * o) with a fixed reduction order, so one
// launch evaluates every central difference of one tensor.
#include <algorithm>

#include "zgla_internal.h"

namespace zgla {
namespace recur {

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename Tin, typename Ta>
__global__ void recurrent_kernel(int h, long long L, int dk, int dv, int C, int J, const Tin* __restrict__ q,
                                 const Tin* __restrict__ k, const Tin* __restrict__ v, const Ta* __restrict__ g,
                                 const Ta* __restrict__ init, Tin* __restrict__ o, Ta* __restrict__ bounds,
                                 Ta* __restrict__ final_state) {
  extern __shared__ unsigned char smem_raw[];
  Ta* prod = reinterpret_cast<Ta*>(smem_raw);  // [2][dk][J]
  const int hh = blockIdx.x;
  const int c = threadIdx.x / J, jj = threadIdx.x % J;
  const int j = blockIdx.y * J + jj;
  const bool live = c < dk && j < dv;
  const long long st_off = ((long long)hh * dk + c) * dv + j;
  Ta s = (live && init) ? init[st_off] : Ta(0);
  const long long n_state = (long long)h * dk * dv;
  if (live && bounds) bounds[st_off] = s;
  const long long rowq = (long long)hh * L * dk, rowv = (long long)hh * L * dv;
  for (long long t = 0; t < L; ++t) {
    Ta* buf = prod + (t & 1) * dk * J;
    if (live) {
      const Ta a = ex(g[rowq + t * dk + c]);
      const Ta kv = mul_rn<Ta>(ld_in(k + rowq + t * dk + c), ld_in(v + rowv + t * dv + j));
      s = add_rn<Ta>(mul_rn<Ta>(a, s), kv);
      buf[c * J + jj] = mul_rn<Ta>(ld_in(q + rowq + t * dk + c), s);
      if (bounds && (t + 1) % C == 0) bounds[((t + 1) / C) * n_state + st_off] = s;
    }
    __syncthreads();
    if (c == 0 && j < dv) {
      Ta acc = buf[jj];
      for (int cc = 1; cc < dk; ++cc) acc = add_rn<Ta>(acc, buf[cc * J + jj]);
      st_out(o + rowv + t * dv + j, acc);
    }
    // the next token writes the other buffer; the one after that reuses this one, which every reader
    // has finished with by the next barrier
  }
  if (live && final_state) final_state[st_off] = s;
}

// value of tensor `which` (0 q, 1 k, 2 v, 3 g) at flat index i, bumped when it is the perturbed element
__device__ __forceinline__ double fd_val(const double* base, int which, long long i, int p_which, long long p_idx,
                                         double bump) {
  const double x = base[i];
  return (which == p_which && i == p_idx) ? __dadd_rn(x, bump) : x;
}

__global__ void fd_loss_kernel(int h, long long L, int dk, int dv, const double* __restrict__ q,
                               const double* __restrict__ k, const double* __restrict__ v,
                               const double* __restrict__ g, const double* __restrict__ probe, int p_which,
                               long long first, double step, double* __restrict__ losses) {
  extern __shared__ unsigned char smem_raw[];
  const long long n_state = (long long)h * dk * dv;
  double* S = reinterpret_cast<double*>(smem_raw);  // [h][dk][dv]
  double* part = S + n_state;                       // [blockDim.x]
  const long long pert = first + blockIdx.x;
  const long long p_idx = pert >> 1;
  const double bump = (pert & 1) ? -step : step;  // even: base + step, odd: base - step
  for (long long e = threadIdx.x; e < n_state; e += blockDim.x) S[e] = 0.0;
  double acc = 0.0;
  __syncthreads();
  for (long long t = 0; t < L; ++t) {
    for (long long e = threadIdx.x; e < n_state; e += blockDim.x) {
      const int j = (int)(e % dv);
      const int c = (int)((e / dv) % dk);
      const int hh = (int)(e / ((long long)dk * dv));
      const long long ik = ((long long)hh * L + t) * dk + c, iv = ((long long)hh * L + t) * dv + j;
      const double a = exp(fd_val(g, 3, ik, p_which, p_idx, bump));
      const double kv = __dmul_rn(fd_val(k, 1, ik, p_which, p_idx, bump), fd_val(v, 2, iv, p_which, p_idx, bump));
      S[e] = __dadd_rn(__dmul_rn(a, S[e]), kv);
    }
    __syncthreads();
    for (long long pj = threadIdx.x; pj < (long long)h * dv; pj += blockDim.x) {
      const int hh = (int)(pj / dv), j = (int)(pj % dv);
      const long long iq = ((long long)hh * L + t) * dk, io = ((long long)hh * L + t) * dv + j;
      double ot = 0.0;
      for (int c = 0; c < dk; ++c)
        ot = __dadd_rn(ot, __dmul_rn(fd_val(q, 0, iq + c, p_which, p_idx, bump), S[((long long)hh * dk + c) * dv + j]));
      acc = __dadd_rn(acc, __dmul_rn(probe[io], ot));
    }
    __syncthreads();
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = part[0];
    for (int i = 1; i < (int)blockDim.x; ++i) tot = __dadd_rn(tot, part[i]);
    losses[blockIdx.x] = tot;
  }
}

template <typename Tin, typename Ta>
int launch_recurrent(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                     const void* init, void* o, void* bounds, void* final_state, cudaStream_t st) {
  const int dk = s->key_dim, dv = s->value_dim;
  if (dk > 1024) return ZGLA_ERR_UNSUPPORTED;
  const int J = std::max(1, std::min(dv, 256 / dk));
  const int threads = dk * J;
  const size_t smem = 2ull * dk * J * sizeof(Ta);
  dim3 grid((unsigned)s->heads, (unsigned)((dv + J - 1) / J));
  recurrent_kernel<Tin, Ta><<<grid, threads, smem, st>>>(
      s->heads, s->seq_len, dk, dv, s->chunk_len, J, (const Tin*)q, (const Tin*)k, (const Tin*)v, (const Ta*)g,
      (const Ta*)init, (Tin*)o, (Ta*)bounds, (Ta*)final_state);
  return zgla_check_launch();
}

}  // namespace recur
}  // namespace zgla

using namespace zgla::recur;

extern "C" int zgla_recurrent_forward(const zgla_shape* s, const void* q, const void* k, const void* v,
                                      const void* g, const void* init, void* o, void* bounds, void* final_state,
                                      void* stream) {
  if (!s || s->heads < 1 || s->key_dim < 1 || s->value_dim < 1 || s->seq_len < 1 || s->chunk_len < 1 ||
      s->seq_len % s->chunk_len || !q || !k || !v || !g || !o)
    return ZGLA_ERR_DIMS;
  cudaStream_t st = (cudaStream_t)stream;
  switch (s->dtype) {
    case ZGLA_F64: return launch_recurrent<double, double>(s, q, k, v, g, init, o, bounds, final_state, st);
    case ZGLA_F32: return launch_recurrent<float, float>(s, q, k, v, g, init, o, bounds, final_state, st);
    case ZGLA_BF16: return launch_recurrent<__nv_bfloat16, float>(s, q, k, v, g, init, o, bounds, final_state, st);
    default: return ZGLA_ERR_CONFIG;
  }
}

extern "C" long long zgla_fd_max_state(void) { return (200 * 1024 - 256 * 8) / 8; }

extern "C" int zgla_fd_losses(const zgla_shape* s, const double* q, const double* k, const double* v,
                              const double* g, const double* probe, int which, long long first, long long count,
                              double step, double* losses, void* stream) {
  if (!s || s->heads < 1 || s->key_dim < 1 || s->value_dim < 1 || s->seq_len < 1 || which < 0 || which > 3 ||
      first < 0 || count < 0 || !q || !k || !v || !g || !probe || !losses)
    return ZGLA_ERR_DIMS;
  if (s->dtype != ZGLA_F64) return ZGLA_ERR_CONFIG;
  if (!(step > 0.0)) return ZGLA_ERR_DOMAIN;
  const long long n_state = (long long)s->heads * s->key_dim * s->value_dim;
  if (n_state > zgla_fd_max_state()) return ZGLA_ERR_UNSUPPORTED;
  const int threads = 256;
  const size_t smem = (size_t)(n_state + threads) * sizeof(double);
  if (smem > 48 * 1024) {
    if (cudaError_t e = cudaFuncSetAttribute(fd_loss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
      return zgla::cuda_fail(e, "zgla_fd_losses");
  }
  for (long long done = 0; done < count;) {
    const long long n = std::min<long long>(count - done, 65535);
    fd_loss_kernel<<<(unsigned)n, threads, smem, (cudaStream_t)stream>>>(
        s->heads, s->seq_len, s->key_dim, s->value_dim, q, k, v, g, probe, which, first + done, step,
        losses + done);
    if (int rc = zgla_check_launch()) return rc;
    done += n;
  }
  return ZGLA_OK;
}
