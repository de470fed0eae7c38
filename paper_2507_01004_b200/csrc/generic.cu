// Generic (SIMT) GLA kernels: any head dims / chunk length, fp32 or fp64
// accumulation, bf16 / fp32 / fp64 tensors.  These serve the reference's
// function-level API (glasp/gla.py) and the fp32 / fp64 validation modes of
// the ZeCO entry points.  The fused tcgen05 kernels in fast_fwd.cu /
// fast_bwd.cu serve the bf16 ZeCO hot path.
//
// Work decomposition mirrors the reference's chunk structure
// (glasp/gla.py:248-444): per-chunk contributions in parallel over
// (head, chunk, state element), then a scan over chunks in parallel over state
// elements, then per-chunk outputs / gradients in parallel over (head, chunk).
// Inside a chunk the kernels walk tokens with the exact recurrence
// S_t = e^{g_t} (.) S_{t-1} + k_t^T v_t (no factorised exponentials, so any
// strictly negative gate is safe).
#include <cstdio>

#include "zgla_internal.h"

namespace zgla {
namespace generic {

struct Dims {
  int h, dk, dv, C;
  long long L, N;
};

__device__ __forceinline__ long long tok_off(const Dims& d, int hh, long long t, int width) {
  return ((long long)hh * d.L + t) * width;
}

// (1) per-chunk contribution from a zero state: states[n+1] <- KV_n, gam[n] <- sum of g over chunk n
template <typename Tin, typename Ta>
__global__ void chunk_kv_kernel(Dims d, const Tin* __restrict__ k, const Tin* __restrict__ v,
                                const Ta* __restrict__ g, Ta* __restrict__ states, Ta* __restrict__ gam) {
  const int nel = d.dk * d.dv;
  const long long per_chunk = (nel + blockDim.x - 1) / blockDim.x;
  const long long b = blockIdx.x;
  const int hh = (int)(b / (d.N * per_chunk));
  const long long n = (b / per_chunk) % d.N;
  const int e = (int)(b % per_chunk) * blockDim.x + threadIdx.x;
  if (e >= nel) return;
  const int c = e / d.dv, j = e % d.dv;
  const long long t0 = n * d.C;
  Ta s = 0, gs = 0;
  for (int t = 0; t < d.C; ++t) {
    const Ta gt = g[tok_off(d, hh, t0 + t, d.dk) + c];
    s = ex(gt) * s + (Ta)ld_in(k + tok_off(d, hh, t0 + t, d.dk) + c) * (Ta)ld_in(v + tok_off(d, hh, t0 + t, d.dv) + j);
    gs += gt;
  }
  states[((n + 1) * d.h + hh) * nel + e] = s;
  if (j == 0) gam[(n * d.h + hh) * d.dk + c] = gs;
}

// (2) scan over chunks: states[n+1] = e^{gam_n} states[n] + KV_n (in place), cum[n+1] = cum[n] + gam_n
template <typename Ta>
__global__ void state_scan_kernel(Dims d, const Ta* __restrict__ init, Ta* __restrict__ states,
                                  Ta* __restrict__ cum, const Ta* __restrict__ gam) {
  const int nel = d.dk * d.dv;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)d.h * nel) return;
  const int hh = (int)(idx / nel), e = (int)(idx % nel), c = e / d.dv, j = e % d.dv;
  Ta s = init ? init[idx] : (Ta)0;
  states[(long long)hh * nel + e] = s;
  for (long long n = 0; n < d.N; ++n) {
    Ta* p = states + ((n + 1) * d.h + hh) * nel + e;
    s = ex(gam[(n * d.h + hh) * d.dk + c]) * s + *p;
    *p = s;
  }
  if (j == 0 && cum) {
    Ta cm = 0;
    cum[(long long)hh * d.dk + c] = 0;
    for (long long n = 0; n < d.N; ++n) {
      cm += gam[(n * d.h + hh) * d.dk + c];
      cum[((n + 1) * d.h + hh) * d.dk + c] = cm;
    }
  }
}

// (3) outputs of one chunk from its (lifted) start state, token recurrence
template <typename Tin, typename Ta>
__global__ void chunk_out_kernel(Dims d, const Tin* __restrict__ q, const Tin* __restrict__ k,
                                 const Tin* __restrict__ v, const Ta* __restrict__ g, const Ta* __restrict__ states,
                                 const Ta* __restrict__ cum, const Ta* __restrict__ prev, Tin* __restrict__ o) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ta* S = reinterpret_cast<Ta*>(smem_raw);  // [dk][dv]
  Ta* qs = S + d.dk * d.dv;
  Ta* ks = qs + d.dk;
  Ta* as = ks + d.dk;
  Ta* vs = as + d.dk;
  const int hh = (int)(blockIdx.x / d.N);
  const long long n = blockIdx.x % d.N;
  const int nel = d.dk * d.dv, tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < nel; e += nt) {
    Ta s = states[(n * d.h + hh) * nel + e];
    if (prev) s += ex(cum[(n * d.h + hh) * d.dk + e / d.dv]) * prev[(long long)hh * nel + e];
    S[e] = s;
  }
  for (int t = 0; t < d.C; ++t) {
    const long long tok = n * d.C + t;
    for (int c = tid; c < d.dk; c += nt) {
      qs[c] = ld_in(q + tok_off(d, hh, tok, d.dk) + c);
      ks[c] = ld_in(k + tok_off(d, hh, tok, d.dk) + c);
      as[c] = ex(g[tok_off(d, hh, tok, d.dk) + c]);
    }
    for (int j = tid; j < d.dv; j += nt) vs[j] = ld_in(v + tok_off(d, hh, tok, d.dv) + j);
    __syncthreads();
    for (int e = tid; e < nel; e += nt) {
      const int c = e / d.dv, j = e % d.dv;
      S[e] = as[c] * S[e] + ks[c] * vs[j];
    }
    __syncthreads();
    for (int j = tid; j < d.dv; j += nt) {
      Ta acc = 0;
      for (int c = 0; c < d.dk; ++c) acc += qs[c] * S[c * d.dv + j];
      st_out(o + tok_off(d, hh, tok, d.dv) + j, acc);
    }
    __syncthreads();
  }
}

// (4) per-chunk state cotangent from the chunk's own outputs: QDO_n = sum_t e^{logb_t} q_t^T dO_t
template <typename Tin, typename Ta>
__global__ void rev_chunk_kernel(Dims d, const Tin* __restrict__ q, const Ta* __restrict__ g,
                                 const Tin* __restrict__ dout, Ta* __restrict__ rev, Ta* __restrict__ gam) {
  const int nel = d.dk * d.dv;
  const long long per_chunk = (nel + blockDim.x - 1) / blockDim.x;
  const long long b = blockIdx.x;
  const int hh = (int)(b / (d.N * per_chunk));
  const long long n = (b / per_chunk) % d.N;
  const int e = (int)(b % per_chunk) * blockDim.x + threadIdx.x;
  if (e >= nel) return;
  const int c = e / d.dv, j = e % d.dv;
  const long long t0 = n * d.C;
  Ta acc = 0, gs = 0;
  for (int t = d.C - 1; t >= 0; --t) {
    const Ta gt = g[tok_off(d, hh, t0 + t, d.dk) + c];
    acc = ex(gt) * (acc + (Ta)ld_in(q + tok_off(d, hh, t0 + t, d.dk) + c) *
                              (Ta)ld_in(dout + tok_off(d, hh, t0 + t, d.dv) + j));
    gs += gt;
  }
  rev[(n * d.h + hh) * nel + e] = acc;
  if (j == 0) gam[(n * d.h + hh) * d.dk + c] = gs;
}

// (5) right-to-left scan: rev[N] = seed, rev[n] = e^{gam_n} rev[n+1] + QDO_n (in place)
template <typename Ta>
__global__ void rev_scan_kernel(Dims d, const Ta* __restrict__ seed, Ta* __restrict__ rev,
                                const Ta* __restrict__ gam) {
  const int nel = d.dk * d.dv;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)d.h * nel) return;
  const int hh = (int)(idx / nel), e = (int)(idx % nel), c = e / d.dv;
  Ta s = seed ? seed[idx] : (Ta)0;
  rev[(d.N * d.h + hh) * nel + e] = s;
  for (long long n = d.N - 1; n >= 0; --n) {
    Ta* p = rev + (n * d.h + hh) * nel + e;
    s = ex(gam[(n * d.h + hh) * d.dk + c]) * s + *p;
    *p = s;
  }
}

// (6) gradients of one chunk.  Forward token walk from the lifted start state gives dq and
// the chunk-end state; reverse walk from the lifted end cotangent gives dk, dv and
// dg_t = sum_{t'>=t in chunk}(q.dq - k.dk) + rowsum(S_end (.) dS_end)  (the chunk-local form
// of glasp/gla.py:438-443: the suffix sum beyond the chunk equals the boundary rowsum).
template <typename Tin, typename Ta>
__global__ void chunk_bwd_kernel(Dims d, const Tin* __restrict__ q, const Tin* __restrict__ k,
                                 const Tin* __restrict__ v, const Ta* __restrict__ g, const Tin* __restrict__ dout,
                                 const Ta* __restrict__ states, const Ta* __restrict__ cum,
                                 const Ta* __restrict__ prev, const Ta* __restrict__ rev,
                                 const Ta* __restrict__ ds_next, Tin* __restrict__ dq, Tin* __restrict__ dk,
                                 Tin* __restrict__ dv, Ta* __restrict__ dg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = d.dv + 1;
  Ta* S = reinterpret_cast<Ta*>(smem_raw);  // [dk][dv+1]: forward state, then reused for the cotangent
  Ta* D = S;
  Ta* dqs = S + d.dk * ld;                  // [C][dk]
  Ta* qs = dqs + d.C * d.dk;
  Ta* ks = qs + d.dk;
  Ta* as = ks + d.dk;
  Ta* tail = as + d.dk;
  Ta* vs = tail + d.dk;
  Ta* dos = vs + d.dv;
  const int hh = (int)(blockIdx.x / d.N);
  const long long n = blockIdx.x % d.N;
  const int nel = d.dk * d.dv, tid = threadIdx.x, nt = blockDim.x;
  const Ta* cumN = cum + (d.N * d.h + hh) * d.dk;
  // lifted end-of-chunk cotangent dS_{n+1} = rev[n+1] + e^{cum_N - cum_{n+1}} ds_next (glasp/gla.py:393-394)
  auto dend = [&](int c, int j) -> Ta {
    const long long e = (long long)c * d.dv + j;
    Ta r = rev[((n + 1) * d.h + hh) * nel + e];
    if (ds_next) r += ex(cumN[c] - cum[((n + 1) * d.h + hh) * d.dk + c]) * ds_next[(long long)hh * nel + e];
    return r;
  };
  for (int e = tid; e < nel; e += nt) {
    const int c = e / d.dv, j = e % d.dv;
    Ta s = states[(n * d.h + hh) * nel + e];
    if (prev) s += ex(cum[(n * d.h + hh) * d.dk + c]) * prev[(long long)hh * nel + e];
    S[c * ld + j] = s;
  }
  __syncthreads();
  // forward walk: dq_t = dO_t S_t^T
  for (int t = 0; t < d.C; ++t) {
    const long long tok = n * d.C + t;
    for (int c = tid; c < d.dk; c += nt) {
      ks[c] = ld_in(k + tok_off(d, hh, tok, d.dk) + c);
      as[c] = ex(g[tok_off(d, hh, tok, d.dk) + c]);
    }
    for (int j = tid; j < d.dv; j += nt) {
      vs[j] = ld_in(v + tok_off(d, hh, tok, d.dv) + j);
      dos[j] = ld_in(dout + tok_off(d, hh, tok, d.dv) + j);
    }
    __syncthreads();
    for (int e = tid; e < nel; e += nt) {
      const int c = e / d.dv, j = e % d.dv;
      S[c * ld + j] = as[c] * S[c * ld + j] + ks[c] * vs[j];
    }
    __syncthreads();
    for (int c = tid; c < d.dk; c += nt) {
      Ta acc = 0;
      for (int j = 0; j < d.dv; ++j) acc += dos[j] * S[c * ld + j];
      dqs[t * d.dk + c] = acc;
      st_out(dq + tok_off(d, hh, tok, d.dk) + c, acc);
    }
    __syncthreads();
  }
  // boundary term rowsum(S_{n+1} (.) dS_{n+1})
  for (int c = tid; c < d.dk; c += nt) {
    Ta acc = 0;
    for (int j = 0; j < d.dv; ++j) acc += S[c * ld + j] * dend(c, j);
    tail[c] = acc;
  }
  __syncthreads();
  for (int e = tid; e < nel; e += nt) {
    const int c = e / d.dv, j = e % d.dv;
    D[c * ld + j] = dend(c, j);
  }
  __syncthreads();
  // reverse walk
  for (int t = d.C - 1; t >= 0; --t) {
    const long long tok = n * d.C + t;
    for (int c = tid; c < d.dk; c += nt) {
      qs[c] = ld_in(q + tok_off(d, hh, tok, d.dk) + c);
      ks[c] = ld_in(k + tok_off(d, hh, tok, d.dk) + c);
      as[c] = ex(g[tok_off(d, hh, tok, d.dk) + c]);
    }
    for (int j = tid; j < d.dv; j += nt) {
      vs[j] = ld_in(v + tok_off(d, hh, tok, d.dv) + j);
      dos[j] = ld_in(dout + tok_off(d, hh, tok, d.dv) + j);
    }
    __syncthreads();
    for (int e = tid; e < nel; e += nt) {
      const int c = e / d.dv, j = e % d.dv;
      D[c * ld + j] += qs[c] * dos[j];
    }
    __syncthreads();
    for (int c = tid; c < d.dk; c += nt) {
      Ta acc = 0;
      for (int j = 0; j < d.dv; ++j) acc += D[c * ld + j] * vs[j];
      st_out(dk + tok_off(d, hh, tok, d.dk) + c, acc);
      tail[c] += qs[c] * dqs[t * d.dk + c] - ks[c] * acc;
      dg[tok_off(d, hh, tok, d.dk) + c] = tail[c];
    }
    for (int j = tid; j < d.dv; j += nt) {
      Ta acc = 0;
      for (int c = 0; c < d.dk; ++c) acc += ks[c] * D[c * ld + j];
      st_out(dv + tok_off(d, hh, tok, d.dv) + j, acc);
    }
    __syncthreads();
    for (int e = tid; e < nel; e += nt) {
      const int c = e / d.dv, j = e % d.dv;
      D[c * ld + j] *= as[c];
    }
    __syncthreads();
  }
}

template <typename Ta>
__global__ void global_correct_kernel(long long n_states, int h, int dk, int dv, const Ta* __restrict__ states,
                                      const Ta* __restrict__ cum, const Ta* __restrict__ prev, Ta* __restrict__ out) {
  const long long nel = (long long)h * dk * dv;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_states * nel) return;
  const long long n = idx / nel, r = idx % nel;
  const long long hc = r / dv;  // (hh*dk + c)
  out[idx] = ex(cum[n * h * dk + hc]) * prev[r] + states[idx];
}

template <typename Ta>
__global__ void revcum_kernel(int h, long long L, int width, const Ta* __restrict__ x, Ta* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)h * width) return;
  const int hh = (int)(idx / width), c = (int)(idx % width);
  Ta acc = 0;
  for (long long t = L - 1; t >= 0; --t) {
    const long long o = ((long long)hh * L + t) * width + c;
    acc += x[o];
    out[o] = acc;
  }
}

template <typename Ta>
__global__ void chunk_scalings_kernel(int h, int C, int dk, const Ta* __restrict__ g, Ta* __restrict__ decay,
                                      Ta* __restrict__ from_start, Ta* __restrict__ to_end) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= h * dk) return;
  const int hh = idx / dk, c = idx % dk;
  Ta tot = 0;
  for (int t = 0; t < C; ++t) tot += g[((long long)hh * C + t) * dk + c];
  Ta lb = 0;
  for (int t = 0; t < C; ++t) {
    const long long o = ((long long)hh * C + t) * dk + c;
    lb += g[o];
    from_start[o] = ex(lb);
    to_end[o] = ex(tot - lb);
  }
  decay[idx] = ex(tot);
}

template <typename Ta>
__global__ void check_log_decay_kernel(long long n, const Ta* __restrict__ g, int* bad) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  int b = 0;
  for (; i < n; i += stride) {
    const Ta x = g[i];
    if (!(x < (Ta)0) || !isfinite(x)) b = 1;
  }
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

// ---------------------------------------------------------------- host side

template <typename Ta>
struct Ws {
  Ta *states, *rev, *cum, *gam;
};

template <typename Ta>
Ws<Ta> carve(const Dims& d, void* ws) {
  Ws<Ta> w;
  const long long st = (d.N + 1) * d.h * d.dk * d.dv;
  w.states = reinterpret_cast<Ta*>(ws);
  w.rev = w.states + st;
  w.cum = w.rev + st;
  w.gam = w.cum + (d.N + 1) * d.h * d.dk;
  return w;
}

long long ws_bytes(const zgla_shape* s) {
  const long long N = s->seq_len / s->chunk_len;
  const long long st = (N + 1) * s->heads * (long long)s->key_dim * s->value_dim;
  const long long vec = (2 * N + 1) * s->heads * (long long)s->key_dim;
  return (2 * st + vec) * (s->dtype == ZGLA_F64 ? 8 : 4);
}

static inline unsigned blocks_for(long long n, int t) { return (unsigned)((n + t - 1) / t); }

template <typename Tin, typename Ta>
int local_scan(const Dims& d, const void* k, const void* v, const void* g, const void* init, Ta* states, Ta* cum,
               Ta* gam, cudaStream_t st) {
  const int nel = d.dk * d.dv;
  const long long per_chunk = (nel + 127) / 128;
  chunk_kv_kernel<Tin, Ta><<<(unsigned)(d.h * d.N * per_chunk), 128, 0, st>>>(
      d, (const Tin*)k, (const Tin*)v, (const Ta*)g, states, gam);
  state_scan_kernel<Ta><<<blocks_for((long long)d.h * nel, 128), 128, 0, st>>>(d, (const Ta*)init, states, cum, gam);
  return zgla_check_launch();
}

template <typename Tin, typename Ta>
int outputs(const Dims& d, const void* q, const void* k, const void* v, const void* g, const Ta* states,
            const Ta* cum, const Ta* prev, void* o, cudaStream_t st) {
  const size_t smem = ((size_t)d.dk * d.dv + 3 * d.dk + d.dv) * sizeof(Ta);
  if (smem > 220 * 1024) return ZGLA_ERR_UNSUPPORTED;
  cudaFuncSetAttribute(chunk_out_kernel<Tin, Ta>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chunk_out_kernel<Tin, Ta><<<(unsigned)(d.h * d.N), 256, smem, st>>>(d, (const Tin*)q, (const Tin*)k,
                                                                       (const Tin*)v, (const Ta*)g, states, cum,
                                                                       prev, (Tin*)o);
  return zgla_check_launch();
}

template <typename Tin, typename Ta>
int rev_scan(const Dims& d, const void* q, const void* g, const void* dout, const void* seed, Ta* rev, Ta* gam,
             cudaStream_t st) {
  const int nel = d.dk * d.dv;
  const long long per_chunk = (nel + 127) / 128;
  rev_chunk_kernel<Tin, Ta><<<(unsigned)(d.h * d.N * per_chunk), 128, 0, st>>>(d, (const Tin*)q, (const Ta*)g,
                                                                                (const Tin*)dout, rev, gam);
  rev_scan_kernel<Ta><<<blocks_for((long long)d.h * nel, 128), 128, 0, st>>>(d, (const Ta*)seed, rev, gam);
  return zgla_check_launch();
}

template <typename Tin, typename Ta>
int chunk_bwd(const Dims& d, const void* q, const void* k, const void* v, const void* g, const void* dout,
              const Ta* states, const Ta* cum, const Ta* prev, const Ta* rev, const Ta* ds_next, void* dq, void* dk,
              void* dv, void* dg, cudaStream_t st) {
  const size_t smem = ((size_t)d.dk * (d.dv + 1) + (size_t)d.C * d.dk + 4 * d.dk + 2 * d.dv) * sizeof(Ta);
  if (smem > 220 * 1024) return ZGLA_ERR_UNSUPPORTED;
  cudaFuncSetAttribute(chunk_bwd_kernel<Tin, Ta>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chunk_bwd_kernel<Tin, Ta><<<(unsigned)(d.h * d.N), 256, smem, st>>>(
      d, (const Tin*)q, (const Tin*)k, (const Tin*)v, (const Ta*)g, (const Tin*)dout, states, cum, prev, rev,
      ds_next, (Tin*)dq, (Tin*)dk, (Tin*)dv, (Ta*)dg);
  return zgla_check_launch();
}

// ----- dtype dispatch ------------------------------------------------------

Dims dims_of(const zgla_shape* s) {
  Dims d;
  d.h = s->heads;
  d.dk = s->key_dim;
  d.dv = s->value_dim;
  d.C = s->chunk_len;
  d.L = s->seq_len;
  d.N = s->seq_len / s->chunk_len;
  return d;
}

#define ZGLA_DISPATCH(s, FN, ...)                                              \
  ((s)->dtype == ZGLA_BF16  ? FN<__nv_bfloat16, float>(__VA_ARGS__)          \
   : (s)->dtype == ZGLA_F32 ? FN<float, float>(__VA_ARGS__)                  \
                            : FN<double, double>(__VA_ARGS__))

template <typename Tin, typename Ta>
int do_local_state_scan(const zgla_shape* s, const void* k, const void* v, const void* g, const void* init,
                        void* states, void* cum, void* ws, cudaStream_t st) {
  Dims d = dims_of(s);
  Ws<Ta> w = carve<Ta>(d, ws);
  return local_scan<Tin, Ta>(d, k, v, g, init, (Ta*)states, (Ta*)cum, w.gam, st);
}

template <typename Tin, typename Ta>
int do_forward_outputs(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                       const void* states, const void* cum, const void* prev, void* o, cudaStream_t st) {
  return outputs<Tin, Ta>(dims_of(s), q, k, v, g, (const Ta*)states, (const Ta*)cum, (const Ta*)prev, o, st);
}

template <typename Tin, typename Ta>
int do_reverse_boundary_scan(const zgla_shape* s, const void* q, const void* g, const void* dout,
                             const void* seed, void* rev, void* ws, cudaStream_t st) {
  Dims d = dims_of(s);
  Ws<Ta> w = carve<Ta>(d, ws);
  return rev_scan<Tin, Ta>(d, q, g, dout, seed, (Ta*)rev, w.gam, st);
}

template <typename Ta>
__global__ void lift_saved_kernel(Dims d, const Ta* __restrict__ saved, const Ta* __restrict__ gam,
                                  Ta* __restrict__ states, Ta* __restrict__ cum) {
  // copies saved local states into the workspace and rebuilds cum from gam
  const int nel = d.dk * d.dv;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)d.h * nel) return;
  const int hh = (int)(idx / nel), e = (int)(idx % nel), c = e / d.dv, j = e % d.dv;
  for (long long n = 0; n <= d.N; ++n) states[(n * d.h + hh) * nel + e] = saved[(n * d.h + hh) * nel + e];
  if (j == 0) {
    Ta cm = 0;
    cum[(long long)hh * d.dk + c] = 0;
    for (long long n = 0; n < d.N; ++n) {
      cm += gam[(n * d.h + hh) * d.dk + c];
      cum[((n + 1) * d.h + hh) * d.dk + c] = cm;
    }
  }
}

template <typename Ta>
__global__ void copy_last_kernel(long long count, const Ta* __restrict__ src, Ta* __restrict__ dst) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) dst[i] = src[i];
}

template <typename Tin, typename Ta>
int do_backward(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g, const void* dout,
                const void* prev, const void* ds_next, const void* saved, void* dq, void* dk, void* dv, void* dg,
                void* ds_boundary, void* ws, cudaStream_t st) {
  Dims d = dims_of(s);
  Ws<Ta> w = carve<Ta>(d, ws);
  int rc;
  if (saved) {
    // need only the chunk gammas: reuse the local-scan kernel's gamma output (KV lands in rev, overwritten below)
    const int nel = d.dk * d.dv;
    const long long per_chunk = (nel + 127) / 128;
    chunk_kv_kernel<Tin, Ta><<<(unsigned)(d.h * d.N * per_chunk), 128, 0, st>>>(d, (const Tin*)k, (const Tin*)v,
                                                                                 (const Ta*)g, w.rev, w.gam);
    lift_saved_kernel<Ta><<<blocks_for((long long)d.h * nel, 128), 128, 0, st>>>(d, (const Ta*)saved, w.gam,
                                                                                 w.states, w.cum);
    rc = zgla_check_launch();
  } else {
    rc = local_scan<Tin, Ta>(d, k, v, g, nullptr, w.states, w.cum, w.gam, st);
  }
  if (rc) return rc;
  rc = rev_scan<Tin, Ta>(d, q, g, dout, nullptr, w.rev, w.gam, st);
  if (rc) return rc;
  rc = chunk_bwd<Tin, Ta>(d, q, k, v, g, dout, w.states, w.cum, (const Ta*)prev, w.rev, (const Ta*)ds_next, dq, dk,
                          dv, dg, st);
  if (rc) return rc;
  if (ds_boundary) {
    // ds_boundary = rev[0] + e^{cum_N} ds_next  (glasp/gla.py:393-395 at n = 0)
    const long long nel = (long long)d.h * d.dk * d.dv;
    if (ds_next)
      global_correct_kernel<Ta><<<blocks_for(nel, 256), 256, 0, st>>>(1, d.h, d.dk, d.dv, w.rev,
                                                                       w.cum + d.N * d.h * d.dk, (const Ta*)ds_next,
                                                                       (Ta*)ds_boundary);
    else
      copy_last_kernel<Ta><<<blocks_for(nel, 256), 256, 0, st>>>(nel, w.rev, (Ta*)ds_boundary);
  }
  return zgla_check_launch();
}

// ZeCO entry points in the validation modes (and for bf16 shapes outside the fast path)
template <typename Tin, typename Ta>
int do_zeco_fwd_local(const zgla_shape* s, const void* k, const void* v, const void* g, void* ws, void* s_local,
                      void* g_tot, cudaStream_t st) {
  Dims d = dims_of(s);
  Ws<Ta> w = carve<Ta>(d, ws);
  int rc = local_scan<Tin, Ta>(d, k, v, g, nullptr, w.states, w.cum, w.gam, st);
  if (rc) return rc;
  const long long nel = (long long)d.h * d.dk * d.dv;
  copy_last_kernel<Ta><<<blocks_for(nel, 256), 256, 0, st>>>(nel, w.states + d.N * nel, (Ta*)s_local);
  copy_last_kernel<Ta><<<blocks_for((long long)d.h * d.dk, 256), 256, 0, st>>>((long long)d.h * d.dk,
                                                                                w.cum + d.N * d.h * d.dk, (Ta*)g_tot);
  return zgla_check_launch();
}

template <typename Tin, typename Ta>
int do_zeco_fwd_output(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g, void* ws,
                       const void* s_prev, void* o, cudaStream_t st) {
  Dims d = dims_of(s);
  Ws<Ta> w = carve<Ta>(d, ws);
  return outputs<Tin, Ta>(d, q, k, v, g, w.states, w.cum, (const Ta*)s_prev, o, st);
}

template <typename Tin, typename Ta>
int do_zeco_bwd_local(const zgla_shape* s, const void* q, const void* g, const void* dout, void* ws, void* ds0,
                      cudaStream_t st) {
  Dims d = dims_of(s);
  Ws<Ta> w = carve<Ta>(d, ws);
  int rc = rev_scan<Tin, Ta>(d, q, g, dout, nullptr, w.rev, w.gam, st);
  if (rc) return rc;
  const long long nel = (long long)d.h * d.dk * d.dv;
  copy_last_kernel<Ta><<<blocks_for(nel, 256), 256, 0, st>>>(nel, w.rev, (Ta*)ds0);
  return zgla_check_launch();
}

template <typename Tin, typename Ta>
int do_zeco_bwd_output(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                       const void* dout, void* ws, const void* s_prev, const void* ds_next, void* dq, void* dk,
                       void* dv, void* dg, cudaStream_t st) {
  Dims d = dims_of(s);
  Ws<Ta> w = carve<Ta>(d, ws);
  return chunk_bwd<Tin, Ta>(d, q, k, v, g, dout, w.states, w.cum, (const Ta*)s_prev, w.rev, (const Ta*)ds_next, dq,
                            dk, dv, dg, st);
}

}  // namespace generic
}  // namespace zgla

// ============================================================== C ABI (generic)
using namespace zgla;
using namespace zgla::generic;

static int validate(const zgla_shape* s) {
  if (!s || s->heads < 1 || s->key_dim < 1 || s->value_dim < 1 || s->seq_len < 1 || s->chunk_len < 1)
    return ZGLA_ERR_DIMS;
  if (s->seq_len % s->chunk_len) return ZGLA_ERR_DIMS;
  if (s->dtype < ZGLA_BF16 || s->dtype > ZGLA_F64) return ZGLA_ERR_CONFIG;
  return ZGLA_OK;
}

extern "C" long long zgla_workspace_bytes(const zgla_shape* s) {
  if (validate(s)) return -1;
  return ws_bytes(s);
}

extern "C" int zgla_local_state_scan(const zgla_shape* s, const void* k, const void* v, const void* g,
                                     const void* init, void* states_out, void* cum_out, void* ws, void* stream) {
  if (int rc = validate(s)) return rc;
  return ZGLA_DISPATCH(s, do_local_state_scan, s, k, v, g, init, states_out, cum_out, ws, (cudaStream_t)stream);
}

extern "C" int zgla_forward_outputs(const zgla_shape* s, const void* q, const void* k, const void* v,
                                    const void* g, const void* states, const void* cum, const void* prev, void* o,
                                    void* stream) {
  if (int rc = validate(s)) return rc;
  return ZGLA_DISPATCH(s, do_forward_outputs, s, q, k, v, g, states, cum, prev, o, (cudaStream_t)stream);
}

extern "C" int zgla_global_correct(const zgla_shape* s, int n_states, const void* states, const void* cum,
                                   const void* prev, void* out, void* stream) {
  if (!s || n_states < 1) return ZGLA_ERR_DIMS;
  const long long nel = (long long)n_states * s->heads * s->key_dim * s->value_dim;
  if (s->dtype == ZGLA_F64)
    global_correct_kernel<double><<<blocks_for(nel, 256), 256, 0, (cudaStream_t)stream>>>(
        n_states, s->heads, s->key_dim, s->value_dim, (const double*)states, (const double*)cum,
        (const double*)prev, (double*)out);
  else
    global_correct_kernel<float><<<blocks_for(nel, 256), 256, 0, (cudaStream_t)stream>>>(
        n_states, s->heads, s->key_dim, s->value_dim, (const float*)states, (const float*)cum, (const float*)prev,
        (float*)out);
  return zgla_check_launch();
}

extern "C" int zgla_reverse_boundary_scan(const zgla_shape* s, const void* q, const void* g, const void* d_out,
                                          const void* seed, void* rev_out, void* ws, void* stream) {
  if (int rc = validate(s)) return rc;
  return ZGLA_DISPATCH(s, do_reverse_boundary_scan, s, q, g, d_out, seed, rev_out, ws, (cudaStream_t)stream);
}

extern "C" int zgla_backward(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                             const void* d_out, const void* prev, const void* ds_next, const void* saved_states,
                             void* dq, void* dk, void* dv, void* dg, void* ds_boundary, void* ws, void* stream) {
  if (int rc = validate(s)) return rc;
  return ZGLA_DISPATCH(s, do_backward, s, q, k, v, g, d_out, prev, ds_next, saved_states, dq, dk, dv, dg,
                       ds_boundary, ws, (cudaStream_t)stream);
}

extern "C" int zgla_revcum(const zgla_shape* s, int d, const void* x, void* out, void* stream) {
  if (!s || d < 1 || s->seq_len < 1) return ZGLA_ERR_DIMS;
  const long long n = (long long)s->heads * d;
  if (s->dtype == ZGLA_F64)
    revcum_kernel<double><<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(s->heads, s->seq_len, d,
                                                                                 (const double*)x, (double*)out);
  else
    revcum_kernel<float><<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(s->heads, s->seq_len, d,
                                                                                (const float*)x, (float*)out);
  return zgla_check_launch();
}

extern "C" int zgla_chunk_scalings(const zgla_shape* s, const void* g_chunk, void* chunk_decay, void* from_start,
                                   void* to_end, void* stream) {
  if (!s || s->chunk_len < 1) return ZGLA_ERR_DIMS;
  const int n = s->heads * s->key_dim;
  if (s->dtype == ZGLA_F64)
    chunk_scalings_kernel<double><<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
        s->heads, s->chunk_len, s->key_dim, (const double*)g_chunk, (double*)chunk_decay, (double*)from_start,
        (double*)to_end);
  else
    chunk_scalings_kernel<float><<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
        s->heads, s->chunk_len, s->key_dim, (const float*)g_chunk, (float*)chunk_decay, (float*)from_start,
        (float*)to_end);
  return zgla_check_launch();
}

extern "C" int zgla_check_log_decay(long long n, int dtype, const void* g, int* bad_dev, void* stream) {
  if (n < 0) return ZGLA_ERR_DIMS;
  if (n == 0) return ZGLA_OK;
  const unsigned blocks = (unsigned)std::min<long long>(blocks_for(n, 256), 4 * 148);
  if (dtype == ZGLA_F64)
    check_log_decay_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(n, (const double*)g, bad_dev);
  else
    check_log_decay_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(n, (const float*)g, bad_dev);
  return zgla_check_launch();
}

// generic implementations of the ZeCO entry points (validation modes); the
// bf16 fast path in fast_*.cu takes precedence when it applies (see api.cu)
namespace zgla {
int generic_zeco_fwd_local(const zgla_shape* s, const void* k, const void* v, const void* g, void* ws, void* s_local,
                           void* g_tot, cudaStream_t st) {
  return ZGLA_DISPATCH(s, do_zeco_fwd_local, s, k, v, g, ws, s_local, g_tot, st);
}
int generic_zeco_fwd_output(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                            void* ws, const void* s_prev, void* o, cudaStream_t st) {
  return ZGLA_DISPATCH(s, do_zeco_fwd_output, s, q, k, v, g, ws, s_prev, o, st);
}
int generic_zeco_bwd_local(const zgla_shape* s, const void* q, const void* g, const void* dout, void* ws,
                           void* ds0, cudaStream_t st) {
  return ZGLA_DISPATCH(s, do_zeco_bwd_local, s, q, g, dout, ws, ds0, st);
}
int generic_zeco_bwd_output(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                            const void* dout, void* ws, const void* s_prev, const void* ds_next, void* dq, void* dk,
                            void* dv, void* dg, cudaStream_t st) {
  return ZGLA_DISPATCH(s, do_zeco_bwd_output, s, q, k, v, g, dout, ws, s_prev, ds_next, dq, dk, dv, dg, st);
}
long long generic_ws_bytes(const zgla_shape* s) { return ws_bytes(s); }
}  // namespace zgla
