// Internal helpers shared by the CUDA translation units.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/zeco_gla.h"

namespace zgla {

void set_error(const char* msg);
extern unsigned long long* g_trace_buf;  // zgla_set_trace (diagnostics)
extern int g_trace_cta;
int cuda_fail(cudaError_t e, const char* where);

template <typename T>
struct Acc {
  using type = float;
};
template <>
struct Acc<double> {
  using type = double;
};

__device__ __forceinline__ float ld_in(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_in(const float* p) { return *p; }
__device__ __forceinline__ double ld_in(const double* p) { return *p; }
__device__ __forceinline__ void st_out(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }
__device__ __forceinline__ void st_out(float* p, float x) { *p = x; }
__device__ __forceinline__ void st_out(double* p, double x) { *p = x; }
__device__ __forceinline__ float ex(float x) { return expf(x); }
__device__ __forceinline__ double ex(double x) { return exp(x); }

}  // namespace zgla

extern "C" int zgla_check_launch_impl(const char* where);
#define zgla_check_launch() zgla_check_launch_impl(__func__)
