// Shared device/host helpers for the SHLR B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace shlr_b200 {

// ---------------------------------------------------------------- errors
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line,
                  cudaGetErrorString(e));
    throw CudaError(buf);
  }
}
#define SHLR_CUDA(x) ::shlr_b200::cuda_check((x), #x, __FILE__, __LINE__)
#define SHLR_LAUNCH_CHECK() ::shlr_b200::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// --------------------------------------------------------------- complex
struct __align__(8) c32 {
  float x, y;
};

__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  return make_float2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) {
  return make_float2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) {
  return make_float2(a.x * s, a.y * s);
}
__host__ __device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// acc += a * b
__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
}

// --------------------------------------------------------------- helpers
__host__ __device__ __forceinline__ int dagger_src(int i, int n) {
  // virtual_coil_dagger (proj/src/hankel.cpp:99-113): out[i] = conj(v[(2 floor(n/2) + n - i) mod n])
  return (2 * (n / 2) + n - i) % n;
}

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    SHLR_CUDA(cudaGetDevice(&dev));
    SHLR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

}  // namespace shlr_b200
