// Issue-rate probe: legacy warp-level mma.sync m16n8k8 TF32 against FFMA on
// sm_100a.  Decides whether a register-fragment 3xTF32 contraction can beat
// the FP32 CUDA-core chunk GEMMs of the subspace SVT.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mma_rate mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void k_mma(float* out, int iters) {
  float c[ACC][4];
  for (int a = 0; a < ACC; ++a)
    for (int i = 0; i < 4; ++i) c[a][i] = 0.f;
  unsigned a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = threadIdx.x * 5, a3 = threadIdx.x * 7;
  unsigned b0 = threadIdx.x * 11, b1 = threadIdx.x * 13;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int a = 0; a < ACC; ++a)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[a][0]), "+f"(c[a][1]), "+f"(c[a][2]), "+f"(c[a][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int a = 0; a < ACC; ++a)
    for (int i = 0; i < 4; ++i) s += c[a][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 8 independent mma.sync per iteration interleaved with NALU independent
// ALU instructions (FADD / LOP3 chains on other registers): does the legacy
// HMMA path leave the issue port free for other work?
template <int NALU>
__global__ void k_mix(float* out, int iters) {
  float c[8][4];
  for (int a = 0; a < 8; ++a)
    for (int i = 0; i < 4; ++i) c[a][i] = 0.f;
  unsigned a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = threadIdx.x * 5, a3 = threadIdx.x * 7;
  unsigned b0 = threadIdx.x * 11, b1 = threadIdx.x * 13;
  float f[16];
  unsigned u[16];
  for (int i = 0; i < 16; ++i) { f[i] = (float)threadIdx.x + i; u[i] = threadIdx.x * (i + 17); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[a][0]), "+f"(c[a][1]), "+f"(c[a][2]), "+f"(c[a][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
#pragma unroll
      for (int k = 0; k < NALU / 8; ++k) {
        const int j = (a * (NALU / 8) + k) & 15;
        if (k & 1) asm volatile("add.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(1.0f));
        else asm volatile("lop3.b32 %0, %0, %1, 0x55, 0x96;" : "+r"(u[j]) : "r"(0x9e3779b9u));
      }
    }
  }
  float s = 0.f;
  for (int a = 0; a < 8; ++a)
    for (int i = 0; i < 4; ++i) s += c[a][i];
  for (int i = 0; i < 16; ++i) s += f[i] + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NALU>
void run_mix(float* out, int sms, cudaEvent_t e0, cudaEvent_t e1) {
  const int iters = 20000;
  for (int warps : {4, 12, 16}) {
    float ms;
    k_mix<NALU><<<sms, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    k_mix<NALU><<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * 1.965e9 / iters;  // cycles per iteration (8 mma + NALU alu per warp)
    printf("mix: %2d warps/SM, 8 mma + %3d alu per iteration: %.1f cycles/iteration/SM  (%.2f per warp-iteration per SMSP)\n", warps,
           NALU, cyc, cyc / ((warps + 3) / 4));
  }
}

template <int ACC>
__global__ void k_ffma(float* out, int iters, float x, float y) {
  float c[ACC];
  for (int a = 0; a < ACC; ++a) c[a] = (float)a;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int a = 0; a < ACC; ++a) c[a] = fmaf(c[a], x, y);
  }
  float s = 0.f;
  for (int a = 0; a < ACC; ++a) s += c[a];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    const int nt = warps * 32;
    float ms;
    k_mma<8><<<sms, nt>>>(out, 100);
    cudaEventRecord(e0);
    k_mma<8><<<sms, nt>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = (double)sms * warps * iters * 8;
    const double tf = mmas * 16 * 8 * 8 * 2 / (ms * 1e-3) / 1e12;
    printf("mma.sync m16n8k8 tf32: %2d warps/SM  %.3f ms  %.1f TFLOP/s dense  (%.2f mma/clk/SM at 1.965 GHz)\n", warps, ms,
           tf, mmas / sms / (ms * 1e-3 * 1.965e9));
    k_ffma<16><<<sms, nt>>>(out, 100, 1.0001f, 0.5f);
    cudaEventRecord(e0);
    k_ffma<16><<<sms, nt>>>(out, iters, 1.0001f, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f = (double)sms * nt * iters * 16 * 2;
    printf("ffma:                   %2d warps/SM  %.3f ms  %.1f TFLOP/s\n", warps, ms, f / (ms * 1e-3) / 1e12);
  }
  run_mix<0>(out, sms, e0, e1);
  run_mix<16>(out, sms, e0, e1);
  run_mix<32>(out, sms, e0, e1);
  run_mix<64>(out, sms, e0, e1);
  run_mix<128>(out, sms, e0, e1);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
