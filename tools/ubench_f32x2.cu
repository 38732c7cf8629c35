// Microbenchmark: issue/throughput of scalar FP32 (FADD/FFMA) vs packed FP32x2 (FADD2/FFMA2) on
// sm_100a.  Each thread runs 8 independent dependency chains; reports Gop/s (scalar lanes).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float2 a) { return *reinterpret_cast<u64*>(&a); }
__device__ __forceinline__ float2 upk(u64 a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  u64 r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return upk(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  u64 r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return upk(r);
}
constexpr int IT = 4096, CH = 8;
__global__ void k_ffma(float* out, float s) {
  float a[CH];
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fmaf(a[c], s, 0.5f);
  float t = 0;
  for (int c = 0; c < CH; ++c) t += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma2(float* out, float s) {
  float2 a[CH];
  for (int c = 0; c < CH; ++c) a[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  const float2 s2 = make_float2(s, s), h = make_float2(0.5f, 0.5f);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fma2(a[c], s2, h);
  float t = 0;
  for (int c = 0; c < CH; ++c) t += a[c].x + a[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_fadd(float* out, float s) {
  float a[CH];
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] + s;
  float t = 0;
  for (int c = 0; c < CH; ++c) t += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_fadd2(float* out, float s) {
  float2 a[CH];
  for (int c = 0; c < CH; ++c) a[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  const float2 s2 = make_float2(s, s);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = add2(a[c], s2);
  float t = 0;
  for (int c = 0; c < CH; ++c) t += a[c].x + a[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
// mixed: one FFMA2 + one integer op per step (does the packed op co-issue with ALU work?)
int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * 8, threads = 256;
  float* out;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct K { const char* n; void (*f)(float*, float); double lanes; };
  K ks[] = {{"FFMA", k_ffma, 1}, {"FFMA2", k_ffma2, 2}, {"FADD", k_fadd, 1}, {"FADD2", k_fadd2, 2}};
  for (auto& k : ks) {
    k.f<<<blocks, threads>>>(out, 0.999f);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k.f<<<blocks, threads>>>(out, 0.999f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double instr = 5.0 * blocks * threads * (double)IT * CH;  // thread-instructions
    printf("%-6s %8.1f G thread-instr/s  %8.1f G lane-ops/s  (%.3f ms)\n", k.n, instr / ms / 1e6,
           instr * k.lanes / ms / 1e6, ms / 5);
  }
  return 0;
}
