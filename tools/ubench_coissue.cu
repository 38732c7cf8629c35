// Microbenchmark: does a packed FP32x2 instruction (FFMA2, 2 FMA-pipe cycles per warp) leave its
// second issue cycle to other pipes?  Interleaves FFMA2 (or FFMA) chains with integer ALU chains
// and with shared-memory loads; compares against each stream alone.
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
constexpr int IT = 2048, CH = 8;
template <int F, int A, int S>  // F: 0 none, 1 FFMA x2, 2 FFMA2; A: int ALU ops per step; S: LDS per step
__global__ void k(float* out, float s, int salt) {
  __shared__ float2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float2(i, i + 1);
  __syncthreads();
  float2 a[CH];
  unsigned u[CH];
  float2 l[CH];
  for (int c = 0; c < CH; ++c) {
    a[c] = make_float2(threadIdx.x * 1e-3f + c, c);
    u[c] = threadIdx.x * 7 + c + salt;
    l[c] = make_float2(0, 0);
  }
  const float2 s2 = make_float2(s, s), h = make_float2(0.5f, 0.5f);
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (F == 1) {
        a[c].x = fmaf(a[c].x, s, 0.5f);
        a[c].y = fmaf(a[c].y, s, 0.5f);
      }
      if (F == 2) a[c] = fma2(a[c], s2, h);
#pragma unroll
      for (int q = 0; q < A; ++q) asm volatile("lop3.b32 %0, %0, %1, 0x5a5a5a5a, 0x96;" : "+r"(u[c]) : "r"(u[(c + 1) % CH]));
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const float2 v = sm[(u[c] + q * 33 + i) & 1023];
        l[c].x += 0.f * v.x;  // keep the load live without an FP dependency chain on a[]
        asm volatile("" : "+f"(l[c].x));
      }
    }
  }
  float t = 0;
  for (int c = 0; c < CH; ++c) t += a[c].x + a[c].y + (float)u[c] + l[c].x;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int F, int A, int S>
void run(const char* name, float* out, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<F, A, S><<<blocks, threads>>>(out, 0.999f, 1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<F, A, S><<<blocks, threads>>>(out, 0.999f, r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double steps = 5.0 * blocks * threads / 32 * (double)IT * CH;  // warp-steps
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;  // SM cycles elapsed
  printf("%-28s %.3f ms/launch  %.3f SMSP-cycles per warp-step\n", name, ms / 5, cyc * nsm * 4 / steps);
}
int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * 8, threads = 256;
  float* out;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  run<1, 0, 0>("2x FFMA", out, blocks, threads);
  run<2, 0, 0>("1x FFMA2", out, blocks, threads);
  run<0, 2, 0>("2x LOP3", out, blocks, threads);
  run<1, 2, 0>("2x FFMA + 2x LOP3", out, blocks, threads);
  run<2, 2, 0>("1x FFMA2 + 2x LOP3", out, blocks, threads);
  run<2, 1, 0>("1x FFMA2 + 1x LOP3", out, blocks, threads);
  run<0, 0, 1>("1x LDS.64", out, blocks, threads);
  run<1, 0, 1>("2x FFMA + 1x LDS.64", out, blocks, threads);
  run<2, 0, 1>("1x FFMA2 + 1x LDS.64", out, blocks, threads);
  return 0;
}
