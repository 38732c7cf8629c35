// conv.cuh — pieces shared by the y / z passes (passes.cu) and the persistent 2D kernel
// (update.cu): twiddle tables, the three-component pass configuration, the Khat multiply and the
// K-Z / K-Y2D transform body (a3 of SURVEY §8(a); nz == 1: y forward . Khat . y inverse).
#pragma once
#include "common.cuh"
#include "regfft.cuh"

namespace mcq {

// twiddles of the y / z passes: the plan table of regfft.cuh (MCQ_REGTAB, default) or the base
// table tw[m] = exp(-2 pi i m / L)
constexpr int PASS_TWS = MCQ_REGTAB ? 0 : 1;
template <int L, int E>
__host__ __device__ constexpr int pass_twn() { return MCQ_REGTAB ? reg_tw_size<L, E>() : (L < 2 ? 2 : L); }
template <int L, int E, int NT>
__device__ __forceinline__ void pass_tw(float2* tw, const float2* __restrict__ gtw) {
  if constexpr (MCQ_REGTAB) {
    reg_tw_build<L, E, NT>(tw, gtw);
  } else {
#pragma unroll
    for (int j = 0; j < (L + NT - 1) / NT; ++j) {
      const int m = threadIdx.x + j * NT;
      if (m < L) tw[m] = gtw[m * (kTwMax / L)];
    }
  }
}

template <int L, int NTT = 256>
struct ZCfg {  // three-component passes with the Khat multiply (K-Z, K-Y2D); NTT: target threads
  static constexpr int E = L <= 16 ? L : 8;
  static constexpr int TL = L / E;
  static constexpr int C0 = NTT / TL;
  static constexpr int C = C0 < 4 ? 4 : (C0 > 64 ? 64 : C0);
  static constexpr int NT = C * TL;
  static constexpr int TWN = pass_twn<L, E>();
  static constexpr size_t SMEM = (size_t)(TWN + (TL > 1 ? 3 * L * C : 0)) * sizeof(float2);
};

// shared-memory address of (line l, position pos) for column c: [l][pos][c]
template <int L, int C>
struct ColAddr {
  int c;
  __device__ __forceinline__ int operator()(int l, int pos) const { return (l * L + pos) * C + c; }
};

// ---------------------------------------------------------------- Khat multiply
// Khat is real and stored folded and interleaved: [Lz/2+1][Ly/2+1][P][6]; off-diagonal components
// flip sign across the half axis they are odd in (XY: x,y; XZ: x,z; YZ: y,z).  kx is never folded.
__device__ __forceinline__ void khat_apply(const float* __restrict__ khat, const Dims& d, int kx, int ky, int kz,
                                           float2& mx, float2& my, float2& mz) {
  const int hy = d.Ly / 2, hz = d.Lz / 2;
  const int kyf = ky <= hy ? ky : d.Ly - ky;
  const int kzf = kz <= hz ? kz : d.Lz - kz;
  const float sy = ky <= hy ? 1.f : -1.f;
  const float sz = kz <= hz ? 1.f : -1.f;
  const unsigned b = (((unsigned)kzf * (hy + 1) + kyf) * d.kpitch + kx - d.kxoff) * 3;  // float2 index
  const float2* k2 = reinterpret_cast<const float2*>(khat) + b;
  const float2 k01 = __ldg(k2), k23 = __ldg(k2 + 1), k45 = __ldg(k2 + 2);
  const float kxx = k01.x, kyy = k01.y, kzz = k23.x;
  const float kxy = sy * k23.y;
  const float kxz = sz * k45.x;
  const float kyz = sy * sz * k45.y;
  // packed: each output component is one FMUL2 + two FFMA2 on (re, im)
  const float2 bx = fma2(bc2(kxz), mz, fma2(bc2(kxy), my, mul2(bc2(kxx), mx)));
  const float2 by = fma2(bc2(kyz), mz, fma2(bc2(kyy), my, mul2(bc2(kxy), mx)));
  const float2 bz = fma2(bc2(kzz), mz, fma2(bc2(kyz), my, mul2(bc2(kxz), mx)));
  mx = bx;
  my = by;
  mz = bz;
}

// ---------------------------------------------------------------- K-Z / K-Y2D
// Y2D = false: lines along z of Y[3][nz][Ly][P] at ky = blockIdx.y (K-Z);
// Y2D = true : lines along y of X[3][1][ny][P] (nz == 1, kz = 0).
// the body with explicit (virtual) block indices: a grid of its own (k_conv) or a share of a
// persistent kernel's work (k_persist2d, update.cu); sm = the dynamic shared memory
template <int L, bool Y2D, int NTT = 256>
__device__ __forceinline__ void conv_body(float2* __restrict__ Y, const float* __restrict__ khat, const Dims& d,
                                          const float2* __restrict__ gtw, int bx, int by, float2* sm) {
  using Cf = ZCfg<L, NTT>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C;
  float2* tw = sm;
  pdl_trigger();
  pass_tw<L, E, Cf::NT>(tw, gtw);
  __syncthreads();
  pdl_wait();
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  const int kx = bx * C + c, ky = Y2D ? 0 : by;
  const bool ok = kx < d.NKX;
  const int nin = Y2D ? d.ny : d.nz;
  const unsigned lstride = Y2D ? (unsigned)d.P : (unsigned)d.Ly * d.P;        // between line elements
  const unsigned cstr = Y2D ? (unsigned)d.ny * d.P : (unsigned)d.nz * d.Ly * d.P;  // between components
  const unsigned base = (unsigned)ky * d.P + kx;
  float2 v[3][E];
#pragma unroll
  for (int g = 0; g < 3; ++g)
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      v[g][i] = (2 * i < E && ok && p < nin) ? Y[base + g * cstr + p * lstride] : make_float2(0.f, 0.f);
    }
  const ColAddr<L, C> A{c};
  reg_fft<L, E, 3, false, PASS_TWS>(v, sm + Cf::TWN, A, tw, t);
  if (ok) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      khat_apply(khat, d, kx, Y2D ? p : ky, Y2D ? 0 : p, v[0][i], v[1][i], v[2][i]);
      if ((i & 1) == 1) asm volatile("" ::: "memory");  // bound load hoisting (register budget)
    }
  }
  reg_fft<L, E, 3, true, PASS_TWS>(v, sm + Cf::TWN, A, tw, t);
  if (ok) {
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int p = t + TL * i;
        if (2 * i < E && p < nin) Y[base + g * cstr + p * lstride] = v[g][i];
      }
  }
}

template <int L, bool Y2D>
__global__ void __launch_bounds__(ZCfg<L>::NT) k_conv(float2* __restrict__ Y, const float* __restrict__ khat, Dims d,
                                                      const float2* __restrict__ gtw) {
  extern __shared__ __align__(128) float2 sm[];
  conv_body<L, Y2D>(Y, khat, d, gtw, blockIdx.x, blockIdx.y, sm);
}


}  // namespace mcq
