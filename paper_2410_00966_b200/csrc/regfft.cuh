// regfft.cuh — register-resident Stockham FFT stages for sm_100a.
//
// A line of length L (power of two) is spread over TL = L/E threads of a CTA; thread t owns the
// E positions  p_i = t + TL*i  (i < E)  before the first stage and after the last one.  Every
// radix-R stage (R <= E, R in {2,4,8,16}) is a register codelet; consecutive stages exchange
// data through shared memory once, so an FFT of S stages costs S-1 smem round trips and the
// input/output stay in registers, ready to be loaded from / stored to HBM or fused with the
// next operation (the Khat multiply, the LLG update).  Stage (Ns = product of earlier radices):
//     butterfly b in [0, L/R), k = b mod Ns:
//     v[r] = x[b + r L/R] * w_{Ns R}^{r k},  v = DFT_R(v),  y[(b - k) R + k + r Ns] = v[r]
// Thread t runs butterflies b = t + q*TL (q < E/R) whose inputs are exactly its positions
// p_{q + r E/R}; in the last stage (Ns R = L) the outputs land on the same positions.
// Twiddles come from a per-plan table in shared memory (reg_tw_build): for every stage with
// Ns > 1 the R factors w_{Ns R}^{r k} of butterfly class k are read with R/2 16-byte loads at
// immediate offsets (stride Ns pairs) from one base address (reg_tw_slot).
#pragma once
#include "common.cuh"  // kTwMax
#include "fft.cuh"

namespace mcq {

template <int L, int E>
__host__ __device__ constexpr int reg_radix(int Ns) {
  constexpr int RMAX = cmin(16, cmin(E, L));
  constexpr int lm = ilog2c(RMAX);
  constexpr int lr = ilog2c(L);
  constexpr int first = (lr % lm) ? (1 << (lr % lm)) : RMAX;
  return Ns == 1 ? first : RMAX;
}

// offset of stage Ns's twiddle block in the plan table, and the table size (complex entries)
template <int L, int E>
__host__ __device__ constexpr int reg_tw_off(int Ns) {
  int off = 0;
  for (int n = 1; n < Ns && n < L;) {
    const int R = reg_radix<L, E>(n);
    if (n > 1) off += n * R;
    n *= R;
  }
  return off;
}
template <int L, int E>
__host__ __device__ constexpr int reg_tw_size() {
  const int s = reg_tw_off<L, E>(L);
  return s < 2 ? 2 : s;
}

// Slot of factor r of class k in a stage's block.  MCQ_TWSOA: pairs (2 r2, 2 r2 + 1) of all
// classes side by side — [r2][k][2] — so the 16-byte loads of a warp's consecutive classes are
// consecutive (the [k][r] layout put them R * 8 bytes apart: 59 % of K-U's excess shared
// wavefronts at configs[4], ncu r2h); [k][r] otherwise.
#ifndef MCQ_TWSOA
#define MCQ_TWSOA 1
#endif
template <int R, int Ns>
__host__ __device__ constexpr int reg_tw_slot(int k, int r) {
  return MCQ_TWSOA ? ((r >> 1) * Ns + k) * 2 + (r & 1) : k * R + r;
}

// Fill the plan table from the global fp64-generated table gtw[m] = exp(-2 pi i m / kTwMax)
// (stage Ns, radix R, class k < Ns, factor r < R: w_{Ns R}^{r k}).  Caller synchronises.
template <int L, int E, int NT, int Ns = 1, int OFF = 0>
__device__ __forceinline__ void reg_tw_build(float2* st, const float2* __restrict__ gtw) {
  if constexpr (Ns < L) {
    constexpr int R = reg_radix<L, E>(Ns);
    if constexpr (Ns > 1) {
#pragma unroll
      for (int j = 0; j < (Ns * R + NT - 1) / NT; ++j) {
        const int e = threadIdx.x + j * NT;
        if (e < Ns * R) st[OFF + reg_tw_slot<R, Ns>(e / R, e & (R - 1))] = gtw[((e & (R - 1)) * (e / R)) * (kTwMax / (Ns * R))];
      }
    }
    reg_tw_build<L, E, NT, Ns * R, OFF + (Ns > 1 ? Ns * R : 0)>(st, gtw);
  }
}

// v[l][i]: NLT lines per thread.  A(l, pos): shared-memory index of element pos of the
// thread's line l.  TWS == 0: st is the plan's twiddle table (reg_tw_build), 16-byte aligned;
// TWS > 0: st is a base table, st[m * TWS] = exp(-2 pi i m / L) (fewer live registers when a
// thread runs many small-radix butterflies).
template <int L, int E, int NLT, bool INV, int TWS, int Ns, class Addr>
__device__ __forceinline__ void reg_stage(float2 (&v)[NLT][E], float2* __restrict__ sm, const Addr& A,
                                          const float2* __restrict__ st, int t) {
  if constexpr (Ns < L) {
    constexpr int R = reg_radix<L, E>(Ns);
    constexpr int TL = L / E;
    constexpr int NB = E / R;
    constexpr bool LAST = (Ns * R == L);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int b = t + q * TL;
      const int k = b & (Ns - 1);
      // twiddles depend only on the butterfly, so all NLT lines of the thread share them
      float2 w[R];
      if constexpr (Ns > 1 && TWS == 0) {  // plan table: R/2 16-byte loads from one base
        const float4* w4 = reinterpret_cast<const float4*>(st + reg_tw_off<L, E>(Ns) + reg_tw_slot<R, Ns>(k, 0));
#pragma unroll
        for (int r2 = 0; r2 < R / 2; ++r2) {
          const float4 p = w4[MCQ_TWSOA ? r2 * Ns : r2];
          w[2 * r2] = make_float2(p.x, INV ? -p.y : p.y);
          w[2 * r2 + 1] = make_float2(p.z, INV ? -p.w : p.w);
        }
      } else if constexpr (Ns > 1) {  // base table st[m * TWS] = exp(-2 pi i m / L)
#pragma unroll
        for (int r = 1; r < R; ++r) {
          w[r] = st[(r * k * (L / (Ns * R))) * TWS];
          if (INV) w[r].y = -w[r].y;
        }
      }
#pragma unroll
      for (int l = 0; l < NLT; ++l) {
        float2 x[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          x[r] = v[l][q + r * NB];
          if (Ns > 1 && r > 0) x[r] = cmul(x[r], w[r]);
        }
        dft<R, INV>(x);
        if (LAST) {
#pragma unroll
          for (int r = 0; r < R; ++r) v[l][q + r * NB] = x[r];
        } else {
          const int base = (b - k) * R + k;
#pragma unroll
          for (int r = 0; r < R; ++r) sm[A(l, base + r * Ns)] = x[r];
        }
      }
    }
    if constexpr (!LAST) {
      __syncthreads();
#pragma unroll
      for (int l = 0; l < NLT; ++l)
#pragma unroll
        for (int i = 0; i < E; ++i) v[l][i] = sm[A(l, t + TL * i)];
      __syncthreads();  // the next stage stores into the same buffer
      reg_stage<L, E, NLT, INV, TWS, Ns * R, Addr>(v, sm, A, st, t);
    }
  }
}

#ifndef MCQ_REGTAB
#define MCQ_REGTAB 0  // plan twiddle tables in the y / z passes (measured: K-Y 37.6 vs 35.3 us, K-Z equal)
#endif
template <int L, int E, int NLT, bool INV, int TWS = 0, class Addr>
__device__ __forceinline__ void reg_fft(float2 (&v)[NLT][E], float2* __restrict__ sm, const Addr& A,
                                        const float2* __restrict__ st, int t) {
  static_assert((L & (L - 1)) == 0 && E <= L && L % E == 0, "plan");
  reg_stage<L, E, NLT, INV, TWS, 1, Addr>(v, sm, A, st, t);
}

}  // namespace mcq
