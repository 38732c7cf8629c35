// update.cu — the fused per-stage update kernel K-U, the cavity kernel K-CAV and layout helpers.
//
// K-U (one launch per RK4 stage), one CTA = RY full x-rows at one z,
// TL = N2/E threads per row; thread t of a row owns the packed positions n = t + TL*i (i < E),
// i.e. the cell pairs x = 2n, 2n+1:
//   0. the TMA engine (cp.async.bulk, two mbarriers) stages into shared memory the CTA's rows of
//      the demag spectrum X'[c][z][y][0..N2] and of the stage state m_s (its rows, the y-halo
//      rows and the z-1 / z+1 rows) — issued by one thread, in flight while phase A computes;
//   A. demag x-C2R: Z_n = E_n + i O_n (packed half-length real transform), register-resident
//      inverse FFT -> z_n = B(2n) + i B(2n+1);
//   B. per cell: B' = demag + B_ext + exchange (6-neighbour, C9; neighbours from shared memory)
//      + anisotropy (C10) + B_rms (Gamma(t_s) + a sinc(w t_s)) (eq:bcav P:239), LLG
//      torque (eq:llg P:184), RK4 stage combine + renormalisation (C1, C2); at stage 4 the
//      overlap partial sum B_rms . m_{n+1} in fp64;
//   C. packed forward FFT of m_{s+1} rows (still in registers), real-to-half-complex
//      post-processing through shared memory -> X[c][z][y][0..N2] for the next stage.
// Ms is folded into the kernel spectrum, so the transforms act on m directly.
#include "common.cuh"
#include "regfft.cuh"
#include "tma.cuh"
#include "conv.cuh"
#include <cooperative_groups.h>
#include "../../include/mcq.h"

#ifndef MCQ_UE
#define MCQ_UE 4   // packed row positions per thread in K-U (register budget: 4 beat 8 by 27%)
#endif
#ifndef MCQ_UROWS
#define MCQ_UROWS 0  // stage the m_n / acc / B_rms rows by TMA too (measured slower: 91 vs 82 us,
                     // the extra 18 KB per CTA costs a resident CTA per SM)
#endif

namespace mcq {

#ifndef MCQ_UZG
#define MCQ_UZG 1  // N2 >= 256: the exchange stencil's z neighbours read from HBM / L2 at the cell
                   // update instead of TMA-staged tiles — 12 KB less shared memory per CTA at N2 = 512,
                   // so 5 CTAs per SM fit instead of 4 (ncu r2l: shared memory was K-U's occupancy
                   // limit; configs[4] K-U 2241 -> 2181 us).  At N2 = 128 registers limit occupancy
                   // and the late loads only add latency (67.3 -> 70.1 us): staged there.
#endif
#ifndef MCQ_UYG
#define MCQ_UYG 0  // N2 >= 256: the y neighbours from L2 too (the tile then holds the CTA's own rows
                   // only; measured slower: configs[4] K-U 2221 vs 2187 us, also with 6 CTAs/SM)
#endif
#ifndef MCQ_UPLAN
#define MCQ_UPLAN 1  // K-U row FFTs read a per-plan twiddle table (0: the strided base table)
#endif
template <int N2>
struct UCfg {
#ifndef MCQ_UE_BIG
#define MCQ_UE_BIG MCQ_UE  // positions per thread for N2 >= 256 (experiment knob)
#endif
  static constexpr int EU = N2 >= 256 ? MCQ_UE_BIG : MCQ_UE;
  static constexpr int E = N2 < EU ? N2 : EU;
  static constexpr int TL = N2 / E;                       // threads per row
  static constexpr int RY0 = 128 / TL;
  // at most 16 rows, but at least one full warp (NT >= 32): the warp reductions below use the
  // full mask (tiny rows, nx <= 8, would otherwise leave lanes 16-31 inactive)
  static constexpr int RY1 = RY0 < 1 ? 1 : (RY0 > 16 ? 16 : RY0);
  static constexpr int RY = RY1 * TL < 32 ? 32 / TL : RY1;
  static constexpr int NT = RY * TL;
  // row pitch (complex): a pad slot every 16 positions; even, so rows are 16-byte aligned for TMA
  static constexpr int P0 = N2 + (N2 >= 16 ? N2 / 16 : 1);
  static constexpr int PITCH = P0 + (P0 & 1);
  // staged m_s tile (floats, nx <= N2 cells per row): [3][RY+2][nx] at z, [3][RY][nx] at z-1, z+1
  static constexpr bool UYG = MCQ_UYG && N2 >= 256;  // y neighbours from HBM / L2: no halo rows
  static constexpr int HY = UYG ? 0 : 1;             // halo rows above / below the CTA's rows
  static constexpr int TILE_C = 3 * (RY + 2 * HY) * N2;
  static constexpr int TILE_Z = 3 * RY * N2;
  // the row FFTs' per-plan twiddle table (regfft.cuh: R factors of a butterfly class contiguous,
  // 16-byte loads) and the packing twiddles w_Lx^n, n < N2, then the X rows / exchange buffer
  static constexpr int PLAN = MCQ_UPLAN ? ((reg_tw_size<N2, E>() + 1) & ~1) : 0;
  static constexpr int TWB = MCQ_UPLAN ? N2 : 2 * N2;  // base table entries
  static constexpr size_t XS_BYTES = (size_t)(PLAN + TWB + 3 * RY * PITCH) * sizeof(float2);
  // + the CTA's rows of m_n, the RK4 accumulator and the B_rms map ([3][RY][nx] each, TMA path),
  // so every HBM read of the kernel is in flight while phase A runs
  static constexpr bool UZG = MCQ_UZG && N2 >= 256;  // z neighbours from HBM / L2, not staged
  static constexpr size_t SMEM = XS_BYTES + (size_t)(TILE_C + ((MCQ_UROWS ? 3 : 0) + (UZG ? 0 : 2)) * TILE_Z) * sizeof(float);
};

__device__ __forceinline__ float3 cross3(float3 a, float3 b) {
  return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float3 nrm3(float3 v) {
  const float n2 = dot3(v, v);
  if (!(n2 <= 0.f)) {  // NaN propagates (vacuum stays 0): the divergence guard sees it
    const float r = rsqrtf(n2);
    return make_float3(v.x * r, v.y * r, v.z * r);
  }
  return make_float3(0.f, 0.f, 0.f);
}
__device__ __forceinline__ float3 ld3(const float* __restrict__ p, long long N, long long i) {
  return make_float3(__ldg(p + i), __ldg(p + N + i), __ldg(p + 2 * N + i));
}
__device__ __forceinline__ float3 sm3(const float* p, int cs, int i) { return make_float3(p[i], p[cs + i], p[2 * cs + i]); }

// shared-memory address of element pos of component-line l of row yl.  N2 >= 128 (one row per
// warp): pos ^ ((pos >> 2) & 15) — every Stockham store (positions (b - k) R + k + r Ns) and load
// (t + TL i) of the radix-4/2 row transforms takes 2 wavefronts per warp, the minimum for 256 B
// (the 1-in-16 padding it replaces left 1/3 of the wavefronts as bank conflicts: round 1 ncu);
// shorter rows (several per warp) keep the padding
#ifndef MCQ_USWZ
#define MCQ_USWZ 1  // XOR-swizzled row exchange buffer for N2 >= 128 (0: 1-in-16 padding)
#endif
template <int N2>
struct RowAddr {
  int yl;
  __device__ __forceinline__ int operator()(int l, int pos) const {
    if constexpr (MCQ_USWZ && N2 >= 128) return (l * UCfg<N2>::RY + yl) * UCfg<N2>::PITCH + (pos ^ ((pos >> 2) & 15));
    else return (l * UCfg<N2>::RY + yl) * UCfg<N2>::PITCH + pos + (N2 >= 16 ? (pos >> 4) : 0);
  }
};

// One cell from register inputs: state m, in-mesh neighbours nb[k] (valid where ok[k]), m_n,
// the RK4 accumulator so far, the cavity + excitation field bcav * gmul (added iff gmul != 0:
// B_rms * (Gamma + a sinc) for one mode, or the summed field of all modes with gmul = 1) and
// the demag field.  Computes B' and, by mode, the field (Bout),
// the max torque, or the RK4 stage update (returns m_{s+1}, writes the new accumulator to
// acc_out).  All memory traffic (and the overlap sums) stays in the caller.
// Thermal noise (reading C-TH): the c-th output of SplitMix64 started at state `seed`, and the
// standard normal 3-vector of a cell from the two words at counters c0, c0 + 1 (Box-Muller on
// u1 = (h >> 40 + 1) 2^-24 in (0, 1], u2 = (h & 0xFFFFFF) 2^-24; eta = (cos0, sin0, cos1)).
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long seed, unsigned long long c) {
  unsigned long long z = seed + (c + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float3 thermal_eta(unsigned long long seed, unsigned long long c0) {
  const unsigned long long h0 = splitmix64(seed, c0), h1 = splitmix64(seed, c0 + 1ull);
  float s0, k0, s1, k1;
  const float r0 = sqrtf(-2.f * logf(((float)(h0 >> 40) + 1.f) * 0x1p-24f));
  const float r1 = sqrtf(-2.f * logf(((float)(h1 >> 40) + 1.f) * 0x1p-24f));
  sincospif(2.f * ((float)(h0 & 0xFFFFFFull) * 0x1p-24f), &s0, &k0);
  sincospif(2.f * ((float)(h1 & 0xFFFFFFull) * 0x1p-24f), &s1, &k1);
  return make_float3(r0 * k0, r0 * s0, r1 * k1);
}

template <int GEN, int FM, int FS>
__device__ __forceinline__ float3 cell_core(const UpdateArgs& a, float3 m, const float3 (&nb)[6], const bool (&ok)[6],
                                            float3 mn, float3 ap, float3 bcav, float gmul, float3 Bd,
                                            float& tmax, float3& acc_out, float3& Bout) {
  const int mode = FM >= 0 ? FM : a.mode;  // FM: the mode fixed at compile time (hot LLG instance)
  const int stage_ = FS > 0 ? FS : a.stage;  // FS: the RK4 stage fixed at compile time
  if (mode == MODE_X0) return m;
  float3 B = make_float3(0.f, 0.f, 0.f);
  if (dot3(m, m) > 0.f) {
    B = Bd;
    if (a.terms & MCQ_TERM_ZEEMAN) {
      B.x += a.bext[0];
      B.y += a.bext[1];
      B.z += a.bext[2];
    }
    if (a.terms & MCQ_TERM_EXCHANGE) {
      float3 acc = make_float3(0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const float coef = a.ex[k >> 1];
        if (ok[k] && dot3(nb[k], nb[k]) > 0.f) {  // in the mesh and magnetic (C9)
          acc.x += coef * (nb[k].x - m.x);
          acc.y += coef * (nb[k].y - m.y);
          acc.z += coef * (nb[k].z - m.z);
        }
      }
      B.x += acc.x;
      B.y += acc.y;
      B.z += acc.z;
    }
    if (a.terms & MCQ_TERM_ANIS) {
      if (a.ku != 0.f) {
        const float mu = m.x * a.u[0] + m.y * a.u[1] + m.z * a.u[2];
        B.x += a.ku * mu * a.u[0];
        B.y += a.ku * mu * a.u[1];
        B.z += a.ku * mu * a.u[2];
      }
      if (a.kc != 0.f) {
        const float m1 = m.x * a.c1[0] + m.y * a.c1[1] + m.z * a.c1[2];
        const float m2 = m.x * a.c2[0] + m.y * a.c2[1] + m.z * a.c2[2];
        const float m3 = m.x * a.c3[0] + m.y * a.c3[1] + m.z * a.c3[2];
        const float f1 = -a.kc * m1 * (m2 * m2 + m3 * m3);
        const float f2 = -a.kc * m2 * (m1 * m1 + m3 * m3);
        const float f3 = -a.kc * m3 * (m1 * m1 + m2 * m2);
        B.x += f1 * a.c1[0] + f2 * a.c2[0] + f3 * a.c3[0];
        B.y += f1 * a.c1[1] + f2 * a.c2[1] + f3 * a.c3[1];
        B.z += f1 * a.c1[2] + f2 * a.c2[2] + f3 * a.c3[2];
      }
    }
    if (GEN && (a.terms & MCQ_TERM_DMI) && (a.dmi[0] != 0.f || a.dmi[1] != 0.f)) {
      // interfacial DMI, central differences, Neumann ghosts (own m) outside the mesh / in vacuum
      float3 g[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) g[k] = (ok[k] && dot3(nb[k], nb[k]) > 0.f) ? nb[k] : m;
      B.x += a.dmi[0] * (g[1].z - g[0].z);
      B.y += a.dmi[1] * (g[3].z - g[2].z);
      B.z -= a.dmi[0] * (g[1].x - g[0].x) + a.dmi[1] * (g[3].y - g[2].y);
    }
    if (gmul != 0.f) {
      B.x += bcav.x * gmul;
      B.y += bcav.y * gmul;
      B.z += bcav.z * gmul;
    }
  }
  if (mode == MODE_FIELD) {
    Bout = B;
    return m;
  }
  const float3 mxB = cross3(m, B);
  if (mode == MODE_MAXTORQUE) {
    tmax = fmaxf(tmax, sqrtf(dot3(mxB, mxB)));
    return m;
  }
  const float3 mmxB = cross3(m, mxB);
  float3 k;
  if (mode == MODE_LLG || (GEN == 2 && mode == MODE_DP)) {
    k = make_float3(-a.gl * (mxB.x + a.alpha * mmxB.x), -a.gl * (mxB.y + a.alpha * mmxB.y),
                    -a.gl * (mxB.z + a.alpha * mmxB.z));
  } else {  // MODE_RELAX: -gamma m x (m x B)
    k = make_float3(-a.gamma * mmxB.x, -a.gamma * mmxB.y, -a.gamma * mmxB.z);
  }
  const int stage = stage_;
  if (stage == 1) mn = m;
  if (GEN == 2 && mode == MODE_DP) {  // ap = sum_{j < s} comb[j-1] k_j from the caller (reading C-DP)
    const float cs = a.comb[stage - 1];
    const float3 inc = make_float3(ap.x + cs * k.x, ap.y + cs * k.y, ap.z + cs * k.z);
    acc_out = k;
    if (stage == 7) {  // error estimate of this cell; the state is the step result itself
      const float3 e = make_float3(a.h * inc.x, a.h * inc.y, a.h * inc.z);
      tmax = fmaxf(tmax, sqrtf(dot3(e, e)));
      return m;
    }
    return nrm3(make_float3(mn.x + a.h * inc.x, mn.y + a.h * inc.y, mn.z + a.h * inc.z));
  }
  float3 out;
  if (stage < 4) {
    acc_out = (stage == 1) ? k : make_float3(ap.x + 2.f * k.x, ap.y + 2.f * k.y, ap.z + 2.f * k.z);
    out = nrm3(make_float3(mn.x + a.h * k.x, mn.y + a.h * k.y, mn.z + a.h * k.z));
  } else {
    out = nrm3(make_float3(mn.x + a.dt6 * (ap.x + k.x), mn.y + a.dt6 * (ap.y + k.y), mn.z + a.dt6 * (ap.z + k.z)));
  }
  return out;
}

// paired access to cells (x, x+1) of an SoA component: one 8-byte access when the index is even
// (nx even), else two 4-byte ones; `two` = the second cell exists.
__device__ __forceinline__ float2 ld_pair(const float* __restrict__ p, unsigned i, bool vec, bool two) {
  if (vec) return __ldg(reinterpret_cast<const float2*>(p + i));
  return make_float2(__ldg(p + i), two ? __ldg(p + i + 1) : 0.f);
}
__device__ __forceinline__ void st_pair(float* __restrict__ p, unsigned i, float2 v, bool vec, bool two) {
  if (vec) {
    *reinterpret_cast<float2*>(p + i) = v;
  } else {
    p[i] = v.x;
    if (two) p[i + 1] = v.y;
  }
}
__device__ __forceinline__ float2 sm_pair(const float* p) { return *reinterpret_cast<const float2*>(p); }

#ifndef MCQ_UMINB
#define MCQ_UMINB 5  // min resident CTAs per SM requested from ptxas (96-register cap: 84.8 vs 86.8 us on configs[1])
#endif
// MM: cavity modes compiled in (1, 2 or kMaxModes with a.nmodes <= MM at run time); GEN: 0 the
// plain RK4 instances, 1 + interfacial DMI and the thermal draw, 2 + the Dormand-Prince stages
// FM >= 0: the update mode fixed at compile time — the plain RK4 instance (<N2, 1, 0, MODE_LLG>)
// then carries no FIELD / MAXTORQUE / X0 / RELAX code, a third less SASS (instruction-cache
// misses showed as 'no_instruction' stalls in ncu); FM = -1: the mode from the arguments
// the body with explicit (virtual) block indices (bx, by) of a (gx, gy) grid: a grid of its own
// (k_update) or a share of the persistent 2D kernel (k_persist2d); NOTMA: the plain-load staging
// (the persistent kernel re-enters the body and does not re-arm mbarriers)
template <int N2, int MM, int GEN, int FM, int FS, bool NOTMA = false>
__device__ __forceinline__ void update_body(const UpdateArgs& a, const float2* __restrict__ gtw, int bx, int by,
                                            int gx, int gy, float2* sm) {
  const int mode = FM >= 0 ? FM : a.mode;
  const int stage_ = FS > 0 ? FS : a.stage;  // FS: the RK4 stage fixed at compile time (hot instances)
  using Cf = UCfg<N2>;
  constexpr int E = Cf::E, TL = Cf::TL, RY = Cf::RY, NT = Cf::NT, LX = 2 * N2, PITCH = Cf::PITCH;
  // the row FFTs' plan table (16-byte twiddle loads at immediate offsets; the strided base
  // table it replaces had 2-4-way bank conflicts in the late stages) and w_Lx^n for the packing
  float2* ptw = sm;                // row-FFT plan table (MCQ_UPLAN)
  float2* tw = sm + Cf::PLAN;       // w_Lx^m, m < TWB
  float2* xs = tw + Cf::TWB;        // [3][RY][PITCH]: X rows (staged by TMA), then the FFT exchange buffer
  float* tc = reinterpret_cast<float*>(reinterpret_cast<char*>(sm) + Cf::XS_BYTES);  // [3][RY+2][nx]
  float* tzm = tc + Cf::TILE_C;                                                       // [3][RY][nx]
  float* tzp = tzm + (Cf::UZG ? 0 : Cf::TILE_Z);
  float* tmn = tzp + (Cf::UZG ? 0 : Cf::TILE_Z);  // [3][RY][nx]: m_n, acc, B_rms rows (TMA path)
  float* tap = tmn + Cf::TILE_Z;
  float* tbr = tap + Cf::TILE_Z;
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ double red[32 * kNPart];
  __shared__ float redf[32];

  const Dims& d = a.d;
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const long long N = d.cs;                        // component stride of the state arrays
  const int y0 = bx * RY, z = by;  // z: local plane (X rows, partials)
  const int zs = z + d.zoff;                       // storage plane of the (halo'd) state arrays
  const bool zlo = d.zg0 + z > 0, zhi = d.zg0 + z < d.nzg - 1;  // global z neighbours exist
  const int nrow = min(RY, ny - y0);
  constexpr int HY = Cf::HY;
  const int ylo = y0 > 0 ? y0 - HY : 0, yhi = min(y0 + RY - 1 + HY, ny - 1);  // staged m_s rows at z
  const int nxp = nx + (nx & 1);                                     // tile row pitch (8-byte pairs)
  const int csc = (RY + 2 * HY) * nxp, csz = RY * nxp;               // component pitches of the tiles
  const bool use_demag = a.demag && (a.terms & MCQ_TERM_DEMAG) && mode != MODE_X0;
  const bool tma = !NOTMA && (nx & 3) == 0 && (d.P & 1) == 0;
  const bool trows = tma && MCQ_UROWS;
  const bool st_mode = mode == MODE_LLG || mode == MODE_RELAX;
  const bool ld_mn = trows && st_mode && stage_ > 1;  // m_n and the accumulator: stages 2-4
  const bool ld_br = trows && a.brms[0] && (mode == MODE_LLG || mode == MODE_FIELD);

  // ---------------- 0: TMA staging (bars[0]: X rows, bars[1]: m_s tile) ----------------
  // thread 0 initialises the barriers and issues every copy at once, so the copies' latency
  // overlaps the twiddle-table load below; the other threads see the initialised barriers
  // after the __syncthreads and only then wait on them
  pdl_trigger();
  if (tma && threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    pdl_wait();  // the copies read the previous kernels' output
    if (use_demag) {
      const uint32_t bx = (uint32_t)(N2 + 2) * 8;  // N2+1 columns rounded to 16 bytes (<= PITCH)
      mbar_arrive_expect_tx(&bars[0], 3u * nrow * bx);
      for (int c = 0; c < 3; ++c)
        for (int r = 0; r < nrow; ++r)
          tma_load_1d(xs + (c * RY + r) * PITCH, a.X + ((size_t)(c * nz + z) * ny + y0 + r) * d.P, bx, &bars[0]);
    }
    const uint32_t bc = (uint32_t)(yhi - ylo + 1) * nx * 4, bz = (uint32_t)nrow * nx * 4;
    const bool stz = !Cf::UZG;  // z-neighbour rows staged
    mbar_arrive_expect_tx(&bars[1], 3 * (bc + (stz && zlo ? bz : 0) + (stz && zhi ? bz : 0) + (ld_mn ? 2 * bz : 0) +
                                         (ld_br ? bz : 0)));
    const long long rows = ((long long)zs * ny + y0) * nx;  // the CTA's rows at z (contiguous)
    for (int c = 0; c < 3; ++c) {
      const float* src = a.mS + c * N;
      tma_load_1d(tc + c * csc + (ylo - (y0 - HY)) * nx, src + ((long long)zs * ny + ylo) * nx, bc, &bars[1]);
      if (stz && zlo) tma_load_1d(tzm + c * csz, src + ((long long)(zs - 1) * ny + y0) * nx, bz, &bars[1]);
      if (stz && zhi) tma_load_1d(tzp + c * csz, src + ((long long)(zs + 1) * ny + y0) * nx, bz, &bars[1]);
      if (ld_mn) {
        tma_load_1d(tmn + c * csz, a.mN + c * N + rows, bz, &bars[1]);
        tma_load_1d(tap + c * csz, a.acc + c * N + rows, bz, &bars[1]);
      }
      if (ld_br) tma_load_1d(tbr + c * csz, a.brms[0] + c * N + rows, bz, &bars[1]);
    }
  }
  {  // twiddle table: every load in flight at once (a serial load -> store loop was the top stall
     // of the N2 = 512 instance, ncu r2t: 8 dependent L2 round trips per CTA)
    constexpr int TWB = Cf::TWB, NL = (TWB + NT - 1) / NT;
    float2 w[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int m = threadIdx.x + j * NT;
      w[j] = (m < TWB) ? __ldg(gtw + m * (kTwMax / LX)) : make_float2(0.f, 0.f);
    }
    if constexpr (MCQ_UPLAN) reg_tw_build<N2, E, NT>(ptw, gtw);
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (threadIdx.x + j * NT < TWB) tw[threadIdx.x + j * NT] = w[j];
  }
  pdl_wait();
  __syncthreads();
  if (!tma) {  // fallback (unaligned rows): cooperative coalesced loads into the same layout
    for (int c = 0; c < 3; ++c) {
      if (use_demag)
        for (int e = threadIdx.x; e < nrow * (N2 + 1); e += NT) {
          const int r = e / (N2 + 1), k = e - r * (N2 + 1);
          xs[(c * RY + r) * PITCH + k] = a.X[((size_t)(c * nz + z) * ny + y0 + r) * d.P + k];
        }
      const float* src = a.mS + c * N;
      for (int e = threadIdx.x; e < (yhi - ylo + 1) * nx; e += NT) {
        const int r = e / nx, x = e - r * nx;
        tc[c * csc + (ylo - (y0 - HY) + r) * nxp + x] = src[((long long)zs * ny + ylo) * nx + e];
      }
      if (!Cf::UZG)
        for (int e = threadIdx.x; e < nrow * nx; e += NT) {
          const int r = e / nx, x = e - r * nx;
          if (zlo) tzm[c * csz + r * nxp + x] = src[((long long)(zs - 1) * ny + y0) * nx + e];
          if (zhi) tzp[c * csz + r * nxp + x] = src[((long long)(zs + 1) * ny + y0) * nx + e];
        }
    }
    __syncthreads();
  }

  const int yl = threadIdx.x / TL, t = threadIdx.x % TL, y = y0 + yl;
  const bool rowok = y < ny;
  const RowAddr<N2> A{yl};
  float2 v[3][E];

  // ---------------- A: demag rows (packed x-C2R) ----------------
  if (use_demag) {
    if (tma) mbar_wait(&bars[0], 0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2* row = xs + (c * RY + yl) * PITCH;  // raw staged row (unpadded positions)
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int n = t + TL * i;
        float2 zn = make_float2(0.f, 0.f);
        if (rowok) {
          const float2 xk = row[n], xn = cconj(row[N2 - n]);
          const float2 ev = cadd(xk, xn);
          const float2 od = cmul(csub(xk, xn), cconj(tw[n]));  // * w^{-n}
          zn = make_float2(ev.x - od.y, ev.y + od.x);           // E + i O
        }
        v[c][i] = zn;
      }
    }
    __syncthreads();  // the staged rows are read before the FFT reuses the buffer
    if constexpr (MCQ_UPLAN) reg_fft<N2, E, 3, true, 0>(v, xs, A, ptw, t);
    else reg_fft<N2, E, 3, true, 2>(v, xs, A, tw, t);
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int i = 0; i < E; ++i) v[c][i] = make_float2(0.f, 0.f);
  }

  // ---------------- B: per-cell fields, torque, RK4 ----------------
  if (tma) mbar_wait(&bars[1], 0);
  // per mode k: gsum_k = Gamma_k(t_s) + a_k sinc(w_k t_s) (stage time t_s, C3)
  const int nm = MM > 1 ? a.nmodes : 1;
  float gs[MM];
  bool any_cav = false;
#pragma unroll
  for (int k = 0; k < MM; ++k) {
    float gc = 0.f, ge = 0.f;
    if (k < nm && (mode == MODE_LLG || mode == MODE_FIELD || mode == MODE_DP)) {
      const int si = (mode == MODE_FIELD) ? 0 : stage_ - 1;
      gc = (a.terms & MCQ_TERM_CAVITY) ? a.cav->gc[k][si] : 0.f;
      ge = (a.terms & MCQ_TERM_EXCITATION) ? a.cav->ge[k][si] : 0.f;
    }
    gs[k] = gc + ge;
    any_cav = any_cav || gs[k] != 0.f;
  }
  const float gsum = gs[0];
  // thermal draw of this step: counters 2 (n N + g) (+1), N the global cell count (C-TH)
  const unsigned long long th_base =
      (GEN && a.th != 0.f) ? 2ull * (unsigned long long)(*a.thstep) * ((unsigned long long)nx * ny * d.nzg) : 0ull;
  double wacc[MM];
#pragma unroll
  for (int k = 0; k < MM; ++k) wacc[k] = 0.0;
  const bool dp = GEN == 2 && mode == MODE_DP;
  // overlaps (and the trace's sum m) of the step result: RK4 stage 4's output, DP stage 7's input
  const bool wsum = (mode == MODE_LLG && stage_ == 4) || (dp && stage_ == 7);
  float tmax = 0.f;
  const bool tr = a.trace && wsum;
  const unsigned rowbase = (unsigned)nx * (y + (unsigned)ny * zs);  // 32-bit indices (< 2^32 elements)
  const unsigned Nu = (unsigned)N;
  const float* trow = tc + (yl + HY) * nxp;  // this row inside the z tile
  const bool vec = (nx & 1) == 0;           // global pairs are 8-byte aligned
  const bool st = mode == MODE_LLG || mode == MODE_RELAX || (dp && stage_ < 7);  // writes a state
  const bool need_mn = st && stage_ > 1, need_acc = !dp && st && stage_ > 1;
  const bool need_br = a.brms[0] && (gsum != 0.f || wsum);
  const bool th_st = GEN && a.eta && mode == MODE_LLG && stage_ == 1;  // thermal draw stored
  const bool th_ld = GEN && a.eta && mode == MODE_LLG && stage_ > 1;   // and reloaded
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int x0 = 2 * (t + TL * i);
    if (2 * i >= E) {  // x0 >= N2 >= nx: zero padding, statically (prunes the C2R's last stage
#pragma unroll       // outputs and the R2C's first-stage inputs)
      for (int c = 0; c < 3; ++c) v[c][i] = make_float2(0.f, 0.f);
      continue;
    }
    float2 o[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    if (rowok && x0 < nx) {
      const bool two = x0 + 1 < nx;
      const unsigned idx = rowbase + x0;
      // the pair (x0, x0+1) and its neighbours from the staged tile; m_n, acc, B_rms from HBM
      float2 mc[3], ym[3], yp[3], zm[3], zp[3], mn2[3], ap2[3], br2[3];
      float xl[3], xr[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float* r = trow + c * csc;
        mc[c] = sm_pair(r + x0);
        if constexpr (Cf::UYG) {
          ym[c] = y > 0 ? ld_pair(a.mS, c * Nu + idx - nx, vec, two) : mc[c];
          yp[c] = y < ny - 1 ? ld_pair(a.mS, c * Nu + idx + nx, vec, two) : mc[c];
        } else {
          ym[c] = y > 0 ? sm_pair(r - nxp + x0) : mc[c];
          yp[c] = y < ny - 1 ? sm_pair(r + nxp + x0) : mc[c];
        }
        if constexpr (Cf::UZG) {
          const unsigned pl = (unsigned)nx * ny;  // plane stride (the halo planes of a slab included)
          zm[c] = zlo ? ld_pair(a.mS, c * Nu + idx - pl, vec, two) : mc[c];
          zp[c] = zhi ? ld_pair(a.mS, c * Nu + idx + pl, vec, two) : mc[c];
        } else {
          zm[c] = zlo ? sm_pair(tzm + c * csz + yl * nxp + x0) : mc[c];
          zp[c] = zhi ? sm_pair(tzp + c * csz + yl * nxp + x0) : mc[c];
        }
        xl[c] = x0 > 0 ? r[x0 - 1] : 0.f;
        xr[c] = x0 + 2 < nx ? r[x0 + 2] : 0.f;
        const int so = c * csz + yl * nxp + x0;  // staged rows (TMA path)
        mn2[c] = need_mn ? (trows ? sm_pair(tmn + so) : ld_pair(a.mN, c * Nu + idx, vec, two)) : make_float2(0.f, 0.f);
        ap2[c] = need_acc ? (trows ? sm_pair(tap + so) : ld_pair(a.acc, c * Nu + idx, vec, two)) : make_float2(0.f, 0.f);
        br2[c] = need_br ? (trows ? sm_pair(tbr + so) : ld_pair(a.brms[0], c * Nu + idx, vec, two))
                         : make_float2(a.brms_u[0][c], a.brms_u[0][c]);
      }
      if (dp) {  // ap = sum_{j < s} comb[j-1] k_j (the earlier stages' slopes, from HBM)
        // two slopes per iteration: their loads are in flight together (same summation order)
#pragma unroll 1
        for (int j = 1; j < stage_; j += 2) {
          float2 kk[2][3];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const float* Kj = a.K + (size_t)(j + q - 1) * 3 * Nu;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              kk[q][c] = j + q < stage_ ? ld_pair(Kj, c * Nu + idx, vec, two) : make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (j + q < stage_) {
              const float w = a.comb[j + q - 1];
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                ap2[c].x += w * kk[q][c].x;
                ap2[c].y += w * kk[q][c].y;
              }
            }
          }
        }
      }
      // the step's thermal draw: drawn by stage 1 and stored, reloaded by stages 2-4 (the
      // same values a redraw would give, at 12 bytes per cell instead of the generator's cost)
      float2 th2[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      if (GEN && a.th != 0.f) {
        if (th_ld) {
#pragma unroll
          for (int c = 0; c < 3; ++c) th2[c] = ld_pair(a.eta, c * Nu + idx, vec, two);
        } else {
          const unsigned long long g0 = ((unsigned long long)(d.zg0 + z) * ny + y) * nx + x0;
          const float3 e0 = thermal_eta(a.th_seed, th_base + 2ull * g0);
          const float3 e1 = two ? thermal_eta(a.th_seed, th_base + 2ull * (g0 + 1ull)) : e0;
          th2[0] = make_float2(e0.x, e1.x);
          th2[1] = make_float2(e0.y, e1.y);
          th2[2] = make_float2(e0.z, e1.z);
          if (th_st) {
#pragma unroll
            for (int c = 0; c < 3; ++c) st_pair(a.eta, c * Nu + idx, th2[c], vec, two);
          }
        }
      }
      float2 bk2[MM > 1 ? MM - 1 : 1][3];  // extra modes' B_rms (maps or uniform values)
#pragma unroll
      for (int k = 1; k < MM; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          bk2[k - 1][c] = (k < nm && a.brms[k] && (gs[k] != 0.f || wsum))
                              ? ld_pair(a.brms[k], c * Nu + idx, vec, two)
                              : make_float2(a.brms_u[k][c], a.brms_u[k][c]);
      float2 acc2[3], bf2[3];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !two) break;
        const int x = x0 + h;
#define MCQ_PICK(p) (h ? (p).y : (p).x)
        const float3 m = make_float3(MCQ_PICK(mc[0]), MCQ_PICK(mc[1]), MCQ_PICK(mc[2]));
        const bool ok[6] = {x > 0, x < nx - 1, y > 0, y < ny - 1, zlo, zhi};
        float3 nb[6];
        nb[0] = h ? make_float3(mc[0].x, mc[1].x, mc[2].x) : make_float3(xl[0], xl[1], xl[2]);
        nb[1] = h ? make_float3(xr[0], xr[1], xr[2]) : make_float3(mc[0].y, mc[1].y, mc[2].y);
        nb[2] = make_float3(MCQ_PICK(ym[0]), MCQ_PICK(ym[1]), MCQ_PICK(ym[2]));
        nb[3] = make_float3(MCQ_PICK(yp[0]), MCQ_PICK(yp[1]), MCQ_PICK(yp[2]));
        nb[4] = make_float3(MCQ_PICK(zm[0]), MCQ_PICK(zm[1]), MCQ_PICK(zm[2]));
        nb[5] = make_float3(MCQ_PICK(zp[0]), MCQ_PICK(zp[1]), MCQ_PICK(zp[2]));
        const float3 mn = make_float3(MCQ_PICK(mn2[0]), MCQ_PICK(mn2[1]), MCQ_PICK(mn2[2]));
        const float3 ap = make_float3(MCQ_PICK(ap2[0]), MCQ_PICK(ap2[1]), MCQ_PICK(ap2[2]));
        const float3 br = make_float3(MCQ_PICK(br2[0]), MCQ_PICK(br2[1]), MCQ_PICK(br2[2]));
        float3 Bd = make_float3(MCQ_PICK(v[0][i]), MCQ_PICK(v[1][i]), MCQ_PICK(v[2][i]));
        if (GEN && a.th != 0.f) {
          Bd.x += a.th * MCQ_PICK(th2[0]);
          Bd.y += a.th * MCQ_PICK(th2[1]);
          Bd.z += a.th * MCQ_PICK(th2[2]);
        }
        float3 accn = make_float3(0.f, 0.f, 0.f), Bf = make_float3(0.f, 0.f, 0.f);
        float3 out;
        if constexpr (MM == 1) {
          out = cell_core<GEN, FM, FS>(a, m, nb, ok, mn, ap, br, gsum, Bd, tmax, accn, Bf);
        } else {
          float3 bcav = make_float3(br.x * gsum, br.y * gsum, br.z * gsum);
#pragma unroll
          for (int k = 1; k < MM; ++k) {
            if (k < nm) {
              bcav.x += MCQ_PICK(bk2[k - 1][0]) * gs[k];
              bcav.y += MCQ_PICK(bk2[k - 1][1]) * gs[k];
              bcav.z += MCQ_PICK(bk2[k - 1][2]) * gs[k];
            }
          }
          out = cell_core<GEN, FM, FS>(a, m, nb, ok, mn, ap, bcav, any_cav ? 1.f : 0.f, Bd, tmax, accn, Bf);
        }
        if (wsum) {
          wacc[0] += (double)(br.x * out.x) + (double)(br.y * out.y) + (double)(br.z * out.z);
#pragma unroll
          for (int k = 1; k < MM; ++k)
            if (k < nm)
              wacc[k] += (double)(MCQ_PICK(bk2[k - 1][0]) * out.x) + (double)(MCQ_PICK(bk2[k - 1][1]) * out.y) +
                         (double)(MCQ_PICK(bk2[k - 1][2]) * out.z);
        }
#undef MCQ_PICK
        if (h) {
          o[0].y = out.x; o[1].y = out.y; o[2].y = out.z;
          acc2[0].y = accn.x; acc2[1].y = accn.y; acc2[2].y = accn.z;
          bf2[0].y = Bf.x; bf2[1].y = Bf.y; bf2[2].y = Bf.z;
        } else {
          o[0].x = out.x; o[1].x = out.y; o[2].x = out.z;
          acc2[0].x = accn.x; acc2[1].x = accn.y; acc2[2].x = accn.z;
          bf2[0].x = Bf.x; bf2[1].x = Bf.y; bf2[2].x = Bf.z;
        }
      }
      if (!two) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          o[c].y = 0.f;
          acc2[c].y = 0.f;
          bf2[c].y = 0.f;
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (mode == MODE_FIELD) st_pair(a.bout, c * Nu + idx, bf2[c], vec, two);
        if (st) {
          st_pair(a.mOut, c * Nu + idx, o[c], vec, two);
          // z-slab halos: remote stores into the neighbours' halo planes (P2P over NVLink)
          if (a.halo_lo && z == 0) st_pair(a.halo_lo, c * Nu + (unsigned)nx * (y + (unsigned)ny * (nz + 1)) + x0, o[c], vec, two);
          if (a.halo_hi && z == nz - 1) st_pair(a.halo_hi, c * Nu + (unsigned)nx * y + x0, o[c], vec, two);
          if (dp)
            st_pair(a.K + (size_t)(stage_ - 1) * 3 * Nu, c * Nu + idx, acc2[c], vec, two);  // k_s
          else if (stage_ < 4)
            st_pair(a.acc, c * Nu + idx, acc2[c], vec, two);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) v[c][i] = o[c];
  }

  if ((a.halo_lo && z == 0) || (a.halo_hi && z == nz - 1)) __threadfence_system();

  // ---------------- reductions ----------------
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (NT + 31) / 32;
  float3 msum = make_float3(0.f, 0.f, 0.f);  // from the packed new state in v (0 outside the mesh)
  if (tr) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      msum.x += v[0][i].x + v[0][i].y;
      msum.y += v[1][i].x + v[1][i].y;
      msum.z += v[2][i].x + v[2][i].y;
    }
  }
  if (wsum) {  // RK4 stage 4 / Dormand-Prince stage 7: the step result's partials
    // one quantity at a time (few live registers): W_k of the compiled modes, then sum m
    auto warp_sum = [&](double q, int k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) q += __shfl_down_sync(0xffffffffu, q, o);
      if (lane == 0) red[warp * kNPart + k] = q;
    };
#pragma unroll
    for (int k = 0; k < kMaxModes; ++k) {
      if (k < MM)
        warp_sum(wacc[k < MM ? k : 0], k);
      else if (lane == 0)
        red[warp * kNPart + k] = 0.0;
    }
    if (tr) {
      warp_sum((double)msum.x, kPartM);
      warp_sum((double)msum.y, kPartM + 1);
      warp_sum((double)msum.z, kPartM + 2);
    }
    __syncthreads();
    if (threadIdx.x < kNPart) {  // fixed order over the warps: deterministic; [q][CTA] layout
      double s = 0.0;
      if (threadIdx.x < kPartM || tr)
        for (int w = 0; w < nw; ++w) s += red[w * kNPart + threadIdx.x];
      const int nps = gx * gy;
      a.partials[threadIdx.x * nps + by * gx + bx] = s;
      // divergence guard at no per-cell cost: br . m_{n+1} is NaN for any non-finite m_{n+1}
      // (0 * inf and 0 * NaN are NaN), so a non-finite W_0 partial flags the step
      if (threadIdx.x == 0 && a.nonfinite && !isfinite(s)) atomicOr(a.nonfinite, 1);
    }
  }
  if (dp && stage_ == 7) {  // the step's error estimate: max over cells (fp32 bits, >= 0)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_down_sync(0xffffffffu, tmax, o));
    if (lane == 0) redf[warp] = tmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      float s = 0.f;
      for (int w = 0; w < nw; ++w) s = fmaxf(s, redf[w]);
      atomicMax(a.maxbits, __float_as_uint(s));
    }
  }
  if (mode == MODE_MAXTORQUE) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_down_sync(0xffffffffu, tmax, o));
    if (lane == 0) redf[warp] = tmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      float s = 0.f;
      for (int w = 0; w < nw; ++w) s = fmaxf(s, redf[w]);
      atomicMax(a.maxbits, __float_as_uint(s));
    }
    return;
  }
  if (mode == MODE_FIELD) return;

  // ---------------- C: packed x-R2C of the new rows ----------------
  if (!use_demag) __syncthreads();  // xs may still hold staged rows of other threads' reads
  if constexpr (MCQ_UPLAN) reg_fft<N2, E, 3, false, 0>(v, xs, A, ptw, t);
  else reg_fft<N2, E, 3, false, 2>(v, xs, A, tw, t);
  // X_k = (Z_k + conj Z_{N-k})/2 - i/2 w^k (Z_k - conj Z_{N-k}); partners via shared memory
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < E; ++i) xs[A(c, t + TL * i)] = v[c][i];
  __syncthreads();
  if (rowok) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float2* row = a.X + ((size_t)(c * nz + z) * ny + y) * d.P;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + TL * i;
        const float2 zk = v[c][i];
        const float2 zn = cconj(xs[A(c, (N2 - k) & (N2 - 1))]);
        const float2 ev = cadd(zk, zn);
        const float2 wd = cmul(tw[k], csub(zk, zn));
        row[k] = make_float2(0.5f * (ev.x + wd.y), 0.5f * (ev.y - wd.x));
        if (k == 0) row[N2] = make_float2(zk.x - zk.y, 0.f);  // Nyquist: Re Z0 - Im Z0
      }
    }
  }
}

template <int N2, int MM, int GEN, int FM = -1, int FS = 0>
__global__ void __launch_bounds__(UCfg<N2>::NT, MCQ_UMINB) k_update(UpdateArgs a, const float2* __restrict__ gtw) {
  extern __shared__ __align__(128) float2 sm[];
  update_body<N2, MM, GEN, FM, FS>(a, gtw, blockIdx.x, blockIdx.y, gridDim.x, gridDim.y, sm);
}

int update_grid_blocks(const Dims& d) {
  int ry = 1;
  switch (d.N2) {
#define C_(n) \
  case n:     \
    ry = UCfg<n>::RY; \
    break;
    C_(2) C_(4) C_(8) C_(16) C_(32) C_(64) C_(128) C_(256) C_(512)
#undef C_
    default: break;
  }
  return ((d.ny + ry - 1) / ry) * d.nz;
}

#define MCQ_DISPATCH_N2(Nv, ...)                             \
  switch (Nv) {                                              \
    case 2: { constexpr int N2 = 2; __VA_ARGS__; } break;     \
    case 4: { constexpr int N2 = 4; __VA_ARGS__; } break;     \
    case 8: { constexpr int N2 = 8; __VA_ARGS__; } break;     \
    case 16: { constexpr int N2 = 16; __VA_ARGS__; } break;   \
    case 32: { constexpr int N2 = 32; __VA_ARGS__; } break;   \
    case 64: { constexpr int N2 = 64; __VA_ARGS__; } break;   \
    case 128: { constexpr int N2 = 128; __VA_ARGS__; } break; \
    case 256: { constexpr int N2 = 256; __VA_ARGS__; } break; \
    case 512: { constexpr int N2 = 512; __VA_ARGS__; } break; \
    default: break;                                          \
  }

void launch_update(const UpdateArgs& a, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_N2(a.d.N2, {
    using Cf = UCfg<N2>;
    dim3 grid((a.d.ny + Cf::RY - 1) / Cf::RY, a.d.nz);
    const bool xf = a.dmi[0] != 0.f || a.dmi[1] != 0.f || a.th != 0.f;  // extra field terms
    if (a.mode == MODE_DP && a.nmodes > 1)
      launch_pdl(a.d.pdl, k_update<N2, kMaxModes, 2>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (a.mode == MODE_DP)  // one mode: no per-mode registers (the 4-mode general instance spills)
      launch_pdl(a.d.pdl, k_update<N2, 1, 2>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (xf && a.nmodes > 1)
      launch_pdl(a.d.pdl, k_update<N2, kMaxModes, 2>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (xf)  // DMI / thermal without the Dormand-Prince code
      launch_pdl(a.d.pdl, k_update<N2, 1, 1>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (a.nmodes > 2)
      launch_pdl(a.d.pdl, k_update<N2, kMaxModes, 0>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (a.nmodes == 2)  // two modes (bright + dark): half the per-mode registers of MM = 4
      launch_pdl(a.d.pdl, k_update<N2, 2, 0>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (a.mode == MODE_LLG && a.stage == 1)  // the headline path: plain RK4, one mode, per stage
      launch_pdl(a.d.pdl, k_update<N2, 1, 0, MODE_LLG, 1>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (a.mode == MODE_LLG && a.stage == 2)
      launch_pdl(a.d.pdl, k_update<N2, 1, 0, MODE_LLG, 2>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (a.mode == MODE_LLG && a.stage == 3)
      launch_pdl(a.d.pdl, k_update<N2, 1, 0, MODE_LLG, 3>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else if (a.mode == MODE_LLG)
      launch_pdl(a.d.pdl, k_update<N2, 1, 0, MODE_LLG, 4>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
    else
      launch_pdl(a.d.pdl, k_update<N2, 1, 0>, grid, dim3(Cf::NT), Cf::SMEM, st, a, tw);
  })
}

void configure_update_kernels() {
  for (int n = 2; n <= 512; n *= 2) {
    MCQ_DISPATCH_N2(n, {
      const int smem = (int)UCfg<N2>::SMEM;
      cudaFuncSetAttribute(k_update<N2, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, 1, 0, MODE_LLG, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, 1, 0, MODE_LLG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, 1, 0, MODE_LLG, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, 1, 0, MODE_LLG, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, 2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, kMaxModes, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_update<N2, kMaxModes, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    })
  }
}

// ---------------------------------------------------------------- K-CAV
// Stage factors for the step that starts at (alpha_k, t): Gamma_k(t + c dt) = 2 Re(e_{k,c} alpha_k)
// (P:343 with S_n, C_n frozen, reading C3/C5), excitation a_k sinc(w_k (t + c dt)) (C13), per mode.
__device__ void cav_prepare(const CavParams& p, CavState* st) {
  for (int k = 0; k < p.nmodes; ++k)
    for (int s = 0; s < p.nst; ++s) {  // stage nodes c_s of the integrator (RK4 or Dormand-Prince)
      const double er = p.ec_re[k][s], ei = p.ec_im[k][s];
      const double g = 2.0 * (er * st->re[k] - ei * st->im[k]);
      const double x = p.exc_omega[k] * (st->t + p.cst[s] * p.dt);
      const double sc = (x == 0.0) ? 1.0 : sin(x) / x;
      st->gc[k][s] = (float)(p.cav_on[k] ? g : 0.0);
      st->ge[k][s] = (float)(p.exc_amp[k] * sc);
    }
}

__global__ void k_cav_prepare(CavParams p, CavState* st) {
  if (threadIdx.x == 0 && blockIdx.x == 0) cav_prepare(p, st);
}

// ---- overlap reduction, two fixed-order levels (SURVEY §8(e) "per-plane partials"):
//   level 1, per z plane: the plane's K-U CTAs (nbx of them, consecutive in the slab's partial
//     array [q][CTA], CTA = z * nbx + bx) summed by one warp — lane-strided, then a shuffle tree;
//   level 2, K-CAV: the nzg plane sums [zg][q] summed in global z order the same way.
// The tree depends only on nbx and nzg, never on the slab count, so W, alpha and every later
// step are bitwise the same for any z decomposition, and under NCCL only the nzg x kNPart plane
// sums cross the network (all-gather; 14 KB at 512 planes) instead of every CTA's partials.
__device__ __forceinline__ double warp_sum_fixed(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// one warp: the plane sums of local plane zl of a slab's partials (nps = CTAs per slab)
__device__ __forceinline__ void plane_sum(const double* __restrict__ part, int nps, int nbx, int zl, double* out,
                                          int lane, const bool (&use)[kNPart]) {
#pragma unroll
  for (int q = 0; q < kNPart; ++q) {
    double s = 0.0;
    if (use[q])
      for (int b = lane; b < nbx; b += 32) s += part[(size_t)q * nps + zl * nbx + b];
    s = warp_sum_fixed(s);
    if (lane == 0) out[q] = s;
  }
}

__device__ __forceinline__ void cav_use(const CavParams& p, bool (&use)[kNPart]) {
#pragma unroll
  for (int k = 0; k < kNPart; ++k) use[k] = k < kMaxModes ? k < p.nmodes : p.trace != nullptr;
}

// NCCL mode, before the all-gather: this rank's plane sums psum[zl][q]
__global__ void k_plane_sums(CavParams p, const double* __restrict__ partials, int nps, int nbx, int nzl,
                             double* __restrict__ psum) {
  bool use[kNPart];
  cav_use(p, use);
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int zl = warp; zl < nzl; zl += nw) plane_sum(partials, nps, nbx, zl, psum + (size_t)zl * kNPart, lane, use);
}

// Level 2 (and, unless psum_in is given, level 1 for all slabs held here), then per mode
// alpha_{n+1} = e^{-(kappa + i w) dt} alpha_n + i (V_c/hbar) W_{n+1} dt; t += dt (a13).
// partials: per slab [kNPart][nps] (slab-major); psum_in: gathered plane sums [nzg][kNPart].
// a13 from the reduced sums tot[q]: alpha_{n+1}, t, W, the trace row, the next step's stage
// factors (one thread)
__device__ __forceinline__ void cav_finish(const CavParams& p, CavState* st, const double* tot) {
  for (int k = 0; k < p.nmodes; ++k) {
    const double W = p.cav_on[k] ? p.Ms * tot[k] : 0.0;
    const double er = p.ecn_re[k], ei = p.ecn_im[k];
    const double re = er * st->re[k] - ei * st->im[k];
    const double im = er * st->im[k] + ei * st->re[k] + p.vc_over_hbar * W * p.dt;
    st->re[k] = re;
    st->im[k] = im;
    st->W[k] = W;
  }
  st->t += p.dt;
  st->step += 1;
  if (p.th_count) *p.thstep += 1;  // thermal noise step: never restarted by a memory reset
  if (p.trace && st->step % p.trace_every == 0) {  // NEXT-3: the per-step observables
    const long long r = st->trace_rows;
    if (r < p.trace_cap) {
      double* row = p.trace + r * kTraceCols;
      row[0] = st->t;
      row[1] = tot[kPartM] * p.inv_nmag;
      row[2] = tot[kPartM + 1] * p.inv_nmag;
      row[3] = tot[kPartM + 2] * p.inv_nmag;
      row[4] = st->re[0];
      row[5] = st->im[0];
      row[6] = p.Ms * tot[0];
      row[7] = (double)st->step;
    }
    st->trace_rows = r + 1;
  }
  cav_prepare(p, st);
}

constexpr int kCavThreads = 1024;
constexpr int kMaxPlanes = 512;
__global__ void __launch_bounds__(kCavThreads) k_cavity(CavParams p, CavState* st, const double* __restrict__ partials,
                                                        int nps, int nbx, int nzl, int nzg,
                                                        const double* __restrict__ psum_in) {
  __shared__ double ps[kMaxPlanes * kNPart];
  __shared__ double tot[kNPart];
  pdl_trigger();
  pdl_wait();
  bool use[kNPart];
  cav_use(p, use);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (psum_in) {
    for (int i = threadIdx.x; i < nzg * kNPart; i += kCavThreads) ps[i] = psum_in[i];
  } else {
    for (int zg = warp; zg < nzg; zg += kCavThreads / 32) {
      const int slab = zg / nzl, zl = zg - slab * nzl;
      plane_sum(partials + (size_t)slab * kNPart * nps, nps, nbx, zl, ps + zg * kNPart, lane, use);
    }
  }
  __syncthreads();
  if (warp < kNPart) {  // warp q: the plane sums of quantity q in z order
    double s = 0.0;
    if (use[warp])
      for (int zg = lane; zg < nzg; zg += 32) s += ps[zg * kNPart + warp];
    s = warp_sum_fixed(s);
    if (lane == 0) tot[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) cav_finish(p, st, tot);
}

// ---------------------------------------------------------------- K-P2D: persistent 2D steps
// Grids with nz = 1 and a few thousand cells (BJ configs[0], the 64 x 64 x 1 film of the bias
// sweeps) are launch-latency bound: a step is 9 kernels (4 x (K-Y2D, K-U) + K-CAV) whose work is
// a few microseconds in all (58 us per step measured as separate graph nodes).  One cooperative
// kernel runs all `steps` steps: per stage its CTAs share the K-Y2D work (y forward . Khat .
// y inverse on X, in place), a grid barrier, the K-U work (the same body as k_update, with plain
// staging loads), a barrier; after stage 4 CTA 0 reduces the overlap partials with the same
// fixed-order tree as K-CAV and advances the cavity, a barrier.  The same bodies and arithmetic
// as the separate kernels: bitwise the same trajectory (tests/test_gpu_persist2d.py).
struct Persist2DArgs {
  UpdateArgs u[4];  // stages 1..4
  CavParams cp;
  CavState* cav;
  const float* khat;
  int steps;
  int nbx;    // K-U blocks (ny / RY)
  int nconv;  // K-Y2D blocks
};

template <int N2, int L>
__global__ void __launch_bounds__(UCfg<N2>::NT) k_persist2d(Persist2DArgs pa, const float2* __restrict__ gtw) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) float2 sm[];
  __shared__ double tot[kNPart];
  const Dims& d = pa.u[0].d;
  constexpr int NTT = UCfg<N2>::NT;
  for (int step = 0; step < pa.steps; ++step) {
    for (int s = 0; s < 4; ++s) {
      for (int vb = blockIdx.x; vb < pa.nconv; vb += gridDim.x) {
        conv_body<L, true, NTT>(pa.u[s].X, pa.khat, d, gtw, vb, 0, sm);
        __syncthreads();  // the next virtual block reuses the shared twiddles / exchange buffer
      }
      grid.sync();
      for (int vb = blockIdx.x; vb < pa.nbx; vb += gridDim.x) {
        // the stage-specialised bodies of the graph path's k_update instances (same code, same
        // FMA contraction: bitwise the same results)
        if (s == 0) update_body<N2, 1, 0, MODE_LLG, 1, true>(pa.u[0], gtw, vb, 0, pa.nbx, 1, sm);
        else if (s == 1) update_body<N2, 1, 0, MODE_LLG, 2, true>(pa.u[1], gtw, vb, 0, pa.nbx, 1, sm);
        else if (s == 2) update_body<N2, 1, 0, MODE_LLG, 3, true>(pa.u[2], gtw, vb, 0, pa.nbx, 1, sm);
        else update_body<N2, 1, 0, MODE_LLG, 4, true>(pa.u[3], gtw, vb, 0, pa.nbx, 1, sm);
        __syncthreads();
      }
      grid.sync();
    }
    if (blockIdx.x == 0) {  // K-CAV: one plane, the same two-level fixed-order tree
      bool use[kNPart];
      cav_use(pa.cp, use);
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
      __shared__ double ps[kNPart];
      if (warp == 0) plane_sum(pa.u[3].partials, pa.nbx, pa.nbx, 0, ps, lane, use);
      __syncthreads();
      for (int q = warp; q < kNPart; q += nw) {
        double v = (use[q] && lane == 0) ? ps[q] : 0.0;
        v = warp_sum_fixed(v);
        if (lane == 0) tot[q] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0) cav_finish(pa.cp, pa.cav, tot);
    }
    grid.sync();
  }
}

template <int N2, int L>
static int persist2d_launch(const Persist2DArgs& pa, const float2* tw, cudaStream_t st) {
  using Cu = UCfg<N2>;
  using Cc = ZCfg<L, Cu::NT>;
  const size_t smem = Cu::SMEM > Cc::SMEM ? Cu::SMEM : Cc::SMEM;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_persist2d<N2, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  int per_sm = 0, dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_persist2d<N2, L>, Cu::NT, smem);
  Persist2DArgs copy = pa;
  copy.nbx = (pa.u[0].d.ny + Cu::RY - 1) / Cu::RY;
  copy.nconv = (pa.u[0].d.NKX + Cc::C - 1) / Cc::C;
  int grid = copy.nbx > copy.nconv ? copy.nbx : copy.nconv;
  if (grid > per_sm * nsm) grid = per_sm * nsm;
  if (grid < 1) return -1;
  void* args[] = {&copy, const_cast<float2**>(&tw)};
  return cudaLaunchCooperativeKernel((void*)k_persist2d<N2, L>, dim3(grid), dim3(Cu::NT), args, smem, st) == cudaSuccess
             ? 0
             : -1;
}

int launch_persist2d(const UpdateArgs u[4], const CavParams& cp, CavState* cav, const float* khat, int steps,
                     const float2* tw, cudaStream_t s) {
  Persist2DArgs pa{};
  for (int i = 0; i < 4; ++i) pa.u[i] = u[i];
  pa.cp = cp;
  pa.cav = cav;
  pa.khat = khat;
  pa.steps = steps;
  const int N2 = u[0].d.N2, L = u[0].d.Ly;
#define P2D(n2, l) \
  if (N2 == n2 && L == l) return persist2d_launch<n2, l>(pa, tw, s);
  P2D(32, 64) P2D(32, 128) P2D(64, 64) P2D(64, 128) P2D(64, 256) P2D(128, 128) P2D(128, 256)
#undef P2D
  return -1;
}

void launch_cavity(const CavParams& p, CavState* st, const double* partials, int nps, int nbx, int nzl, int nzg,
                   const double* psum_in, cudaStream_t s) {
  launch_pdl(p.pdl, k_cavity, dim3(1), dim3(kCavThreads), 0, s, p, st, partials, nps, nbx, nzl, nzg, psum_in);
}

void launch_plane_sums(const CavParams& p, const double* partials, int nps, int nbx, int nzl, double* psum,
                       cudaStream_t s) {
  const int warps = nzl < 32 ? nzl : 32;
  k_plane_sums<<<1, 32 * warps, 0, s>>>(p, partials, nps, nbx, nzl, psum);
}

void launch_cav_prepare(const CavParams& p, CavState* st, cudaStream_t s) {
  k_cav_prepare<<<1, 32, 0, s>>>(p, st);
}

// ---------------------------------------------------------------- K-IO
// AoS (interleaved, x fastest) <-> SoA state layout.  `N` cells; the SoA side has component
// stride `cs` and starts `off` cells into each component (halo planes of a z slab).
// aos_to_soa normalises, applies the geometry mask and counts magnetic cells with a zero
// vector in *bad (EINVAL).
__global__ void k_aos_to_soa(const float* __restrict__ in, float* __restrict__ out, const uint8_t* __restrict__ mask,
                             long long N, long long cs, long long off, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    float3 v = make_float3(in[3 * i], in[3 * i + 1], in[3 * i + 2]);
    const bool mag = mask ? (mask[i] != 0) : true;
    if (!mag) {
      v = make_float3(0.f, 0.f, 0.f);
    } else {
      const float n2 = dot3(v, v);
      if (!(n2 > 0.f) || !isfinite(n2)) {
        atomicAdd(bad, 1);
        v = make_float3(0.f, 0.f, 0.f);
      } else if (fabsf(n2 - 1.0f) > 1e-6f) {  // already-unit vectors (a saved state) kept bit-exact
        const float r = 1.0f / sqrtf(n2);
        v = make_float3(v.x * r, v.y * r, v.z * r);
      }
    }
    out[off + i] = v.x;
    out[cs + off + i] = v.y;
    out[2 * cs + off + i] = v.z;
  }
}

__global__ void k_soa_to_aos(const float* __restrict__ in, float* __restrict__ out, long long N, long long cs,
                             long long off) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    out[3 * i] = in[off + i];
    out[3 * i + 1] = in[cs + off + i];
    out[3 * i + 2] = in[2 * cs + off + i];
  }
}

__global__ void k_deinterleave(const float* __restrict__ in, float* __restrict__ out, long long N, long long cs,
                               long long off) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    out[off + i] = in[3 * i];
    out[cs + off + i] = in[3 * i + 1];
    out[2 * cs + off + i] = in[3 * i + 2];
  }
}

static int io_blocks(long long N) {
  long long b = (N + 255) / 256;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

void launch_aos_to_soa(const float* in, float* out, const uint8_t* mask, long long N, long long cs, long long off,
                       int* bad, cudaStream_t s) {
  k_aos_to_soa<<<io_blocks(N), 256, 0, s>>>(in, out, mask, N, cs, off, bad);
}

void launch_soa_to_aos(const float* in, float* out, long long N, long long cs, long long off, cudaStream_t s) {
  k_soa_to_aos<<<io_blocks(N), 256, 0, s>>>(in, out, N, cs, off);
}

void launch_deinterleave(const float* in, float* out, long long N, long long cs, long long off, cudaStream_t s) {
  k_deinterleave<<<io_blocks(N), 256, 0, s>>>(in, out, N, cs, off);
}

}  // namespace mcq
