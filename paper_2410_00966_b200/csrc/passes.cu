// passes.cu — the y and z passes of the zero-padded demag FFT convolution (a2-a4 of SURVEY §8(a)).
//
// B_demag = -mu0 IFFT( Khat . FFT(M) ) restricted to the grid, with M = Ms m zero-padded to
// (Lx, Ly, Lz) (reading C11).  The x transforms live in the update kernel (update.cu); here,
// with the row layout of common.cuh (kx fastest):
//   K-Y  (k_yfwd):  X[3][nz][ny][P] -> Y[3][nz][Ly][P], forward along y, input rows >= ny are 0
//   K-Z  (k_zconv): per (ky, kx) column of Y: forward along z (planes >= nz are 0), the
//                   symmetric 3x3 multiply by the real folded Khat, inverse along z, keep nz
//   K-YI (k_yinv):  Y -> X, inverse along y, keep the first ny rows
//   K-Y2D(k_y2d):   nz == 1: forward y, Khat multiply, inverse y in one pass, in place on X
// A CTA owns C adjacent kx columns (a warp's global accesses are contiguous C*8-byte row
// segments).  Lines are transformed with the register-resident FFT of regfft.cuh: data go
// HBM -> registers -> (S-1 smem exchanges) -> registers -> HBM; K-Z / K-Y2D keep the three
// components of a column in one thread and multiply by Khat in registers between the forward
// and the inverse transform.
// (A thread-block-cluster variant fusing y and z per kx plane through DSMEM was built and
// measured 2-3x slower than this schedule on B200 — shared-memory-limited occupancy in a
// compute-bound pass.)
#include <cuda.h>  // CUtensorMap (the encode call itself goes through cudaGetDriverEntryPoint)

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "regfft.cuh"
#include "tma.cuh"
#include "conv.cuh"
#include "zconv2.cuh"
#include "zconv3.cuh"

namespace mcq {

// CW > 0: a configuration with CW columns per CTA (a separate narrow launch for the last kx
// column beyond the final 16-column tile was measured slower: the extra kernel boundary costs
// more than the mostly idle tile it replaces)
#ifndef MCQ_YE
#define MCQ_YE 16   // points per thread per line in K-Y / K-YI
#endif
#ifndef MCQ_YNT
#define MCQ_YNT 256  // target threads per CTA in K-Y / K-YI
#endif
#ifndef MCQ_YCMIN
#define MCQ_YCMIN 8  // fewest kx columns per K-Y / K-YI CTA (64-byte row segments; sets C at L = 1024)
#endif
template <int L, int CW = 0>
struct PassCfg {  // single-component passes (K-Y, K-YI)
  static constexpr int E = L < MCQ_YE ? L : MCQ_YE;
  static constexpr int TL = L / E;
  static constexpr int C0 = MCQ_YNT / TL;
  static constexpr int C = CW > 0 ? CW : (C0 < MCQ_YCMIN ? MCQ_YCMIN : (C0 > 64 ? 64 : C0));
  static constexpr int NT = C * TL;
  static constexpr int TWN = pass_twn<L, E>();  // twiddle table (complex)
  static constexpr size_t SMEM = (size_t)(TWN + (TL > 1 ? L * C : 0)) * sizeof(float2);
};

// ---------------------------------------------------------------- K-Y forward / inverse
// grid (column tiles, 3 nz): blockIdx.y = (z descending, component inner) — the passes meet the
// planes the previous kernel (K-U, z ascending) wrote last, while they are still in L2.
// SPLIT: kx-slab-major Y (z slabs over NS ranks, common.cuh); the single-slab instance has no
// owner arithmetic.  No integer division in the prologue (it was ~1/4 of a thread's work).
template <int L, bool INV, bool SPLIT, int CW = 0>
__global__ void __launch_bounds__(PassCfg<L, CW>::NT) k_ypass(const float2* __restrict__ in, float2* __restrict__ out,
                                                              Dims d, const float2* __restrict__ gtw, int comp0,
                                                              int ncomp) {
  using Cf = PassCfg<L, CW>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C;
  extern __shared__ __align__(128) float2 sm[];
  float2* tw = sm;  // plan twiddles
  pdl_trigger();
  pass_tw<L, E, Cf::NT>(tw, gtw);
  __syncthreads();
  pdl_wait();
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  // components [comp0, comp0 + ncomp): all three in one launch, or one at a time when the slab
  // transpose of each component overlaps the next component's pass (mcq.cu, Enq::demag)
  const int rest = blockIdx.y, comp = comp0 + (ncomp == 3 ? rest % 3 : 0), z = d.nz - 1 - (ncomp == 3 ? rest / 3 : rest);
  const int kx = blockIdx.x * C + c;
  const bool ok = kx < d.NKX;
  const int nin = INV ? L : d.ny, nout = INV ? d.ny : L;
  // X side: X[c][z][y][P]; Y side: Y[q][c][z][ky][KXS] (q = kx slab; single slab: Y[c][z][ky][P])
  int q = 0, kxl = kx;
  if constexpr (SPLIT) {
    q = kx_owner(d, kx);
    kxl = kx - (q > 0 ? kx_first(d, q) : 0);
  }
  // 32-bit element indices (every buffer holds < 2^32 elements)
  const unsigned xoff = ((unsigned)(comp * d.nz + z) * d.ny) * d.P + kx;
  const unsigned yoff = ((unsigned)(q * 3 + comp) * d.nz + z) * (unsigned)L * d.KXS + kxl;
  const unsigned sin_ = INV ? d.KXS : d.P, sout = INV ? d.P : d.KXS;
  // this thread's first row and the step between its rows (32-bit offsets from the uniform base)
  const unsigned ib = (INV ? yoff : xoff) + (unsigned)t * sin_, ob = (INV ? xoff : yoff) + (unsigned)t * sout;
  const unsigned istep = (unsigned)TL * sin_, ostep = (unsigned)TL * sout;
  float2 v[1][E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int p = t + TL * i;
    // zero padding: forward input rows >= ny <= Ly/2 are zero, i.e. every i >= E/2 (p >= L/2)
    // statically, so the first stage's butterflies fold those operands away
    v[0][i] = (!INV && 2 * i >= E) ? make_float2(0.f, 0.f)
                                  : ((ok && p < nin) ? in[ib + i * istep] : make_float2(0.f, 0.f));
  }
  reg_fft<L, E, 1, INV, PASS_TWS>(v, sm + Cf::TWN, ColAddr<L, C>{c}, tw, t);
  if (ok) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      if ((!INV || 2 * i < E) && p < nout) out[ob + i * ostep] = v[0][i];  // inverse: rows < ny only
    }
  }
}

// ---------------------------------------------------------------- K-Z, component-sequential
// Low-register variant: the three component lines of a column pass through the register FFT
// one after another (a thread holds E points of ONE line at a time); forward results are parked
// in the shared exchange buffer at the thread's own positions, the K-hat multiply reads and
// writes them there, and the inverse transforms reload them.  ~60 registers instead of ~128, so
// twice the warps per SM for the same shared memory.
#ifndef MCQ_ZSE
#define MCQ_ZSE 16  // points per thread per line in the component-sequential K-Z
#endif
#ifndef MCQ_ZTAB
#define MCQ_ZTAB 1  // plan twiddle table in K-Z (fewer registers: 64 vs 104)
#endif
#ifndef MCQ_ZPF
#define MCQ_ZPF 1   // load component g+1 before transforming g (with ZTAB: 123.3 vs 127.3 us)
#endif
#ifndef MCQ_ZNT
#define MCQ_ZNT 256  // target threads per CTA in K-Z
#endif
#ifndef MCQ_ZPAIR
#define MCQ_ZPAIR 1  // order K-Z rows as (0, Ly/2, 1, Ly-1, 2, ...): shared Khat rows back to back (1.025 vs 1.036 ms/step)
#endif
template <int L, int CW = 0>
struct ZSCfg {
  static constexpr int E = L <= MCQ_ZSE ? L : MCQ_ZSE;
  static constexpr int TL = L / E;
  static constexpr int C0 = MCQ_ZNT / TL;
  static constexpr int C = CW > 0 ? CW : (C0 < 4 ? 4 : (C0 > 64 ? 64 : C0));
  static constexpr int NT = C * TL;
  static constexpr int TWS = MCQ_ZTAB ? 0 : 1;
  static constexpr int TWN = MCQ_ZTAB ? reg_tw_size<L, E>() : (L < 2 ? 2 : L);
  static constexpr size_t SMEM = (size_t)(TWN + 3 * L * C) * sizeof(float2);
};

template <int L, bool SPLIT, int CW = 0>
__global__ void __launch_bounds__(ZSCfg<L, CW>::NT) k_zconv_seq(float2* __restrict__ Y, const float* __restrict__ khat,
                                                                Dims d, const float2* __restrict__ gtw, int nfull) {
  using Cf = ZSCfg<L, CW>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C;
  extern __shared__ __align__(128) float2 sm[];
  float2* tw = sm;
  float2* xch = sm + Cf::TWN;  // [3][L][C]
  pdl_trigger();
  if constexpr (Cf::TWS == 0) {
    reg_tw_build<L, E, Cf::NT>(tw, gtw);
  } else {
    for (int m = threadIdx.x; m < L; m += Cf::NT) tw[m] = gtw[m * (kTwMax / L)];
  }
  __syncthreads();
  pdl_wait();
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  // columns kxl of this rank's kx slab (global kx = kx0 + kxl); z runs over all nzg planes,
  // held as [source rank r][c][zl][ky][KXS] with z = r * nz + zl (NS == 1: Y[c][z][ky][P])
  // the first nlone CTAs are lone-column CTAs whose C lanes take C rows ky of this slab's last
  // column (kxw = C * nfull + 1); the others are column tile (b % nfull) at row b / nfull
  const int nlone = gridDim.x - nfull * d.Ly;
  const bool lone = (int)blockIdx.x < nlone;
  const int b = blockIdx.x - nlone;
  const int kxl = lone ? d.kxw - 1 : (b % nfull) * C + c, kx = d.kx0 + kxl;
#if MCQ_ZPAIR
  // rows ky and Ly - ky read the same folded Khat rows: schedule them back to back (L2 reuse)
  const int kyi = b / nfull, kyh = kyi >> 1;
  const int kyn = kyi == 1 ? d.Ly / 2 : ((kyi & 1) ? d.Ly - kyh : kyh);
#else
  const int kyn = b / nfull;
#endif
  const int ky = lone ? blockIdx.x * C + c : kyn;
  const bool ok = kxl < d.kxw && ky < d.Ly;
  const int kyc = ky < d.Ly ? ky : d.Ly - 1;  // in-range row for address arithmetic
  const int nz = d.nzg, nzl = d.nz;
  // 32-bit element indices (Y holds < 2^32 elements)
  const unsigned row = d.KXS, plane = (unsigned)d.Ly * row;
  const unsigned cbase = (unsigned)kyc * row + kxl;
  // ((r * 3 + g) * nzl + z - r * nzl) planes = g * nzl + z + 2 nzl r with r = z / nzl (SPLIT
  // only: the single-slab instance keeps the plain strength-reduced addressing)
  const unsigned cstr = (unsigned)nzl * plane;
  // z / nzl in fp32: (z + 1/2) / nzl is >= 1/(2 nzl) >= 1e-3 away from an integer and the
  // rounding error is ~1e-7 relative, so the truncation is exact (z < 1024)
  const float inv_nzl = 1.f / (float)nzl;
  auto zaddr = [&](int g, int z) -> unsigned {
    unsigned a = cbase + (unsigned)g * cstr + (unsigned)z * plane;
    if constexpr (SPLIT) a += (unsigned)(2 * nzl * __float2int_rz(((float)z + 0.5f) * inv_nzl)) * plane;
    return a;
  };
  struct GA {
    int g, c;
    __device__ __forceinline__ int operator()(int, int pos) const { return (g * L + pos) * C + c; }
  };
  constexpr int EH = E / 2 > 0 ? E / 2 : 1;  // a thread's nonzero inputs (nz <= L/2)
  float2 pf[EH];
  if constexpr (MCQ_ZPF) {
#pragma unroll
    for (int i = 0; i < EH; ++i) {
      const int p = t + TL * i;
      pf[i] = (ok && p < nz) ? Y[zaddr(0, p)] : make_float2(0.f, 0.f);
    }
  }
#pragma unroll 1
  for (int g = 0; g < 3; ++g) {
    float2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      if constexpr (MCQ_ZPF)
        v[0][i] = 2 * i < E ? pf[i < EH ? i : 0] : make_float2(0.f, 0.f);
      else
        v[0][i] = (2 * i < E && ok && p < nz) ? Y[zaddr(g, p)] : make_float2(0.f, 0.f);
    }
    if constexpr (MCQ_ZPF) {
      if (g < 2) {
#pragma unroll
        for (int i = 0; i < EH; ++i) {
          const int p = t + TL * i;
          pf[i] = (ok && p < nz) ? Y[zaddr(g + 1, p)] : make_float2(0.f, 0.f);
        }
      }
    }
    const GA A{g, c};
    reg_fft<L, E, 1, false, Cf::TWS>(v, xch, A, tw, t);
#pragma unroll
    for (int i = 0; i < E; ++i) xch[A(0, t + TL * i)] = v[0][i];
  }
  if (ok) {  // own positions only: no barrier needed
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      float2 mx = xch[(0 * L + p) * C + c], my = xch[(1 * L + p) * C + c], mz = xch[(2 * L + p) * C + c];
      khat_apply(khat, d, kx, ky, p, mx, my, mz);
      xch[(0 * L + p) * C + c] = mx;
      xch[(1 * L + p) * C + c] = my;
      xch[(2 * L + p) * C + c] = mz;
    }
  }
#pragma unroll 1
  for (int g = 0; g < 3; ++g) {
    const GA A{g, c};
    float2 v[1][E];
#pragma unroll
    for (int i = 0; i < E; ++i) v[0][i] = xch[A(0, t + TL * i)];
    __syncthreads();  // region g is read before its exchanges overwrite it
    reg_fft<L, E, 1, true, Cf::TWS>(v, xch, A, tw, t);
    if (ok) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int p = t + TL * i;
        if (2 * i < E && p < nz) Y[zaddr(g, p)] = v[0][i];
      }
    }
  }
}

// ---------------------------------------------------------------- K-Z, TMA-pipelined
// Persistent CTAs loop over (kx tile, ky) tiles.  For each tile the TMA engine brings the three
// components' nz x C input boxes of Y into a shared-memory stage (3 tensor copies, one
// mbarrier); the copy of the next tile is in flight while this one is transformed (two
// stages), so the SM never waits on HBM latency with its registers idle.
template <int L>
#ifndef MCQ_ZTE
#define MCQ_ZTE 8  // points per thread per line in the pipelined K-Z
#endif
struct ZTCfg {
  static constexpr int E = L <= 16 ? L : MCQ_ZTE;
  static constexpr int TL = L / E;
  static constexpr int C0 = 256 / TL;
  static constexpr int C = C0 < 4 ? 4 : (C0 > 64 ? 64 : C0);
  static constexpr int NT = C * TL;
  static constexpr int TWP = (pass_twn<L, E>() + 15) / 16 * 16;  // twiddle slots, keeps the stages 128 B aligned
  static constexpr int GS = ((L / 2) * C + 15) / 16 * 16;  // per-component box stride (128 B aligned)
  static constexpr int STAGE = 3 * GS;                     // complex per input stage (nz <= L/2)
  static constexpr size_t SMEM = (size_t)(TWP + 2 * STAGE + (TL > 1 ? 3 * L * C : 0)) * sizeof(float2);
};

template <int L, int MINB>
__global__ void __launch_bounds__(ZTCfg<L>::NT, MINB) k_zconv_tma(const __grid_constant__ CUtensorMap tm,
                                                            float2* __restrict__ Y, const float* __restrict__ khat,
                                                            Dims d, const float2* __restrict__ gtw, int ntiles) {
  using Cf = ZTCfg<L>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C;
  extern __shared__ __align__(128) float2 sm[];
  float2* tw = sm;
  float2* stg = sm + Cf::TWP;                 // [2][3][GS]: input stages ([nz][C] per component)
  float2* xch = stg + 2 * Cf::STAGE;          // [3][L][C]
  __shared__ __align__(8) uint64_t bar[2];
  const int nz = d.nz;
  const int nkt = (d.NKX + C - 1) / C;
  const uint32_t box_bytes = (uint32_t)(3 * nz * C * sizeof(float2));
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  pdl_trigger();
  pass_tw<L, E, Cf::NT>(tw, gtw);
  __syncthreads();
  pdl_wait();
  auto issue = [&](int tile, int b) {
    const int kx0 = (tile % nkt) * C, ky = tile / nkt;
    mbar_arrive_expect_tx(&bar[b], box_bytes);
    for (int g = 0; g < 3; ++g) tma_load_3d(stg + b * Cf::STAGE + g * Cf::GS, &tm, kx0, ky, g * nz, &bar[b]);
  };
  if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  const ColAddr<L, C> A{c};
  const size_t plane = (size_t)d.Ly * d.P, cstr = (size_t)nz * plane;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int b = it & 1;
    const int next = tile + gridDim.x;
    if (threadIdx.x == 0 && next < ntiles) issue(next, b ^ 1);
    mbar_wait(&bar[b], (it >> 1) & 1);
    const int kx = (tile % nkt) * C + c, ky = tile / nkt;
    const float2* in = stg + b * Cf::STAGE;
    float2 v[3][E];
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int p = t + TL * i;
        v[g][i] = (2 * i < E && p < nz) ? in[g * Cf::GS + p * C + c] : make_float2(0.f, 0.f);
      }
    reg_fft<L, E, 3, false, PASS_TWS>(v, xch, A, tw, t);
    const bool ok = kx < d.NKX;
    if (ok) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        khat_apply(khat, d, kx, ky, t + TL * i, v[0][i], v[1][i], v[2][i]);
        if ((i & 1) == 1) asm volatile("" ::: "memory");
      }
    }
    reg_fft<L, E, 3, true, PASS_TWS>(v, xch, A, tw, t);
    if (ok) {
      float2* base = Y + (size_t)ky * d.P + kx;
#pragma unroll
      for (int g = 0; g < 3; ++g)
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int p = t + TL * i;
          if (2 * i < E && p < nz) base[g * cstr + p * plane] = v[g][i];
        }
    }
    __syncthreads();  // stage b and xch are free for the next issue / tile
  }
}

// ---------------------------------------------------------------- dispatch
#define MCQ_DISPATCH_L(Lval, ...)                              \
  switch (Lval) {                                              \
    case 2: { constexpr int L = 2; __VA_ARGS__; } break;       \
    case 4: { constexpr int L = 4; __VA_ARGS__; } break;       \
    case 8: { constexpr int L = 8; __VA_ARGS__; } break;       \
    case 16: { constexpr int L = 16; __VA_ARGS__; } break;     \
    case 32: { constexpr int L = 32; __VA_ARGS__; } break;     \
    case 64: { constexpr int L = 64; __VA_ARGS__; } break;     \
    case 128: { constexpr int L = 128; __VA_ARGS__; } break;   \
    case 256: { constexpr int L = 256; __VA_ARGS__; } break;   \
    case 512: { constexpr int L = 512; __VA_ARGS__; } break;   \
    case 1024: { constexpr int L = 1024; __VA_ARGS__; } break; \
    default: break;                                            \
  }

// (lone-column CTAs as in K-Z measured slower here: 38.9 / 37.8 vs 37.8 / 35.6 us)
template <bool INV>
static int launch_ypass(const Dims& d, const float2* in, float2* out, const float2* tw, int comp, cudaStream_t st) {
  int n = 0;
  const int c0 = comp < 0 ? 0 : comp, nc = comp < 0 ? 3 : 1;
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = PassCfg<L>;
    const dim3 grid((d.NKX + Cf::C - 1) / Cf::C, nc * d.nz);
    if (d.NS > 1)
      launch_pdl(d.pdl, k_ypass<L, INV, true>, grid, dim3(Cf::NT), Cf::SMEM, st, in, out, d, tw, c0, nc);
    else
      launch_pdl(d.pdl, k_ypass<L, INV, false>, grid, dim3(Cf::NT), Cf::SMEM, st, in, out, d, tw, c0, nc);
    ++n;
  })
  return n;
}

int launch_yfwd(const Dims& d, const float2* X, float2* Y, const float2* tw, cudaStream_t st, int comp) {
  return launch_ypass<false>(d, X, Y, tw, comp, st);
}

int launch_yinv(const Dims& d, const float2* Y, float2* X, const float2* tw, cudaStream_t st, int comp) {
  return launch_ypass<true>(d, Y, X, tw, comp, st);
}

int launch_zconv(const Dims& d, float2* Y, const float* khat, const float2* tw, cudaStream_t st) {
  int n = 0;
  MCQ_DISPATCH_L(d.Lz, {
    using Cf = ZCfg<L>;
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C, d.Ly);
    launch_pdl(d.pdl, k_conv<L, false>, grid, dim3(Cf::NT), Cf::SMEM, st, Y, khat, d, tw), ++n;
  })
  return n;
}

template <int L, bool SPLIT>
static int zconv_seq_cols(const Dims& d, float2* Y, const float* khat, const float2* tw, int cols, cudaStream_t st) {
  using Cf = ZSCfg<L>;
  const bool lone = cols % Cf::C == 1 && cols > Cf::C;
  const int nfull = lone ? cols / Cf::C : (cols + Cf::C - 1) / Cf::C;
  const int nb = nfull * d.Ly + (lone ? (d.Ly + Cf::C - 1) / Cf::C : 0);
  launch_pdl(d.pdl, k_zconv_seq<L, SPLIT>, dim3(nb), dim3(Cf::NT), Cf::SMEM, st, Y, khat, d, tw, nfull);
  return 1;
}

static int sm_count() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

// K-Z v2 (zconv2.cuh) for Lz = 256 / 512: persistent, 2 CTAs per SM (MCQ_Z2PERSIST = 0: one
// CTA per tile)
// single slab: TMA-staged z columns in K-Z v2 (measured, non-persistent: Lz = 512 3.89 vs 4.51 ms
// with the register prefetch of the next component, which costs 32 registers there; Lz = 256
// 153 vs 110 us — its 8-slot register prefetch is cheap and the TMA lead time short)
#ifndef MCQ_Z2TMA_256
#define MCQ_Z2TMA_256 0
#endif
#ifndef MCQ_Z2TMA_512
#define MCQ_Z2TMA_512 1
#endif

#ifndef MCQ_Z2PERSIST
#define MCQ_Z2PERSIST 0  // one CTA per tile: configs[4] 4.49 vs 5.33 ms, configs[1] 110 vs 153 us (persistent)
#endif
#ifndef MCQ_Z3
#define MCQ_Z3 1  // Lz = 512 (single slab): K-Z v3 (zconv3.cuh); 0: v2 with TMA-staged columns
#endif
#ifndef MCQ_Z3_SPLIT
#define MCQ_Z3_SPLIT 1  // z slabs (received kx-slab blocks, 4D TMA boxes): K-Z v3 too
#endif
#ifndef MCQ_Z3_256
#define MCQ_Z3_256 0  // Lz = 256 (single slab): K-Z v3 (parity-tested, measured slower: 126.6 vs 105.6
                      // us at configs[1] — one channel leaves v2 no hand-over to save); 0: v2
#endif

template <int L, bool SPLIT>
static int zconv2_cols(const Dims& d, float2* Y, const float* khat, const float2* tw, int cols, const void* tmap,
                       cudaStream_t st, bool khat_map = false) {
  using Z = Z2Cfg<L>;
  const int rem = cols % Z::C;
  const int nkt = cols / Z::C + (rem > 1 ? 1 : 0);
  const int nlone = rem == 1 ? (d.Ly + Z::C - 1) / Z::C : 0;
  const int ntiles = nlone + nkt * d.Ly;
  CUtensorMap none;
  memset(&none, 0, sizeof(none));
  if (tmap && khat_map && (L == 512 ? MCQ_Z3 : MCQ_Z3_256) && d.nzg <= L / 2 && (!SPLIT || MCQ_Z3_SPLIT)) {
    // K-Z v3 (zconv3.cuh): 16-column tiles, persistent, MINB CTAs per SM; the lone Nyquist
    // column (NKX = 16 q + 1) by v2's lone-tile launch.  tmap: [v2 box, v3 box, Khat]
    using Z3 = Z3Cfg<L>;
    const CUtensorMap* tm3 = reinterpret_cast<const CUtensorMap*>(tmap) + 1;
    const int rem3 = cols % Z3::C;
    const int nkt3 = cols / Z3::C + (rem3 > 1 ? 1 : 0);
    const int nt3 = nkt3 * d.Ly;
    int n = 0;
    if (nt3 > 0)
      launch_pdl(d.pdl, k_zconv3<L, SPLIT>, dim3(std::min(nt3, Z3::MINB * sm_count())), dim3(Z3::NT), Z3::SMEM, st,
                 Y, khat, d, tw, nkt3, nt3, tm3[0], tm3[1]), ++n;
    if (rem3 == 1) {
      const int nl = (d.Ly + Z::C - 1) / Z::C;
      launch_pdl(d.pdl, k_zconv2<L, SPLIT, false>, dim3(nl), dim3(Z::NT), Z::SMEM, st, Y, khat, d, tw, nkt, nl, nl, 0,
                 none), ++n;
    }
    return n;
  }
  if (!SPLIT && tmap && (L == 256 ? MCQ_Z2TMA_256 : MCQ_Z2TMA_512)) {
    // normal tiles: TMA-staged inputs (persistent); the lone Nyquist-column tiles (if any): the
    // load path, a small launch of its own
    const CUtensorMap& tm = *reinterpret_cast<const CUtensorMap*>(tmap);
    const int nnorm = ntiles - nlone;
    const int grid = MCQ_Z2PERSIST ? std::min(nnorm, Z::MINB * sm_count()) : nnorm;
    int n = 0;
    if (nnorm > 0)
      launch_pdl(d.pdl, k_zconv2<L, false, true>, dim3(grid), dim3(Z::NT), Z::SMEM, st, Y, khat, d, tw, nkt, nlone,
                 ntiles, nlone, tm), ++n;
    if (nlone > 0)
      launch_pdl(d.pdl, k_zconv2<L, false, false>, dim3(nlone), dim3(Z::NT), Z::SMEM, st, Y, khat, d, tw, nkt, nlone,
                 nlone, 0, none), ++n;
    return n;
  }
  const int grid = MCQ_Z2PERSIST ? std::min(ntiles, Z::MINB * sm_count()) : ntiles;
  launch_pdl(d.pdl, k_zconv2<L, SPLIT>, dim3(grid), dim3(Z::NT), Z::SMEM, st, Y, khat, d, tw, nkt, nlone, ntiles, 0,
             none);
  return 1;
}

#ifndef MCQ_ZV2_256
#define MCQ_ZV2_256 1
#endif
#ifndef MCQ_ZV2_512
#define MCQ_ZV2_512 1
#endif

int launch_zconv_seq(const Dims& d, float2* Y, const float* khat, const float2* tw, cudaStream_t st,
                     const void* tmap2, bool khat_map) {
  const int cols = d.kxw;  // valid columns of this slab
  if (cols <= 0) return 0;
  static const char* zv = getenv("MCQ_ZVARIANT");  // experiment override: seq | v2
  bool v2 = d.Lz == 256 ? MCQ_ZV2_256 : MCQ_ZV2_512;
  if (zv && !strcmp(zv, "seq")) v2 = false;
  if (zv && !strcmp(zv, "v2")) v2 = true;
  if (v2 && d.Lz == 256) return d.NS > 1 ? zconv2_cols<256, true>(d, Y, khat, tw, cols, tmap2, st, khat_map)
                                         : zconv2_cols<256, false>(d, Y, khat, tw, cols, tmap2, st, khat_map);
  if (v2 && d.Lz == 512) return d.NS > 1 ? zconv2_cols<512, true>(d, Y, khat, tw, cols, tmap2, st, khat_map)
                                         : zconv2_cols<512, false>(d, Y, khat, tw, cols, tmap2, st, khat_map);
  int n = 0;
  MCQ_DISPATCH_L(d.Lz, {
    n = d.NS > 1 ? zconv_seq_cols<L, true>(d, Y, khat, tw, cols, st) : zconv_seq_cols<L, false>(d, Y, khat, tw, cols, st);
  })
  return n;
}

int zconv2_box_c(int Lz) { return Lz == 256 ? Z2Cfg<256>::C : (Lz == 512 ? Z2Cfg<512>::C : 0); }

int zconv_tma_box_c(int Lz) {
  int c = 0;
  MCQ_DISPATCH_L(Lz, c = ZTCfg<L>::C)
  return c;
}

int launch_zconv_tma(const Dims& d, const void* tmap, float2* Y, const float* khat, const float2* tw,
                     cudaStream_t st) {
  int n = 0;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  static const int minb = getenv("MCQ_ZMINB") ? atoi(getenv("MCQ_ZMINB")) : 1;  // experiment knob
  MCQ_DISPATCH_L(d.Lz, {
    using Cf = ZTCfg<L>;
    static int per_sm[2] = {0, 0};
    const int v = minb >= 3 ? 1 : 0;
    if (!per_sm[v])
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[v], v ? k_zconv_tma<L, 3> : k_zconv_tma<L, 1>, Cf::NT,
                                                    Cf::SMEM);
    const int ntiles = ((d.NKX + Cf::C - 1) / Cf::C) * d.Ly;
    const int cap = nsm * (per_sm[v] > 0 ? per_sm[v] : 1);
    const int grid = ntiles < cap ? ntiles : cap;
    const CUtensorMap& tmr = *reinterpret_cast<const CUtensorMap*>(tmap);
    if (v)
      launch_pdl(d.pdl, k_zconv_tma<L, 3>, dim3(grid), dim3(Cf::NT), Cf::SMEM, st, tmr, Y, khat, d, tw, ntiles);
    else
      launch_pdl(d.pdl, k_zconv_tma<L, 1>, dim3(grid), dim3(Cf::NT), Cf::SMEM, st, tmr, Y, khat, d, tw, ntiles);
    n = 1;
  })
  return n;
}

int launch_y2d(const Dims& d, float2* X, const float* khat, const float2* tw, cudaStream_t st) {
  int n = 0;
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = ZCfg<L>;
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C);
    launch_pdl(d.pdl, k_conv<L, true>, grid, dim3(Cf::NT), Cf::SMEM, st, X, khat, d, tw), ++n;
  })
  return n;
}

// Opt every instantiation into the shared memory it needs (once per process).
void configure_pass_kernels() {
  for (int Lv = 2; Lv <= 1024; Lv *= 2) {
    MCQ_DISPATCH_L(Lv, {
      cudaFuncSetAttribute(k_ypass<L, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PassCfg<L>::SMEM);
      cudaFuncSetAttribute(k_ypass<L, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PassCfg<L>::SMEM);
      cudaFuncSetAttribute(k_ypass<L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PassCfg<L>::SMEM);
      cudaFuncSetAttribute(k_ypass<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PassCfg<L>::SMEM);
      cudaFuncSetAttribute(k_conv<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZCfg<L>::SMEM);
      cudaFuncSetAttribute(k_conv<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZCfg<L>::SMEM);
      cudaFuncSetAttribute(k_zconv_tma<L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZTCfg<L>::SMEM);
      cudaFuncSetAttribute(k_zconv_seq<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZSCfg<L>::SMEM);
      cudaFuncSetAttribute(k_zconv_seq<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZSCfg<L>::SMEM);
      cudaFuncSetAttribute(k_zconv_tma<L, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZTCfg<L>::SMEM);
    })
  }
  cudaFuncSetAttribute(k_zconv2<256, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cfg<256>::SMEM);
  cudaFuncSetAttribute(k_zconv2<512, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cfg<512>::SMEM);
  cudaFuncSetAttribute(k_zconv2<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cfg<256>::SMEM);
  cudaFuncSetAttribute(k_zconv2<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cfg<256>::SMEM);
  cudaFuncSetAttribute(k_zconv2<512, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cfg<512>::SMEM);
  cudaFuncSetAttribute(k_zconv2<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cfg<512>::SMEM);
  cudaFuncSetAttribute(k_zconv3<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z3Cfg<256>::SMEM);
  cudaFuncSetAttribute(k_zconv3<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z3Cfg<512>::SMEM);
  cudaFuncSetAttribute(k_zconv3<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z3Cfg<256>::SMEM);
  cudaFuncSetAttribute(k_zconv3<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z3Cfg<512>::SMEM);
  cudaGetLastError();
}

}  // namespace mcq
