// passes.cu — the y and z passes of the zero-padded demag FFT convolution (a2-a4 of SURVEY §8(a)).
//
// B_demag = -mu0 IFFT( Khat . FFT(M) ) restricted to the grid, with M = Ms m zero-padded to
// (Lx, Ly, Lz) (reading C11).  The x transforms live in the update kernel (update.cu).  All
// spectra are kx-major: X[kx][c][z][y], Y[kx][c][z][ky], Khat[kx][6][kz][ky] (common.cuh).
//
//   K-YZ  (k_yz, default for 3D grids whose kx plane fits a cluster): one thread-block cluster
//         per kx plane.  Phase 1: each CTA y-transforms its z-slab (ny -> Ly, pruned input) into
//         its shared memory.  Phase 2: each CTA takes a ky-slab, gathers the z lines from all
//         CTAs' shared memory (DSMEM), z-transforms (nz -> Lz), multiplies by Khat, inverse
//         z-transforms and scatters the nz kept values back.  Phase 3: inverse y, keep ny rows,
//         write X in place.  HBM traffic: read X, read Khat, write X — the Y round trips of the
//         3-pass schedule never happen.
//   3-pass fallback (planes too large for a cluster, e.g. 512x512x256):
//   K-Y   (k_yfwd):  X -> Y, forward along y;   K-Z (k_zconv): z fwd * Khat * z inv on Y;
//   K-YI  (k_yinv):  Y -> X, inverse along y.
//   K-Y2D (k_y2d):   nz == 1: forward y, Khat multiply, inverse y in one pass, in place on X.
// Lines are transformed with the register-resident FFT of regfft.cuh.
#include <cooperative_groups.h>

#include "common.cuh"
#include "regfft.cuh"

namespace cg = cooperative_groups;

namespace mcq {

template <int L>
__device__ __forceinline__ void load_tw(float2* tw, const float2* __restrict__ gtw) {
  for (int m = threadIdx.x; m < L; m += blockDim.x) tw[m] = gtw[m * (kTwMax / L)];
}

template <int L>
struct RowPitch {  // padded row of L complex: one pad slot every 16 (conflict-free radix-16 stores)
  static constexpr int P = L + (L >= 16 ? L / 16 : 1);
  __device__ static __forceinline__ int at(int pos) { return pos + (L >= 16 ? (pos >> 4) : 0); }
};

template <int L>
struct RowA {  // shared-memory address of element pos of row `line`
  int line;
  __device__ __forceinline__ int operator()(int, int pos) const { return line * RowPitch<L>::P + RowPitch<L>::at(pos); }
};

// B_g = sum_h Khat_gh M_h for row g of the symmetric tensor, with the fold signs
// (XY odd in y, XZ odd in z, YZ odd in both; kx is never folded).
struct KRow {
  int cd, co0, co1, h0, h1;
  __device__ __forceinline__ explicit KRow(int g)
      : cd(g), co0(g == 2 ? 4 : 3), co1(g == 0 ? 4 : 5), h0(g == 0 ? 1 : 0), h1(g == 2 ? 1 : 2) {}
};

__device__ __forceinline__ float fold_sign(int comp, float sy, float sz) {
  return comp == 3 ? sy : (comp == 4 ? sz : (comp == 5 ? sy * sz : 1.f));
}

// ====================================================================== K-YZ (cluster)
template <int LY, int LZ>
struct YZCfg {
  static constexpr int EY = LY < 16 ? LY : 16;
  static constexpr int TLY = LY / EY;
  static constexpr int EZ = LZ <= 16 ? LZ : 8;
  static constexpr int TLZ = LZ / EZ;
  static constexpr int PY = RowPitch<LY>::P;
};

template <int LY, int LZ>
__global__ void __launch_bounds__(512) k_yz(float2* __restrict__ X, const float* __restrict__ khat, Dims d,
                                             const float2* __restrict__ gtw, int ZS, int KC) {
  using Cf = YZCfg<LY, LZ>;
  constexpr int EY = Cf::EY, TLY = Cf::TLY, EZ = Cf::EZ, TLZ = Cf::TLZ, PY = Cf::PY;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int kx = blockIdx.x / CS;
  extern __shared__ float2 sm[];
  float2* twy = sm;
  float2* twz = sm + LY;
  float2* ybuf = sm + LY + LZ;                 // [3][ZS][PY]: y-spectra of this CTA's z-slab
  float2* xch = ybuf + 3 * ZS * PY;            // [3][LZ][KC]: z-line exchange buffer
  load_tw<LY>(twy, gtw);
  load_tw<LZ>(twz, gtw);
  __syncthreads();
  const int tid = threadIdx.x;
  const int nz = d.nz, ny = d.ny;

  // ---------------- phase 1: forward y on the z-slab ----------------
  const int line = tid / TLY, ty = tid - line * TLY;  // line = comp * ZS + zl
  const int comp1 = line / ZS, z1 = rank * ZS + (line - comp1 * ZS);
  float2* xrow = X + ((size_t)(kx * 3 + comp1) * nz + z1) * ny;
  {
    float2 v[1][EY];
#pragma unroll
    for (int i = 0; i < EY; ++i) {
      const int p = ty + TLY * i;
      v[0][i] = p < ny ? xrow[p] : make_float2(0.f, 0.f);
    }
    const RowA<LY> A{line};
    reg_fft<LY, EY, 1, false>(v, ybuf, A, twy, ty);
#pragma unroll
    for (int i = 0; i < EY; ++i) ybuf[A(0, ty + TLY * i)] = v[0][i];
  }
  cl.sync();

  // ---------------- phase 2: z fwd * Khat * z inv on this CTA's ky-slab ----------------
  {
    const int KS = LY / CS, ky0 = rank * KS;
    const int kyl = tid % KC, rest = tid / KC, g = rest % 3, tz = rest / 3;
    const KRow kr(g);
    const int HY = LY / 2 + 1, HZ = LZ / 2 + 1;
    const float* kb = khat + (size_t)kx * 6 * HZ * HY;
    struct XA {
      int g, kyl, KC;
      __device__ __forceinline__ int operator()(int, int pos) const { return (g * LZ + pos) * KC + kyl; }
    } A{g, kyl, KC};
    const int nchunk = (KS + KC - 1) / KC;
    for (int ch = 0; ch < nchunk; ++ch) {
      const int kys = ch * KC + kyl;
      const bool ok = kys < KS;
      const int ky = ky0 + (ok ? kys : 0);
      const int yoff = RowPitch<LY>::at(ky);
      float2 v[1][EZ];
#pragma unroll
      for (int i = 0; i < EZ; ++i) {
        const int z = tz + TLZ * i;
        float2 val = make_float2(0.f, 0.f);
        if (ok && z < nz) {
          const int q = z / ZS;
          const float2* rb = cl.map_shared_rank(ybuf, q);
          val = rb[(g * ZS + (z - q * ZS)) * PY + yoff];
        }
        v[0][i] = val;
      }
      reg_fft<LZ, EZ, 1, false>(v, xch, A, twz, tz);
#pragma unroll
      for (int i = 0; i < EZ; ++i) xch[A(0, tz + TLZ * i)] = v[0][i];
      __syncthreads();
      if (ok) {
        const int kyf = ky <= LY / 2 ? ky : LY - ky;
        const float sy = ky <= LY / 2 ? 1.f : -1.f;
#pragma unroll
        for (int i = 0; i < EZ; ++i) {
          const int kz = tz + TLZ * i;
          const int kzf = kz <= LZ / 2 ? kz : LZ - kz;
          const float sz = kz <= LZ / 2 ? 1.f : -1.f;
          const size_t b = (size_t)kzf * HY + kyf;
          const float kd = __ldg(kb + (size_t)kr.cd * HZ * HY + b);
          const float k0 = fold_sign(kr.co0, sy, sz) * __ldg(kb + (size_t)kr.co0 * HZ * HY + b);
          const float k1 = fold_sign(kr.co1, sy, sz) * __ldg(kb + (size_t)kr.co1 * HZ * HY + b);
          const float2 md = v[0][i];
          const float2 m0 = xch[(kr.h0 * LZ + kz) * KC + kyl], m1 = xch[(kr.h1 * LZ + kz) * KC + kyl];
          v[0][i] = make_float2(kd * md.x + k0 * m0.x + k1 * m1.x, kd * md.y + k0 * m0.y + k1 * m1.y);
          if ((i & 3) == 3) asm volatile("" ::: "memory");
        }
      }
      __syncthreads();
      reg_fft<LZ, EZ, 1, true>(v, xch, A, twz, tz);
#pragma unroll
      for (int i = 0; i < EZ; ++i) {
        const int z = tz + TLZ * i;
        if (ok && z < nz) {
          const int q = z / ZS;
          float2* rb = cl.map_shared_rank(ybuf, q);
          rb[(g * ZS + (z - q * ZS)) * PY + yoff] = v[0][i];
        }
      }
    }
  }
  cl.sync();

  // ---------------- phase 3: inverse y, keep ny rows ----------------
  {
    const RowA<LY> A{line};
    float2 v[1][EY];
#pragma unroll
    for (int i = 0; i < EY; ++i) v[0][i] = ybuf[A(0, ty + TLY * i)];
    __syncthreads();
    reg_fft<LY, EY, 1, true>(v, ybuf, A, twy, ty);
#pragma unroll
    for (int i = 0; i < EY; ++i) {
      const int p = ty + TLY * i;
      if (p < ny) xrow[p] = v[0][i];
    }
  }
}

// ====================================================================== 3-pass fallback
template <int L>
struct RowCfg {  // contiguous-line passes (K-Y, K-YI): LPB lines per CTA
  static constexpr int E = L < 16 ? L : 16;
  static constexpr int TL = L / E;
  static constexpr int LPB0 = 256 / TL;
  static constexpr int LPB = LPB0 < 1 ? 1 : LPB0;
  static constexpr int NT = LPB * TL;
  static constexpr size_t SMEM = (size_t)(L + LPB * RowPitch<L>::P) * sizeof(float2);
};

template <int L, bool INV>
__global__ void __launch_bounds__(RowCfg<L>::NT) k_yline(const float2* __restrict__ in, float2* __restrict__ out,
                                                         long long nlines, int nin, int nout, int in_stride,
                                                         int out_stride, const float2* __restrict__ gtw) {
  using Cf = RowCfg<L>;
  constexpr int E = Cf::E, TL = Cf::TL, LPB = Cf::LPB;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  load_tw<L>(tw, gtw);
  __syncthreads();
  const int ll = threadIdx.x / TL, t = threadIdx.x - ll * TL;
  const long long ln = (long long)blockIdx.x * LPB + ll;
  const bool ok = ln < nlines;
  const float2* src = in + (ok ? ln : 0) * in_stride;
  float2 v[1][E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int p = t + TL * i;
    v[0][i] = (ok && p < nin) ? src[p] : make_float2(0.f, 0.f);
  }
  reg_fft<L, E, 1, INV>(v, sm + L, RowA<L>{ll}, tw, t);
  if (ok) {
    float2* dst = out + ln * out_stride;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      if (p < nout) dst[p] = v[0][i];
    }
  }
}

// K-Z on Y[kx][c][z][ky]: a CTA owns C adjacent ky of one kx; the 3 components in one thread.
template <int L>
struct ZCfg {
  static constexpr int E = L <= 16 ? L : 8;
  static constexpr int TL = L / E;
  static constexpr int C0 = 256 / TL;
  static constexpr int C = C0 < 4 ? 4 : (C0 > 64 ? 64 : C0);
  static constexpr int NT = C * TL;
  static constexpr size_t SMEM = (size_t)(L + 3 * L * C) * sizeof(float2);
};

template <int L, int C>
struct ColA {
  int c;
  __device__ __forceinline__ int operator()(int l, int pos) const { return (l * L + pos) * C + c; }
};

__device__ __forceinline__ void khat_apply(const float* __restrict__ kb, int HY, int HZ, int ky, int kz, int Ly,
                                           int Lz, float2& mx, float2& my, float2& mz) {
  const int kyf = ky <= Ly / 2 ? ky : Ly - ky;
  const int kzf = kz <= Lz / 2 ? kz : Lz - kz;
  const float sy = ky <= Ly / 2 ? 1.f : -1.f;
  const float sz = kz <= Lz / 2 ? 1.f : -1.f;
  const size_t cs = (size_t)HZ * HY;
  const size_t b = (size_t)kzf * HY + kyf;
  const float kxx = __ldg(kb + b), kyy = __ldg(kb + cs + b), kzz = __ldg(kb + 2 * cs + b);
  const float kxy = sy * __ldg(kb + 3 * cs + b);
  const float kxz = sz * __ldg(kb + 4 * cs + b);
  const float kyz = sy * sz * __ldg(kb + 5 * cs + b);
  const float2 bx = make_float2(kxx * mx.x + kxy * my.x + kxz * mz.x, kxx * mx.y + kxy * my.y + kxz * mz.y);
  const float2 by = make_float2(kxy * mx.x + kyy * my.x + kyz * mz.x, kxy * mx.y + kyy * my.y + kyz * mz.y);
  const float2 bz = make_float2(kxz * mx.x + kyz * my.x + kzz * mz.x, kxz * mx.y + kyz * my.y + kzz * mz.y);
  mx = bx;
  my = by;
  mz = bz;
}

template <int L>
__global__ void __launch_bounds__(ZCfg<L>::NT) k_zconv(float2* __restrict__ Y, const float* __restrict__ khat, Dims d,
                                                       const float2* __restrict__ gtw) {
  using Cf = ZCfg<L>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  load_tw<L>(tw, gtw);
  __syncthreads();
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  const int ky = blockIdx.x * C + c, kx = blockIdx.y;
  const bool ok = ky < d.Ly;
  const size_t cstr = (size_t)d.nz * d.Ly;           // between components
  float2* base = Y + (size_t)kx * 3 * cstr + (ok ? ky : 0);
  float2 v[3][E];
#pragma unroll
  for (int g = 0; g < 3; ++g)
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      v[g][i] = (ok && p < d.nz) ? base[g * cstr + (size_t)p * d.Ly] : make_float2(0.f, 0.f);
    }
  const ColA<L, C> A{c};
  reg_fft<L, E, 3, false>(v, sm + L, A, tw, t);
  if (ok) {
    const int HY = d.Ly / 2 + 1, HZ = d.Lz / 2 + 1;
    const float* kb = khat + (size_t)kx * 6 * HZ * HY;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      khat_apply(kb, HY, HZ, ky, t + TL * i, d.Ly, d.Lz, v[0][i], v[1][i], v[2][i]);
      if ((i & 1) == 1) asm volatile("" ::: "memory");
    }
  }
  reg_fft<L, E, 3, true>(v, sm + L, A, tw, t);
  if (ok) {
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int p = t + TL * i;
        if (p < d.nz) base[g * cstr + (size_t)p * d.Ly] = v[g][i];
      }
  }
}

// K-Y2D (nz == 1) on X[kx][c][0][y]: KPB kx values per CTA, the 3 components in one thread.
template <int L>
struct Y2Cfg {
  static constexpr int E = L <= 16 ? L : 8;
  static constexpr int TL = L / E;
  static constexpr int KPB0 = 128 / TL;
  static constexpr int KPB = KPB0 < 1 ? 1 : KPB0;
  static constexpr int NT = KPB * TL;
  static constexpr size_t SMEM = (size_t)(L + 3 * KPB * RowPitch<L>::P) * sizeof(float2);
};

template <int L>
__global__ void __launch_bounds__(Y2Cfg<L>::NT) k_y2d(float2* __restrict__ X, const float* __restrict__ khat, Dims d,
                                                      const float2* __restrict__ gtw) {
  using Cf = Y2Cfg<L>;
  constexpr int E = Cf::E, TL = Cf::TL, KPB = Cf::KPB;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  load_tw<L>(tw, gtw);
  __syncthreads();
  const int kl = threadIdx.x / TL, t = threadIdx.x - kl * TL;
  const int kx = blockIdx.x * KPB + kl;
  const bool ok = kx < d.NKX;
  float2* base = X + (size_t)(ok ? kx : 0) * 3 * d.ny;
  float2 v[3][E];
#pragma unroll
  for (int g = 0; g < 3; ++g)
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      v[g][i] = (ok && p < d.ny) ? base[g * d.ny + p] : make_float2(0.f, 0.f);
    }
  struct A3 {
    int kl;
    __device__ __forceinline__ int operator()(int l, int pos) const {
      return (l * KPB + kl) * RowPitch<L>::P + RowPitch<L>::at(pos);
    }
  } A{kl};
  reg_fft<L, E, 3, false>(v, sm + L, A, tw, t);
  if (ok) {
    const int HY = d.Ly / 2 + 1;
    const float* kb = khat + (size_t)kx * 6 * HY;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      khat_apply(kb, HY, 1, t + TL * i, 0, d.Ly, 1, v[0][i], v[1][i], v[2][i]);
      if ((i & 1) == 1) asm volatile("" ::: "memory");
    }
  }
  reg_fft<L, E, 3, true>(v, sm + L, A, tw, t);
  if (ok) {
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int p = t + TL * i;
        if (p < d.ny) base[g * d.ny + p] = v[g][i];
      }
  }
}

// ====================================================================== dispatch
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

// (LY, LZ) pairs with a cluster kernel instantiated
#define MCQ_YZ_LIST(X_) \
  X_(32, 4) X_(32, 8) X_(32, 16) X_(32, 32) X_(32, 64) \
  X_(64, 4) X_(64, 8) X_(64, 16) X_(64, 32) X_(64, 64) X_(64, 128) \
  X_(128, 4) X_(128, 8) X_(128, 16) X_(128, 32) X_(128, 64) X_(128, 128) X_(128, 256) \
  X_(256, 4) X_(256, 8) X_(256, 16) X_(256, 32) X_(256, 64) X_(256, 128) X_(256, 256) \
  X_(512, 4) X_(512, 8) X_(512, 16) X_(512, 32) X_(512, 64) \
  X_(1024, 4) X_(1024, 8) X_(1024, 16) X_(1024, 32)

static bool yz_instantiated(int LY, int LZ) {
#define X_(a, b) if (LY == a && LZ == b) return true;
  MCQ_YZ_LIST(X_)
#undef X_
  return false;
}

static void yz_consts(int LY, int LZ, int& TLY, int& TLZ, int& PY) {
  const int EY = LY < 16 ? LY : 16, EZ = LZ <= 16 ? LZ : 8;
  TLY = LY / EY;
  TLZ = LZ / EZ;
  PY = LY + (LY >= 16 ? LY / 16 : 1);
}

YZPlan plan_yz(const Dims& d) {
  YZPlan p{};
  if (d.nz < 2 || !yz_instantiated(d.Ly, d.Lz)) return p;
  int TLY, TLZ, PY;
  yz_consts(d.Ly, d.Lz, TLY, TLZ, PY);
  const size_t kLimit = 227 * 1024;
  YZPlan best{};
  for (int CS = 1; CS <= 16; CS *= 2) {
    if (d.nz % CS || d.Ly % CS) continue;
    const int ZS = d.nz / CS;
    const int NT = 3 * ZS * TLY;
    if (NT > 512 || NT < 32 || NT % (3 * TLZ)) continue;  // 512: __launch_bounds__ of k_yz
    const int KC = NT / (3 * TLZ);
    const size_t smem = (size_t)(d.Ly + d.Lz + 3 * ZS * PY + 3 * KC * d.Lz) * sizeof(float2);
    if (smem > kLimit) continue;
    YZPlan c{true, CS, ZS, KC, NT, smem};
    if (!best.ok) best = c;
    if (smem <= kLimit / 2 && NT >= 256) return c;  // two CTAs per SM
  }
  return best;
}

void launch_yz(const Dims& d, const YZPlan& p, float2* X, const float* khat, const float2* tw, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(d.NKX * p.CS);
  cfg.blockDim = dim3(p.NT);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define X_(a, b) \
  if (d.Ly == a && d.Lz == b) { cudaLaunchKernelEx(&cfg, k_yz<a, b>, X, khat, d, tw, p.ZS, p.KC); return; }
  MCQ_YZ_LIST(X_)
#undef X_
}

void launch_yfwd(const Dims& d, const float2* X, float2* Y, const float2* tw, cudaStream_t st) {
  const long long nl = (long long)d.NKX * 3 * d.nz;
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = RowCfg<L>;
    k_yline<L, false><<<(unsigned)((nl + Cf::LPB - 1) / Cf::LPB), Cf::NT, Cf::SMEM, st>>>(X, Y, nl, d.ny, L, d.ny,
                                                                                          L, tw);
  })
}

void launch_yinv(const Dims& d, const float2* Y, float2* X, const float2* tw, cudaStream_t st) {
  const long long nl = (long long)d.NKX * 3 * d.nz;
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = RowCfg<L>;
    k_yline<L, true><<<(unsigned)((nl + Cf::LPB - 1) / Cf::LPB), Cf::NT, Cf::SMEM, st>>>(Y, X, nl, L, d.ny, L, d.ny,
                                                                                         tw);
  })
}

void launch_zconv(const Dims& d, float2* Y, const float* khat, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Lz, {
    using Cf = ZCfg<L>;
    dim3 grid((d.Ly + Cf::C - 1) / Cf::C, d.NKX);
    k_zconv<L><<<grid, Cf::NT, Cf::SMEM, st>>>(Y, khat, d, tw);
  })
}

void launch_y2d(const Dims& d, float2* X, const float* khat, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = Y2Cfg<L>;
    k_y2d<L><<<(d.NKX + Cf::KPB - 1) / Cf::KPB, Cf::NT, Cf::SMEM, st>>>(X, khat, d, tw);
  })
}

// Opt every instantiation into the shared memory / cluster size it needs (once per process).
void configure_pass_kernels() {
  for (int Lv = 2; Lv <= 1024; Lv *= 2) {
    MCQ_DISPATCH_L(Lv, {
      cudaFuncSetAttribute(k_yline<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RowCfg<L>::SMEM);
      cudaFuncSetAttribute(k_yline<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RowCfg<L>::SMEM);
      cudaFuncSetAttribute(k_zconv<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZCfg<L>::SMEM);
      cudaFuncSetAttribute(k_y2d<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Y2Cfg<L>::SMEM);
    })
  }
#define X_(a, b)                                                                                  \
  cudaFuncSetAttribute(k_yz<a, b>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);     \
  cudaFuncSetAttribute(k_yz<a, b>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  MCQ_YZ_LIST(X_)
#undef X_
  cudaGetLastError();
}

}  // namespace mcq
