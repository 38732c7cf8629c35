// passes.cu — the y and z passes of the zero-padded demag FFT convolution (a2-a4 of SURVEY §8(a)).
//
// B_demag = -mu0 IFFT( Khat . FFT(M) ) restricted to the grid, with M = Ms m zero-padded to
// (Lx, Ly, Lz) (reading C11).  The x transforms live in the update kernel (update.cu); here:
//   K-Y  (k_yfwd):  X[3][nz][ny][P] -> Y[3][nz][Ly][P], forward along y, input rows >= ny are 0
//   K-Z  (k_zconv): per (ky, kx) column of Y: forward along z (planes >= nz are 0), the
//                   symmetric 3x3 multiply by the real folded Khat, inverse along z, keep nz
//   K-YI (k_yinv):  Y -> X, inverse along y, keep the first ny rows
//   K-Y2D(k_y2d):   nz == 1: forward y, Khat multiply, inverse y in one pass, in place on X
// A CTA owns C adjacent kx columns (a warp's global accesses are contiguous C*8-byte row
// segments).  Lines are transformed with the register-resident FFT of regfft.cuh: data go
// HBM -> registers -> (S-1 smem exchanges) -> registers -> HBM, and K-Z/K-Y2D multiply by Khat
// in registers between the forward and the inverse transform.
#include "common.cuh"
#include "regfft.cuh"

#ifndef MCQ_ZE
#define MCQ_ZE 8   // complex values per thread per line in K-Z / K-Y2D (register budget)
#endif

namespace mcq {

template <int L>
struct PassCfg {  // single-line passes (K-Y, K-YI)
  static constexpr int E = L < 16 ? L : 16;
  static constexpr int TL = L / E;
  static constexpr int C0 = 256 / TL;
  static constexpr int C = C0 < 8 ? 8 : (C0 > 64 ? 64 : C0);
  static constexpr int NT = C * TL;
  static constexpr size_t SMEM = (size_t)(L + (TL > 1 ? L * C : 0)) * sizeof(float2);
};

template <int L>
struct ZCfg {  // three-component passes with the Khat multiply (K-Z, K-Y2D): one line per thread group
  static constexpr int E = L >= 1024 ? 16 : (L < MCQ_ZE ? L : MCQ_ZE);
  static constexpr int TL = L / E;
  static constexpr int C0 = 256 / TL;  // columns per CTA: NT = 3 * C * TL <= 768
  static constexpr int C = C0 < 4 ? 4 : (C0 > 64 ? 64 : C0);
  static_assert(3 * C * TL <= 1024, "block size");
  static constexpr int NT = 3 * C * TL;
  static constexpr size_t SMEM = (size_t)(L + 3 * L * C) * sizeof(float2);
};

template <int L>
__device__ __forceinline__ void load_tw(float2* tw, const float2* __restrict__ gtw, int nt) {
  for (int m = threadIdx.x; m < L; m += nt) tw[m] = gtw[m * (kTwMax / L)];
  __syncthreads();
}

// shared-memory address of (line l, position pos) for column c: [l][pos][c]
template <int L, int C>
struct ColAddr {
  int c;
  __device__ __forceinline__ int operator()(int l, int pos) const { return (l * L + pos) * C + c; }
};

// ---------------------------------------------------------------- K-Y forward
template <int L>
__global__ void __launch_bounds__(PassCfg<L>::NT) k_yfwd(const float2* __restrict__ X, float2* __restrict__ Y,
                                                         Dims d, const float2* __restrict__ gtw) {
  using Cf = PassCfg<L>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C, NT = Cf::NT;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  load_tw<L>(tw, gtw, NT);
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  const int kx = blockIdx.x * C + c, z = blockIdx.y, comp = blockIdx.z;
  const bool ok = kx < d.NKX;
  const float2* src = X + ((size_t)(comp * d.nz + z) * d.ny) * d.P + kx;
  float2 v[1][E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int p = t + TL * i;
    v[0][i] = (ok && p < d.ny) ? src[(size_t)p * d.P] : make_float2(0.f, 0.f);
  }
  reg_fft<L, E, 1, false>(v, sm + L, ColAddr<L, C>{c}, tw, t);
  if (ok) {
    float2* dst = Y + ((size_t)(comp * d.nz + z) * L) * d.P + kx;
#pragma unroll
    for (int i = 0; i < E; ++i) dst[(size_t)(t + TL * i) * d.P] = v[0][i];
  }
}

// ---------------------------------------------------------------- K-Y inverse
template <int L>
__global__ void __launch_bounds__(PassCfg<L>::NT) k_yinv(const float2* __restrict__ Y, float2* __restrict__ X,
                                                         Dims d, const float2* __restrict__ gtw) {
  using Cf = PassCfg<L>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C, NT = Cf::NT;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  load_tw<L>(tw, gtw, NT);
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  const int kx = blockIdx.x * C + c, z = blockIdx.y, comp = blockIdx.z;
  const bool ok = kx < d.NKX;
  const float2* src = Y + ((size_t)(comp * d.nz + z) * L) * d.P + kx;
  float2 v[1][E];
#pragma unroll
  for (int i = 0; i < E; ++i) v[0][i] = ok ? src[(size_t)(t + TL * i) * d.P] : make_float2(0.f, 0.f);
  reg_fft<L, E, 1, true>(v, sm + L, ColAddr<L, C>{c}, tw, t);
  if (ok) {
    float2* dst = X + ((size_t)(comp * d.nz + z) * d.ny) * d.P + kx;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      if (p < d.ny) dst[(size_t)p * d.P] = v[0][i];
    }
  }
}

// ---------------------------------------------------------------- Khat multiply
// Khat is real and stored folded: [6][Lz/2+1][Ly/2+1][P]; off-diagonal components flip sign
// across the half axis they are odd in (XY: x,y; XZ: x,z; YZ: y,z).  kx is never folded.
__device__ __forceinline__ void khat_apply(const float* __restrict__ khat, const Dims& d, int kx, int ky, int kz,
                                           float2& mx, float2& my, float2& mz) {
  const int hy = d.Ly / 2, hz = d.Lz / 2;
  const int kyf = ky <= hy ? ky : d.Ly - ky;
  const int kzf = kz <= hz ? kz : d.Lz - kz;
  const float sy = ky <= hy ? 1.f : -1.f;
  const float sz = kz <= hz ? 1.f : -1.f;
  const size_t cs = (size_t)(hz + 1) * (hy + 1) * d.P;
  const size_t b = ((size_t)kzf * (hy + 1) + kyf) * d.P + kx;
  const float kxx = __ldg(khat + b), kyy = __ldg(khat + cs + b), kzz = __ldg(khat + 2 * cs + b);
  const float kxy = sy * __ldg(khat + 3 * cs + b);
  const float kxz = sz * __ldg(khat + 4 * cs + b);
  const float kyz = sy * sz * __ldg(khat + 5 * cs + b);
  const float2 bx = make_float2(kxx * mx.x + kxy * my.x + kxz * mz.x, kxx * mx.y + kxy * my.y + kxz * mz.y);
  const float2 by = make_float2(kxy * mx.x + kyy * my.x + kyz * mz.x, kxy * mx.y + kyy * my.y + kyz * mz.y);
  const float2 bz = make_float2(kxz * mx.x + kyz * my.x + kzz * mz.x, kxz * mx.y + kyz * my.y + kzz * mz.y);
  mx = bx;
  my = by;
  mz = bz;
}

// ---------------------------------------------------------------- K-Z / K-Y2D: fwd * Khat * inv
// Thread group (component g, column c) owns one line; the forward transforms leave the three
// components of a point in three different threads, so they meet once in shared memory for the
// multiply: each thread forms its own component B_g = sum_h Khat_gh M_h at its positions.
// AXIS2D = false: lines along z of Y[3][nz][Ly][P] at ky = blockIdx.y (K-Z);
// AXIS2D = true : lines along y of X[3][1][ny][P] (K-Y2D, nz == 1, kz = 0).
template <int L, bool AXIS2D>
__global__ void __launch_bounds__(ZCfg<L>::NT) k_conv(float2* __restrict__ Y, const float* __restrict__ khat, Dims d,
                                                      const float2* __restrict__ gtw) {
  using Cf = ZCfg<L>;
  constexpr int E = Cf::E, TL = Cf::TL, C = Cf::C, NT = Cf::NT;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  float2* xs = sm + L;
  load_tw<L>(tw, gtw, NT);
  const int c = threadIdx.x % C, rest = threadIdx.x / C, g = rest % 3, t = rest / 3;
  const int kx = blockIdx.x * C + c;
  const int ky = AXIS2D ? 0 : blockIdx.y;
  const bool ok = kx < d.NKX;
  const int nin = AXIS2D ? d.ny : d.nz;
  const size_t lstride = AXIS2D ? (size_t)d.P : (size_t)d.Ly * d.P;     // between line elements
  const size_t cstr = AXIS2D ? (size_t)d.ny * d.P : (size_t)d.nz * d.Ly * d.P;
  float2* base = Y + g * cstr + (size_t)ky * d.P + kx;
  float2 v[1][E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int p = t + TL * i;
    v[0][i] = (ok && p < nin) ? base[p * lstride] : make_float2(0.f, 0.f);
  }
  // line l of this thread = component g; element (g, pos, c) at (g L + pos) C + c
  struct A3 {
    int g, c;
    __device__ __forceinline__ int operator()(int, int pos) const { return (g * L + pos) * C + c; }
  } A{g, c};
  reg_fft<L, E, 1, false>(v, xs, A, tw, t);
#pragma unroll
  for (int i = 0; i < E; ++i) xs[A(0, t + TL * i)] = v[0][i];
  __syncthreads();
  if (ok) {
    const int hy = d.Ly / 2, hz = d.Lz / 2;
    const size_t cs = (size_t)(hz + 1) * (hy + 1) * d.P;
    // components of row g of the symmetric tensor: (gg, g0, g1) with signs for the folds
    // g = 0: (XX; XY*My, XZ*Mz)   g = 1: (YY; XY*Mx, YZ*Mz)   g = 2: (ZZ; XZ*Mx, YZ*My)
    const int cd = g, co0 = g == 2 ? 4 : 3, co1 = g == 0 ? 4 : 5;
    const int h0 = g == 0 ? 1 : 0, h1 = g == 2 ? 1 : 2;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      const int kyv = AXIS2D ? p : ky, kzv = AXIS2D ? 0 : p;
      const int kyf = kyv <= hy ? kyv : d.Ly - kyv;
      const int kzf = kzv <= hz ? kzv : d.Lz - kzv;
      const float sy = kyv <= hy ? 1.f : -1.f, sz = kzv <= hz ? 1.f : -1.f;
      const float sgn[6] = {1.f, 1.f, 1.f, sy, sz, sy * sz};
      const size_t b = ((size_t)kzf * (hy + 1) + kyf) * d.P + kx;
      const float kd = __ldg(khat + cd * cs + b);
      const float k0 = sgn[co0] * __ldg(khat + co0 * cs + b);
      const float k1 = sgn[co1] * __ldg(khat + co1 * cs + b);
      const float2 md = v[0][i];
      const float2 m0 = xs[(h0 * L + p) * C + c], m1 = xs[(h1 * L + p) * C + c];
      v[0][i] = make_float2(kd * md.x + k0 * m0.x + k1 * m1.x, kd * md.y + k0 * m0.y + k1 * m1.y);
      if ((i & 3) == 3) asm volatile("" ::: "memory");  // bound load hoisting (register budget)
    }
  }
  __syncthreads();
  reg_fft<L, E, 1, true>(v, xs, A, tw, t);
  if (ok) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int p = t + TL * i;
      if (p < nin) base[p * lstride] = v[0][i];
    }
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

void launch_yfwd(const Dims& d, const float2* X, float2* Y, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = PassCfg<L>;
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C, d.nz, 3);
    k_yfwd<L><<<grid, Cf::NT, Cf::SMEM, st>>>(X, Y, d, tw);
  })
}

void launch_yinv(const Dims& d, const float2* Y, float2* X, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = PassCfg<L>;
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C, d.nz, 3);
    k_yinv<L><<<grid, Cf::NT, Cf::SMEM, st>>>(Y, X, d, tw);
  })
}

void launch_zconv(const Dims& d, float2* Y, const float* khat, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Lz, {
    using Cf = ZCfg<L>;
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C, d.Ly);
    k_conv<L, false><<<grid, Cf::NT, Cf::SMEM, st>>>(Y, khat, d, tw);
  })
}

void launch_y2d(const Dims& d, float2* X, const float* khat, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = ZCfg<L>;
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C);
    k_conv<L, true><<<grid, Cf::NT, Cf::SMEM, st>>>(X, khat, d, tw);
  })
}

// Opt every instantiation into the shared memory it needs (once per process).
void configure_pass_kernels() {
  for (int Lv = 2; Lv <= 1024; Lv *= 2) {
    MCQ_DISPATCH_L(Lv, {
      cudaFuncSetAttribute(k_yfwd<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PassCfg<L>::SMEM);
      cudaFuncSetAttribute(k_yinv<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PassCfg<L>::SMEM);
      cudaFuncSetAttribute(k_conv<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZCfg<L>::SMEM);
      cudaFuncSetAttribute(k_conv<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZCfg<L>::SMEM);
    })
  }
}

}  // namespace mcq
