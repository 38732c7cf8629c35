// passes.cu — the y and z passes of the zero-padded demag FFT convolution (a2-a4 of SURVEY §8(a)).
//
// B_demag = -mu0 IFFT( Khat . FFT(M) ) restricted to the grid, with M = Ms m zero-padded to
// (Lx, Ly, Lz) (reading C11).  The x transforms live in the update kernel (update.cu); here:
//   K-Y  (k_yfwd):  X[3][nz][ny][P] -> Y[3][nz][Ly][P], forward along y, input rows >= ny are 0
//   K-Z  (k_zconv): per (ky, kx) column of Y: forward along z (planes >= nz are 0), the
//                   symmetric 3x3 multiply by the real folded Khat, inverse along z, keep nz
//   K-YI (k_yinv):  Y -> X, inverse along y, keep the first ny rows
//   K-Y2D(k_y2d):   nz == 1: forward y, Khat multiply, inverse y in one pass, in place on X
// Each CTA owns C adjacent kx columns (contiguous in memory, so every global access of a warp
// is a contiguous C*8-byte segment) and the full padded line in shared memory.
#include "common.cuh"
#include "fft.cuh"

namespace mcq {

template <int L>
struct PassCfg {
  static constexpr int C = L >= 512 ? 8 : 16;          // columns per CTA
  static constexpr int E = L < 16 ? L : 16;            // complex values per thread
  static constexpr int NT = L * C / E;                 // threads (single-component passes)
};

template <int L>
__device__ __forceinline__ void load_tw(float2* tw, const float2* __restrict__ gtw, int nt) {
  for (int m = threadIdx.x; m < L; m += nt) tw[m] = gtw[m * (kTwMax / L)];
}

// ---------------------------------------------------------------- K-Y forward
template <int L>
__global__ void __launch_bounds__(PassCfg<L>::NT) k_yfwd(const float2* __restrict__ X, float2* __restrict__ Y,
                                                         Dims d, const float2* __restrict__ gtw) {
  constexpr int C = PassCfg<L>::C, NT = PassCfg<L>::NT;
  using Lay = ColLayout<L, C>;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  float2* s = sm + L;
  load_tw<L>(tw, gtw, NT);
  const int kx0 = blockIdx.x * C, z = blockIdx.y, comp = blockIdx.z;
  const float2* src = X + ((size_t)(comp * d.nz + z) * d.ny) * d.P;
  for (int e = threadIdx.x; e < L * C; e += NT) {
    const int i = e / C, c = e - i * C, kx = kx0 + c;
    float2 v = make_float2(0.f, 0.f);
    if (i < d.ny && kx < d.NKX) v = src[(size_t)i * d.P + kx];
    s[Lay::addr(i, c)] = v;
  }
  __syncthreads();
  block_fft<L, C, NT, false, Lay>(s, tw);
  float2* dst = Y + ((size_t)(comp * d.nz + z) * L) * d.P;
  for (int e = threadIdx.x; e < L * C; e += NT) {
    const int i = e / C, c = e - i * C, kx = kx0 + c;
    if (kx < d.NKX) dst[(size_t)i * d.P + kx] = s[Lay::addr(i, c)];
  }
}

// ---------------------------------------------------------------- K-Y inverse
template <int L>
__global__ void __launch_bounds__(PassCfg<L>::NT) k_yinv(const float2* __restrict__ Y, float2* __restrict__ X,
                                                         Dims d, const float2* __restrict__ gtw) {
  constexpr int C = PassCfg<L>::C, NT = PassCfg<L>::NT;
  using Lay = ColLayout<L, C>;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  float2* s = sm + L;
  load_tw<L>(tw, gtw, NT);
  const int kx0 = blockIdx.x * C, z = blockIdx.y, comp = blockIdx.z;
  const float2* src = Y + ((size_t)(comp * d.nz + z) * L) * d.P;
  for (int e = threadIdx.x; e < L * C; e += NT) {
    const int i = e / C, c = e - i * C, kx = kx0 + c;
    float2 v = make_float2(0.f, 0.f);
    if (kx < d.NKX) v = src[(size_t)i * d.P + kx];
    s[Lay::addr(i, c)] = v;
  }
  __syncthreads();
  block_fft<L, C, NT, true, Lay>(s, tw);
  float2* dst = X + ((size_t)(comp * d.nz + z) * d.ny) * d.P;
  for (int e = threadIdx.x; e < d.ny * C; e += NT) {
    const int i = e / C, c = e - i * C, kx = kx0 + c;
    if (kx < d.NKX) dst[(size_t)i * d.P + kx] = s[Lay::addr(i, c)];
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

// ---------------------------------------------------------------- K-Z: z fwd * Khat * z inv
template <int L>
struct ZCfg {
  static constexpr int C = L >= 512 ? 4 : (L >= 256 ? 8 : 16);
  static constexpr int E = L < 16 ? L : 16;
  static constexpr int NT = 3 * L * C / E;
};

template <int L>
__global__ void __launch_bounds__(ZCfg<L>::NT) k_zconv(float2* __restrict__ Y, const float* __restrict__ khat, Dims d,
                                                       const float2* __restrict__ gtw) {
  constexpr int C = ZCfg<L>::C, NT = ZCfg<L>::NT;
  using Lay = ColLayout<L, C>;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  float2* s = sm + L;
  load_tw<L>(tw, gtw, NT);
  const int kx0 = blockIdx.x * C, ky = blockIdx.y;
  const size_t plane = (size_t)d.Ly * d.P;                 // stride between z planes of one comp
  const size_t comp_stride = (size_t)d.nz * plane;
  float2* base = Y + (size_t)ky * d.P;
  for (int e = threadIdx.x; e < 3 * L * C; e += NT) {
    const int g = e / (L * C), rem = e - g * (L * C), i = rem / C, c = rem - i * C, kx = kx0 + c;
    float2 v = make_float2(0.f, 0.f);
    if (i < d.nz && kx < d.NKX) v = base[g * comp_stride + i * plane + kx];
    s[Lay::addr(i, g * C + c)] = v;
  }
  __syncthreads();
  block_fft<L, 3 * C, NT, false, Lay>(s, tw);
  for (int e = threadIdx.x; e < L * C; e += NT) {
    const int i = e / C, c = e - i * C, kx = kx0 + c;
    if (kx < d.NKX) {
      float2 mx = s[Lay::addr(i, c)], my = s[Lay::addr(i, C + c)], mz = s[Lay::addr(i, 2 * C + c)];
      khat_apply(khat, d, kx, ky, i, mx, my, mz);
      s[Lay::addr(i, c)] = mx;
      s[Lay::addr(i, C + c)] = my;
      s[Lay::addr(i, 2 * C + c)] = mz;
    }
  }
  __syncthreads();
  block_fft<L, 3 * C, NT, true, Lay>(s, tw);
  for (int e = threadIdx.x; e < 3 * d.nz * C; e += NT) {
    const int g = e / (d.nz * C), rem = e - g * (d.nz * C), i = rem / C, c = rem - i * C, kx = kx0 + c;
    if (kx < d.NKX) base[g * comp_stride + i * plane + kx] = s[Lay::addr(i, g * C + c)];
  }
}

// ---------------------------------------------------------------- K-Y2D (nz == 1)
template <int L>
__global__ void __launch_bounds__(ZCfg<L>::NT) k_y2d(float2* __restrict__ X, const float* __restrict__ khat, Dims d,
                                                     const float2* __restrict__ gtw) {
  constexpr int C = ZCfg<L>::C, NT = ZCfg<L>::NT;
  using Lay = ColLayout<L, C>;
  extern __shared__ float2 sm[];
  float2* tw = sm;
  float2* s = sm + L;
  load_tw<L>(tw, gtw, NT);
  const int kx0 = blockIdx.x * C;
  const size_t comp_stride = (size_t)d.ny * d.P;
  for (int e = threadIdx.x; e < 3 * L * C; e += NT) {
    const int g = e / (L * C), rem = e - g * (L * C), i = rem / C, c = rem - i * C, kx = kx0 + c;
    float2 v = make_float2(0.f, 0.f);
    if (i < d.ny && kx < d.NKX) v = X[g * comp_stride + (size_t)i * d.P + kx];
    s[Lay::addr(i, g * C + c)] = v;
  }
  __syncthreads();
  block_fft<L, 3 * C, NT, false, Lay>(s, tw);
  for (int e = threadIdx.x; e < L * C; e += NT) {
    const int i = e / C, c = e - i * C, kx = kx0 + c;
    if (kx < d.NKX) {
      float2 mx = s[Lay::addr(i, c)], my = s[Lay::addr(i, C + c)], mz = s[Lay::addr(i, 2 * C + c)];
      khat_apply(khat, d, kx, i, 0, mx, my, mz);
      s[Lay::addr(i, c)] = mx;
      s[Lay::addr(i, C + c)] = my;
      s[Lay::addr(i, 2 * C + c)] = mz;
    }
  }
  __syncthreads();
  block_fft<L, 3 * C, NT, true, Lay>(s, tw);
  for (int e = threadIdx.x; e < 3 * d.ny * C; e += NT) {
    const int g = e / (d.ny * C), rem = e - g * (d.ny * C), i = rem / C, c = rem - i * C, kx = kx0 + c;
    if (kx < d.NKX) X[g * comp_stride + (size_t)i * d.P + kx] = s[Lay::addr(i, g * C + c)];
  }
}

// ---------------------------------------------------------------- dispatch
#define MCQ_DISPATCH_L(Lval, ...)          \
  switch (Lval) {                           \
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
    default: break;                         \
  }

void launch_yfwd(const Dims& d, const float2* X, float2* Y, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = PassCfg<L>;
    const size_t sm = (size_t)(L + L * Cf::C) * sizeof(float2);
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C, d.nz, 3);
    k_yfwd<L><<<grid, Cf::NT, sm, st>>>(X, Y, d, tw);
  })
}

void launch_yinv(const Dims& d, const float2* Y, float2* X, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = PassCfg<L>;
    const size_t sm = (size_t)(L + L * Cf::C) * sizeof(float2);
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C, d.nz, 3);
    k_yinv<L><<<grid, Cf::NT, sm, st>>>(Y, X, d, tw);
  })
}

void launch_zconv(const Dims& d, float2* Y, const float* khat, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Lz, {
    using Cf = ZCfg<L>;
    const size_t sm = (size_t)(L + 3 * L * Cf::C) * sizeof(float2);
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C, d.Ly);
    k_zconv<L><<<grid, Cf::NT, sm, st>>>(Y, khat, d, tw);
  })
}

void launch_y2d(const Dims& d, float2* X, const float* khat, const float2* tw, cudaStream_t st) {
  MCQ_DISPATCH_L(d.Ly, {
    using Cf = ZCfg<L>;
    const size_t sm = (size_t)(L + 3 * L * Cf::C) * sizeof(float2);
    dim3 grid((d.NKX + Cf::C - 1) / Cf::C);
    k_y2d<L><<<grid, Cf::NT, sm, st>>>(X, khat, d, tw);
  })
}

// Opt every instantiation into the shared memory it needs (once per process).
void configure_pass_kernels() {
  for (int Lv = 2; Lv <= 1024; Lv *= 2) {
    MCQ_DISPATCH_L(Lv, {
      const int a = (int)((L + L * PassCfg<L>::C) * sizeof(float2));
      const int b = (int)((L + 3 * L * ZCfg<L>::C) * sizeof(float2));
      cudaFuncSetAttribute(k_yfwd<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, a);
      cudaFuncSetAttribute(k_yinv<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, a);
      cudaFuncSetAttribute(k_zconv<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
      cudaFuncSetAttribute(k_y2d<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    })
  }
}

}  // namespace mcq
