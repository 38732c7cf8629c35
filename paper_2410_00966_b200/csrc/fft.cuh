// fft.cuh — complex helpers and the radix-2/4/8/16 register DFT codelets used by the
// register-resident Stockham FFT of regfft.cuh (the demag convolution, P:188 / reading C11).
// Forward transforms use w = exp(-2 pi i / L); inverse transforms are unnormalised (the
// 1/(Lx Ly Lz) factor is folded into the kernel spectrum Khat).
#pragma once
#include <cuda_runtime.h>

namespace mcq {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by -i (forward) / +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// ---------------------------------------------------------------- register codelets
template <bool INV>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2& v0, float2& v1, float2& v2, float2& v3) {
  float2 t0 = cadd(v0, v2), t1 = csub(v0, v2);
  float2 t2 = cadd(v1, v3), t3 = mul_mi<INV>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
  constexpr float c = 0.70710678118654752440f;
  float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  // twiddles w8^k, k=1..3
  o1 = INV ? make_float2(c * (o1.x - o1.y), c * (o1.x + o1.y)) : make_float2(c * (o1.x + o1.y), c * (o1.y - o1.x));
  o2 = mul_mi<INV>(o2);
  o3 = INV ? make_float2(-c * (o3.x + o3.y), c * (o3.x - o3.y)) : make_float2(c * (o3.y - o3.x), -c * (o3.x + o3.y));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1);
  v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2);
  v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3);
  v[7] = csub(e3, o3);
}

template <bool INV>
__device__ __forceinline__ void dft16(float2* v) {
  // 16 = 4 x 4 Cooley-Tukey: n = 4 n1 + n2, k = k1 + 4 k2
  constexpr float C1 = 0.92387953251128675613f;  // cos(pi/8)
  constexpr float S1 = 0.38268343236508977173f;  // sin(pi/8)
  constexpr float C2 = 0.70710678118654752440f;
  const float cs[10] = {1.f, C1, C2, S1, 0.f, -S1, -C2, -C1, -1.f, -C1};  // cos(2 pi e / 16), e=0..9
  const float sn[10] = {0.f, S1, C2, C1, 1.f, C1, C2, S1, 0.f, -S1};      // sin(2 pi e / 16)
  float2 a[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    float2 x0 = v[n2], x1 = v[4 + n2], x2 = v[8 + n2], x3 = v[12 + n2];
    dft4<INV>(x0, x1, x2, x3);
    a[n2][0] = x0;
    a[n2][1] = x1;
    a[n2][2] = x2;
    a[n2][3] = x3;
  }
#pragma unroll
  for (int n2 = 1; n2 < 4; ++n2) {
#pragma unroll
    for (int k1 = 1; k1 < 4; ++k1) {
      const int e = n2 * k1;
      float2& x = a[n2][k1];
      if (e == 4) {  // w^4 = -i (fwd) / +i (inv): a swap
        x = mul_mi<INV>(x);
      } else if (e == 2) {  // (c, -+c)
        x = INV ? make_float2(C2 * (x.x - x.y), C2 * (x.x + x.y)) : make_float2(C2 * (x.x + x.y), C2 * (x.y - x.x));
      } else if (e == 6) {  // (-c, -+c)
        x = INV ? make_float2(-C2 * (x.x + x.y), C2 * (x.x - x.y)) : make_float2(C2 * (x.y - x.x), -C2 * (x.x + x.y));
      } else {
        x = cmul(x, make_float2(cs[e], INV ? sn[e] : -sn[e]));
      }
    }
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 x0 = a[0][k1], x1 = a[1][k1], x2 = a[2][k1], x3 = a[3][k1];
    dft4<INV>(x0, x1, x2, x3);
    v[k1] = x0;
    v[k1 + 4] = x1;
    v[k1 + 8] = x2;
    v[k1 + 12] = x3;
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2<INV>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    dft8<INV>(v);
  } else {
    static_assert(R == 16, "radix");
    dft16<INV>(v);
  }
}

__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

}  // namespace mcq
