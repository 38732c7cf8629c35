// fft.cuh — complex helpers and the radix-2/4/8/16 register DFT codelets used by the
// register-resident Stockham FFT of regfft.cuh (the demag convolution, P:188 / reading C11).
// Forward transforms use w = exp(-2 pi i / L); inverse transforms are unnormalised (the
// 1/(Lx Ly Lz) factor is folded into the kernel spectrum Khat).
//
// Arithmetic is done on packed fp32 pairs: sm_100a executes add/sub/mul/fma.rn.f32x2 as one
// FADD2 / FMUL2 / FFMA2 instruction on a 64-bit register pair (re, im), which issues in one
// scheduler slot and occupies the FMA pipe for two cycles — the same fp32 throughput as two
// scalar instructions at half the issue cost (tools/ubench_coissue.cu: FFMA2 + LOP3 in 2.2
// cycles per warp vs 3 issue slots for the scalar pair).  The demag passes are issue-bound,
// so every complex add, subtract and multiply below is one or two packed instructions:
//   a + b, a - b          1 FADD2
//   a * w (complex)       FMUL2 + FFMA2 with the swizzled, half-negated operand (-a.y, a.x)
//   a + (-i) b, a + i b   1 FFMA2 (b swizzled and half-negated, times the constant pair 1)
// Rounding: every packed lane is an IEEE fp32 add / multiply / fused multiply-add, exactly as
// the scalar instructions (only the association of a few constant twiddles differs).
#pragma once
#include <cuda_runtime.h>

namespace mcq {

// ---------------------------------------------------------------- packed fp32x2 primitives
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; add.rn.f32x2 rc, ra, rb; mov.b64 {%0,%1}, rc;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; sub.rn.f32x2 rc, ra, rb; mov.b64 {%0,%1}, rc;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; mul.rn.f32x2 rc, ra, rb; mov.b64 {%0,%1}, rc;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc, rd; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; mov.b64 rc, {%6,%7}; "
      "fma.rn.f32x2 rd, ra, rb, rc; mov.b64 {%0,%1}, rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float2 bc2(float s) { return make_float2(s, s); }

// ---------------------------------------------------------------- complex helpers
// a * b = a * b.x + (-a.y, a.x) * b.y  (FMUL2 + FFMA2 with a swizzled, half-negated operand)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return fma2(make_float2(-a.y, a.x), bc2(b.y), mul2(a, bc2(b.x)));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return sub2(a, b); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return mul2(a, bc2(s)); }
// a + (-i) b  (forward) / a + i b (inverse): one FFMA2
template <bool INV>
__device__ __forceinline__ float2 add_mi(float2 a, float2 b) {
  return INV ? fma2(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a) : fma2(make_float2(b.y, b.x), make_float2(1.f, -1.f), a);
}
// a - (-i) b  (forward) / a - i b (inverse)
template <bool INV>
__device__ __forceinline__ float2 sub_mi(float2 a, float2 b) {
  return INV ? fma2(make_float2(b.y, b.x), make_float2(1.f, -1.f), a) : fma2(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a);
}
// multiply by -i (forward) / +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// ---------------------------------------------------------------- register codelets
template <bool INV>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
  const float2 t = a;
  a = add2(t, b);
  b = sub2(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2& v0, float2& v1, float2& v2, float2& v3) {
  const float2 t0 = add2(v0, v2), t1 = sub2(v0, v2);
  const float2 t2 = add2(v1, v3), t3 = sub2(v1, v3);
  v0 = add2(t0, t2);
  v2 = sub2(t0, t2);
  v1 = add_mi<INV>(t1, t3);  // t1 + (-+i) t3
  v3 = sub_mi<INV>(t1, t3);
}

// x * w8^1 (forward: (1 - i)/sqrt2; inverse: (1 + i)/sqrt2) and x * w8^3
template <bool INV>
__device__ __forceinline__ float2 w8_1(float2 x) {
  constexpr float c = 0.70710678118654752440f;
  // fwd: c (x.x + x.y, x.y - x.x) = c (x + (x.y, -x.x));  inv: c (x.x - x.y, x.y + x.x)
  return mul2(add_mi<INV>(x, x), bc2(c));
}
template <bool INV>
__device__ __forceinline__ float2 w8_3(float2 x) {
  constexpr float c = 0.70710678118654752440f;
  // fwd w8^3 = (-1 - i)/sqrt2: c (x.y - x.x, -x.x - x.y) = -c (x - (x.y, -x.x)) ; inv: conj
  return mul2(sub_mi<INV>(x, x), bc2(-c));
}

template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
  float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = w8_1<INV>(o1);
  o3 = w8_3<INV>(o3);
  v[0] = add2(e0, o0);
  v[4] = sub2(e0, o0);
  v[1] = add2(e1, o1);
  v[5] = sub2(e1, o1);
  v[2] = add_mi<INV>(e2, o2);  // o2 * w8^2 = -+i o2
  v[6] = sub_mi<INV>(e2, o2);
  v[3] = add2(e3, o3);
  v[7] = sub2(e3, o3);
}

template <bool INV>
__device__ __forceinline__ void dft16(float2* v) {
  // 16 = 4 x 4 Cooley-Tukey: n = 4 n1 + n2, k = k1 + 4 k2
  constexpr float C1 = 0.92387953251128675613f;  // cos(pi/8)
  constexpr float S1 = 0.38268343236508977173f;  // sin(pi/8)
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
  // twiddles w16^(n2 k1): e = 1, 3, 9 generic; 2, 6 eighth roots; 4 = -+i (folded into the adds below)
  const float2 w1 = make_float2(C1, INV ? S1 : -S1), w3 = make_float2(S1, INV ? C1 : -C1);
  const float2 w9 = make_float2(-C1, INV ? -S1 : S1);
  a[1][1] = cmul(a[1][1], w1);
  a[1][2] = w8_1<INV>(a[1][2]);
  a[1][3] = cmul(a[1][3], w3);
  a[2][1] = w8_1<INV>(a[2][1]);
  a[2][3] = w8_3<INV>(a[2][3]);
  a[3][1] = cmul(a[3][1], w3);
  a[3][2] = w8_3<INV>(a[3][2]);
  a[3][3] = cmul(a[3][3], w9);
  // a[2][2] carries w16^4 = -+i: folded into the second-level dft4 of column k1 = 2
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 x0 = a[0][k1], x1 = a[1][k1], x2 = a[2][k1], x3 = a[3][k1];
    if (k1 == 2) {  // dft4 with x2 pre-multiplied by -+i
      const float2 t0 = add_mi<INV>(x0, x2), t1 = sub_mi<INV>(x0, x2);
      const float2 t2 = add2(x1, x3), t3 = sub2(x1, x3);
      x0 = add2(t0, t2);
      x2 = sub2(t0, t2);
      x1 = add_mi<INV>(t1, t3);
      x3 = sub_mi<INV>(t1, t3);
    } else {
      dft4<INV>(x0, x1, x2, x3);
    }
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
