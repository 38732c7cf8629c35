// zconv3.cuh — K-Z v3: the z pass (a3 of SURVEY §8(a)) for Lz = 256 and 512 with warp-autonomous
// columns.  Included by passes.cu.
//
// Profiles of the CTA-synchronous designs (k_zconv_seq, and the persistent v2 of zconv2.cuh)
// show the step's three floors — DRAM bytes, shared-memory wavefronts, issue slots, each ~1/3
// of the kernel time — adding up instead of overlapping: every CTA moves through its phases
// (load, exchange, arithmetic, store) in lock step, separated by ~10 __syncthreads per tile,
// and 2 CTAs per SM cannot fill each other's gaps.  Here every warp owns its columns outright:
// its own shared-memory block, exchanges ordered by __syncwarp only, no CTA barrier after the
// twiddle tables are built.  The 8 warps of an SM-resident CTA (16 per SM) drift apart and a
// warp waiting on DRAM overlaps the others' exchanges and arithmetic.
//  * Lz = 256: a warp = 2 adjacent kx columns x 16 threads (16 points each, 16 x 16 transform);
//    Lz = 512: a warp = 1 column x 2 frequency channels x 16 threads (zconv2.cuh's channel
//    split: X[2k + ch] = DFT_256(x[n] w_512^{n ch})[k], channel twiddles folded into the second
//    stage's table, the halves of an inverse output summed through shared memory).
//  * The 8 warps of a CTA take 16 / 8 adjacent columns of one ky, so their loads of a z row
//    cover one 128-byte / 64-byte segment at about the same time (DRAM locality as a
//    CTA-wide tile; the L2 serves the second half of each sector).
//  * Fused Khat multiply (component 2 in registers, 0 and 1 parked at own positions), Khat loads
//    issued in batches of 8 points.
//  * Per-warp block [component][channel][position][column], 16-byte (2 columns) or 8-byte rows,
//    the bank group XOR-ed with bits 4.. of the position: stage stores (16 t + r) and loads
//    (t + 16 i) of a warp take 2 wavefronts.
#pragma once

namespace mcq {

#ifndef MCQ_Z3W
#define MCQ_Z3W 8  // warps per CTA
#endif

template <int L>
struct Z3Cfg {
  static_assert(L == 256 || L == 512, "K-Z v3 handles Lz = 256 and 512");
  static constexpr int NCH = L / 256;  // frequency channels
  static constexpr int LC = 256, E = 16, TL = 16;
  static constexpr int CPW = 2 / NCH;        // columns per warp
  static constexpr int WPC = MCQ_Z3W;        // warps per CTA
  static constexpr int C = CPW * WPC;        // columns per CTA tile
  static constexpr int NT = 32 * WPC;
  static constexpr int PADW = CPW == 2 ? 2 : 0;           // pad complex per 16 positions (2-column rows)
  static constexpr int WLINE = LC * CPW + 16 * PADW;     // complex per (component, channel) block of one warp
  static constexpr int WSM = 3 * NCH * WLINE;  // complex per warp
  static constexpr int TWP = 18;             // twiddle row pitch (complex), bank-spread rows
  static constexpr int TWN = 2 * NCH * 16 * TWP;
  static constexpr int MINB = 2;
  static constexpr size_t SMEM = (size_t)(TWN + WPC * WSM) * sizeof(float2);
};

// index of (position, column) in a warp block.  2-column rows (Lz = 256): 2 pad complex after
// every 16 positions (stage stores 16 t + r and loads t + 16 i: immediate offsets from one base,
// 2 wavefronts per warp); 1-column rows (Lz = 512, where the padding would cost the second
// resident CTA): the position's low 4 bits XOR-ed with bits 4-7
template <int CPW>
__device__ __forceinline__ int z3a(int pos, int cl) {
  if constexpr (CPW == 2) return pos * 2 + cl + (pos >> 4) * 2;
  else return pos ^ ((pos >> 4) & 15);
}

template <int L, bool SPLIT>
__global__ void __launch_bounds__(Z3Cfg<L>::NT, Z3Cfg<L>::MINB) k_zconv3(float2* __restrict__ Y, const float* __restrict__ khat,
                                                                          Dims d, const float2* __restrict__ gtw, int nkt,
                                                                          int nlone) {
  using Z = Z3Cfg<L>;
  constexpr int NCH = Z::NCH, E = Z::E, C = Z::C, NT = Z::NT, TWP = Z::TWP, CPW = Z::CPW;
  constexpr int WLINE = Z::WLINE, EN = 8 * NCH;
  extern __shared__ __align__(16) float2 sm[];
  float2* twf = sm;                   // [ch][k][TWP]: w_L^{r (NCH k + ch)}
  float2* twi = sm + NCH * 16 * TWP;  // [ch][k][TWP]: w_L^{-k (NCH r + ch)}
  pdl_trigger();
  for (int e = threadIdx.x; e < NCH * 256; e += NT) {
    const int ch = e >> 8, k = (e >> 4) & 15, r = e & 15;
    const int ef = (r * (NCH * k + ch)) % L, ei = (k * (NCH * r + ch)) % L;
    twf[(ch * 16 + k) * TWP + r] = gtw[ef * (kTwMax / L)];
    twi[(ch * 16 + k) * TWP + r] = cconj(gtw[ei * (kTwMax / L)]);
  }
  __syncthreads();  // the only CTA-wide barrier
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = CPW == 2 ? (lane & 1) : 0;
  const int t = CPW == 2 ? (lane >> 1) : (lane & 15);
  const int ch = CPW == 2 ? 0 : (lane >> 4);
  const int c = warp * CPW + cl;  // column inside the CTA tile
  const int nz = d.nzg, nzl = d.nz, hy = d.Ly / 2;
  const unsigned row = d.KXS, plane = (unsigned)d.Ly * row, cstr = (unsigned)nzl * plane;
  const unsigned kzs = (unsigned)(hy + 1) * d.P * 3;
  const float inv_nzl = 1.f / (float)nzl;
  // the lane's (kxl, ky): normal tiles = C columns at one ky (rows ky, Ly - ky back to back),
  // lone tiles = the last column at C rows ky
  int kxl, ky;
  const int tile = blockIdx.x;
  if (tile < nlone) {
    kxl = d.kxw - 1;
    ky = tile * C + c;
  } else {
    const int j = tile - nlone, kyi = j / nkt, kt = j - kyi * nkt, kyh = kyi >> 1;
    kxl = kt * C + c;
    ky = kyi == 1 ? hy : ((kyi & 1) ? d.Ly - kyh : kyh);
  }
  const bool ok = kxl < d.kxw && ky < d.Ly;
  const unsigned col = (unsigned)min(ky, d.Ly - 1) * row + min(kxl, d.kxw - 1);
  auto zoff = [&](int z) -> unsigned {  // slabs: R[r][c][zl] blocks, r = z / nzl (exact, z < 1024)
    unsigned a = (unsigned)z * plane;
    if constexpr (SPLIT) a += (unsigned)(2 * nzl * __float2int_rz(((float)z + 0.5f) * inv_nzl)) * plane;
    return a;
  };
  float2* const wb = sm + Z::TWN + warp * Z::WSM;
  float2* const reg0 = wb + ch * WLINE;
  float2* const reg1 = wb + (NCH + ch) * WLINE;
  float2* const reg2 = wb + (2 * NCH + ch) * WLINE;

  // ---- forward: component g, 16 x 16 with one warp-local exchange; park g = 0, 1
  float2 v[E];
#pragma unroll 1
  for (int g = 0; g < 3; ++g) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int z = t + 16 * i;
      v[i] = (i < EN && ok && z < nz) ? Y[col + g * cstr + zoff(z)] : make_float2(0.f, 0.f);
    }
    if (NCH == 2 && ch) {
#pragma unroll
      for (int i = 1; i < E; ++i) v[i] = cmul(v[i], w32c(i));
    }
    float2* R = g == 0 ? reg0 : (g == 1 ? reg1 : reg2);
    dft16<false>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) R[z3a<CPW>(16 * t + r, cl)] = v[r];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = R[z3a<CPW>(t + 16 * i, cl)];
    const float4* w4 = reinterpret_cast<const float4*>(twf + (ch * 16 + t) * TWP);
#pragma unroll
    for (int r2 = 0; r2 < 8; ++r2) {
      const float4 p = w4[r2];
      if (r2 > 0) v[2 * r2] = cmul(v[2 * r2], make_float2(p.x, p.y));
      v[2 * r2 + 1] = cmul(v[2 * r2 + 1], make_float2(p.z, p.w));
    }
    dft16<false>(v);
    if (g < 2) {
#pragma unroll
      for (int i = 0; i < E; ++i) R[z3a<CPW>(t + 16 * i, cl)] = v[i];  // own positions
    }
  }

  // ---- Khat multiply at the own positions (kz = NCH (t + 16 i) + ch), component 2 in v
  if (ok) {
    const int kx = d.kx0 + kxl;
    const int kyf = ky <= hy ? ky : d.Ly - ky;
    const float sy = ky <= hy ? 1.f : -1.f;
    const float2* kb = reinterpret_cast<const float2*>(khat) + ((unsigned)kyf * d.P + kx) * 3;
    constexpr int KB = MCQ_Z2KB;
#pragma unroll
    for (int b = 0; b < E; b += KB) {
      float2 kk[KB][3];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int i = b + j, kz = NCH * (t + 16 * i) + ch;
        const int kzf = i < 8 ? kz : L - kz;  // kz = L/2 (i = 8, t = ch = 0) folds to itself
        const float2* k2 = kb + (unsigned)kzf * kzs;
        kk[j][0] = __ldg(k2);
        kk[j][1] = __ldg(k2 + 1);
        kk[j][2] = __ldg(k2 + 2);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int i = b + j;
        const float sz = i < 8 ? 1.f : -1.f;  // (the odd components vanish at kz = L/2)
        const float2 k01 = kk[j][0], k23 = kk[j][1], k45 = kk[j][2];
        const float kxy = sy * k23.y, kxz = sz * k45.x, kyz = sy * sz * k45.y;
        const int a = z3a<CPW>(t + 16 * i, cl);
        const float2 mx = reg0[a], my = reg1[a], mz = v[i];
        reg0[a] = fma2(bc2(kxz), mz, fma2(bc2(kxy), my, mul2(bc2(k01.x), mx)));
        reg1[a] = fma2(bc2(kyz), mz, fma2(bc2(k01.y), my, mul2(bc2(kxy), mx)));
        v[i] = fma2(bc2(k23.x), mz, fma2(bc2(kyz), my, mul2(bc2(kxz), mx)));
      }
    }
  }

  // ---- inverse: components 2, 1, 0; channel sum; store the nz real planes
#pragma unroll 1
  for (int g = 2; g >= 0; --g) {
    float2* R = g == 0 ? reg0 : (g == 1 ? reg1 : reg2);
    if (g < 2) {
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = R[z3a<CPW>(t + 16 * i, cl)];
    }
    __syncwarp();  // the warp's own-position reads of region g are done before its exchange
    dft16<true>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) R[z3a<CPW>(16 * t + r, cl)] = v[r];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = R[z3a<CPW>(t + 16 * i, cl)];
    const float4* w4 = reinterpret_cast<const float4*>(twi + (ch * 16 + t) * TWP);
#pragma unroll
    for (int r2 = 0; r2 < 8; ++r2) {
      const float4 p = w4[r2];
      if (NCH == 2 || r2 > 0) v[2 * r2] = cmul(v[2 * r2], make_float2(p.x, p.y));
      v[2 * r2 + 1] = cmul(v[2 * r2 + 1], make_float2(p.z, p.w));
    }
    dft16<true>(v);
    if constexpr (NCH == 2) {
      if (ch) {
#pragma unroll
        for (int i = 1; i < E; ++i) v[i] = cmul(v[i], cconj(w32c(i)));
      }
      // channel 0 finishes slots i < 8, channel 1 slots i >= 8: hand the other half over
#pragma unroll
      for (int i = 0; i < E; ++i)
        if ((i < 8) == (ch == 1)) R[z3a<CPW>(t + 16 * i, cl)] = v[i];
      __syncwarp();
      const float2* Pr = ch ? R - WLINE : R + WLINE;  // the partner channel's block
#pragma unroll
      for (int i = 0; i < E; ++i)
        if ((i < 8) == (ch == 0)) v[i] = add2(v[i], Pr[z3a<CPW>(t + 16 * i, cl)]);
    }
    if (ok) {
#pragma unroll
      for (int i = 0; i < EN; ++i) {
        const int z = t + 16 * i;
        if ((NCH == 1 || (i < 8) == (ch == 0)) && z < nz) Y[col + g * cstr + zoff(z)] = v[i];
      }
    }
  }
}

}  // namespace mcq
