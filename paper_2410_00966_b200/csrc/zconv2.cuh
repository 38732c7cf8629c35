// zconv2.cuh — K-Z v2: the z pass (a3 of SURVEY §8(a): forward z FFT, Khat multiply, inverse z
// FFT) for Lz = 256 and 512, the lengths of BJ configs[1]-[4].  Included by passes.cu.
//
// Redesigned for sm_100a from the ncu evidence of the component-sequential kernel k_zconv_seq
// (profiles/r2_zconv_variants.md): it was bound by shared-memory wavefronts (Lz = 512: three radix
// stages, i.e. two full-length exchanges per transform, 25 % bank conflicts) and by exposed load
// latency (the Khat loads of the multiply; every CTA's first-component loads).
//  * Frequency channels.  The zero-padded transform of nz <= L/2 inputs is split by the residue
//    of kz mod NCH (NCH = L/256):  X[NCH k + ch] = DFT_256(x[n] w_L^{n ch})[k], and inverse
//    y[n] = sum_ch w_L^{-n ch} IDFT_256(B_ch)[n]  (n < nz, unnormalised).  Each channel transform
//    is 16 x 16 (two register stages, one shared-memory exchange).  With n = t + 16 i (thread t,
//    slot i) w_L^{ch n} = w_L^{ch t} w_32^{ch i}: the w_32 factors are compile-time slot constants
//    and w_L^{ch t} rides on the second stage's twiddle table — forward w_L^{r (NCH k + ch)},
//    inverse w_L^{-k (NCH r + ch)} (k = class = thread, r = slot) — at no extra cost.  The two
//    channel halves of an inverse output are summed through shared memory, each thread finishing
//    half of its slots.  For L = 256 (NCH = 1) this is the plain 16 x 16 transform with the
//    zero inputs / unused outputs (slots i >= 8) pruned at compile time.
//  * Fused multiply.  Component 2's spectrum stays in registers; the Khat multiply reads the
//    parked components 0 and 1 at the thread's own positions and writes their products back, and
//    the inverse starts with component 2 (no park / reload of it).
//  * One CTA per (kx tile, ky) tile by default (2 resident per SM; the persistent walk,
//    MCQ_Z2PERSIST, measured slower).  At the start of a tile its Khat rows are prefetched into
//    L2 (needed after the three forward transforms).  Lz = 256: component g+1's inputs are loaded
//    into registers during component g's forward transform.  Lz = 512 (TMA = true): the z columns
//    come in by TMA tensor copies into the component regions, a phase ahead, and the results
//    leave by TMA tensor stores (measurements: profiles/r2_zconv_variants.md).
//  * Shared layout [component][channel][position][column] (C = 8: the 64-byte bank half flipped
//    by bit 4 of the position): stage stores (16t + r) and loads (t + 16i) take 2 wavefronts per
//    warp, the minimum for 256 bytes.
// Tiles: C adjacent kx columns at one ky, rows ky and Ly - ky back to back (their folded Khat
// rows are the same: L2 reuse).  If one column is left over (NKX = C q + 1: the Nyquist column),
// "lone" tiles take that column for C rows ky at once instead of a mostly idle tile per ky.
#pragma once

namespace mcq {

#ifndef MCQ_Z2C
#define MCQ_Z2C 16  // kx columns per tile at Lz = 256 (half that at Lz = 512)
#endif
#ifndef MCQ_Z2TMAST
#define MCQ_Z2TMAST 1  // TMA path: the outputs leave through TMA tensor stores of the component boxes
#endif
#ifndef MCQ_Z2KB
#define MCQ_Z2KB 0  // Khat multiply: points per batch of loads in flight (0: 8 at Lz = 256, 4 at 512 —
                    // 8 spilled there, at the 128-register cap of two CTAs per SM)
#endif
#ifndef MCQ_Z2NEXT
#define MCQ_Z2NEXT 1  // load the next tile's component 0 into registers during the inverse phase
#endif

template <int L>
struct Z2Cfg {
  static_assert(L == 256 || L == 512, "K-Z v2 handles Lz = 256 and 512");
  static constexpr int NCH = L / 256;      // frequency channels (kz = NCH k + ch)
  static constexpr int LC = 256, E = 16, TL = 16;
  static constexpr int C = MCQ_Z2C / NCH;  // columns per tile: 128-byte / 64-byte row segments
  static constexpr int NT = C * TL * NCH;  // 256 threads (MCQ_Z2C = 16)
  static constexpr int MINB = 512 / NT;    // resident CTAs per SM the launch bounds ask for
  static constexpr int TWP = 18;           // twiddle row pitch (complex): rows 144 B apart (banks)
  static constexpr int TWN = 2 * NCH * 16 * TWP;
  static constexpr int LINE = LC * C;      // complex per (component, channel) block
  static constexpr size_t SMEM = (size_t)(TWN + 3 * NCH * LINE) * sizeof(float2);
};

// w_32^i (forward sign e^{-2 pi i i / 32}), i < 16: the channel-1 slot constants (L = 512)
__device__ __forceinline__ float2 w32c(int i) {
  constexpr float cs[16] = {1.0f,  9.807852804e-01f,  9.238795325e-01f,  8.314696123e-01f,
                            7.071067812e-01f,  5.555702330e-01f,  3.826834324e-01f,  1.950903220e-01f,
                            0.0f, -1.950903220e-01f, -3.826834324e-01f, -5.555702330e-01f,
                            -7.071067812e-01f, -8.314696123e-01f, -9.238795325e-01f, -9.807852804e-01f};
  // -sin(2 pi i / 32) = cos(2 pi (i + 8) / 32): cs[i + 8] for i < 8, -cs[i - 8] for i >= 8
  return make_float2(cs[i], i < 8 ? cs[(i + 8) & 15] : -cs[(i + 8) & 15]);
}

// index inside a (component, channel) block.  A row of C complex covers C/16 of the 32 banks; for
// C < 16 the row's bank group is XOR-ed with bits 4.. of the position, so both the stage stores
// (positions 16 t + r) and loads (t + 16 i) of a warp spread over all banks (2 wavefronts)
template <int C>
__device__ __forceinline__ int z2a(int pos, int c) {
  int a = pos * C + c;
  if constexpr (C < 16) a ^= ((pos >> 4) & (16 / C - 1)) * C;
  return a;
}

// TMA = true (single slab, normal tiles [tfirst, ntiles)): the z columns come in by TMA tensor
// copies (box: C columns x nz planes of one component) into the component regions themselves —
// component 0 and 2 through region 2, component 1 through region 1 — issued a phase or more
// ahead (next tile's component 0 during this tile's inverse), so no input load holds registers
// or waits on DRAM; the threads read their inputs from the staged box ([z][c]).
template <int L, bool SPLIT, bool TMA = false>
__global__ void __launch_bounds__(Z2Cfg<L>::NT, Z2Cfg<L>::MINB) k_zconv2(float2* __restrict__ Y, const float* __restrict__ khat,
                                                             Dims d, const float2* __restrict__ gtw, int nkt,
                                                             int nlone, int ntiles, int tfirst,
                                                             const __grid_constant__ CUtensorMap tm) {
  using Z = Z2Cfg<L>;
  constexpr int NCH = Z::NCH, E = Z::E, TL = Z::TL, C = Z::C, NT = Z::NT, TWP = Z::TWP, LINE = Z::LINE;
  constexpr int EN = 8 * NCH;  // slots that can carry inputs / outputs (z = t + 16 i < nz <= L/2)
  constexpr int KLN = 3 * C / 16 + 2;  // 128-byte lines a Khat row segment (C x 24 bytes) can touch
  extern __shared__ __align__(128) float2 sm[];
  float2* twf = sm;                   // [ch][k][TWP]: w_L^{r (NCH k + ch)}
  float2* twi = sm + NCH * 16 * TWP;  // [ch][k][TWP]: w_L^{-k (NCH r + ch)}
  float2* buf = sm + Z::TWN;          // [component][channel][LINE]
  pdl_trigger();
  {  // all of a thread's table loads in flight at once (one L2 round trip per CTA, not four)
    constexpr int NE = (NCH * 256 + NT - 1) / NT;
    float2 wf[NE], wi[NE];
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int e = threadIdx.x + j * NT, ch = e >> 8, k = (e >> 4) & 15, r = e & 15;
      const int ef = (r * (NCH * k + ch)) % L, ei = (k * (NCH * r + ch)) % L;
      wf[j] = e < NCH * 256 ? __ldg(gtw + ef * (kTwMax / L)) : make_float2(0.f, 0.f);
      wi[j] = e < NCH * 256 ? __ldg(gtw + ei * (kTwMax / L)) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int e = threadIdx.x + j * NT, ch = e >> 8, k = (e >> 4) & 15, r = e & 15;
      if (e < NCH * 256) {
        twf[(ch * 16 + k) * TWP + r] = wf[j];
        twi[(ch * 16 + k) * TWP + r] = cconj(wi[j]);
      }
    }
  }
  __syncthreads();
  pdl_wait();
  const int c = threadIdx.x % C, t = (threadIdx.x / C) % TL, ch = threadIdx.x / (C * TL);
  const int nz = d.nzg, nzl = d.nz, hy = d.Ly / 2;
  const unsigned row = d.KXS, plane = (unsigned)d.Ly * row, cstr = (unsigned)nzl * plane;
  const unsigned kzs = (unsigned)(hy + 1) * d.kpitch * 3;  // Khat stride between kz rows (float2 units)
  const float inv_nzl = 1.f / (float)nzl, inv_nkt = 1.f / (float)nkt;
  // (kxl, ky) of lane cc in a tile; j / nkt in fp32: (j + 1/2) / nkt is >= 1/(2 nkt) >= 1/128 from
  // an integer and carries < 34 000 * 6e-8 of rounding error, so the truncation is exact
  auto lane_col = [&](int tile, int cc, int& kxl, int& ky) {
    if (tile < nlone) {
      kxl = d.kxw - 1;
      ky = tile * C + cc;
    } else {
      const int j = tile - nlone, kyi = __float2int_rz(((float)j + 0.5f) * inv_nkt), kt = j - kyi * nkt,
                kyh = kyi >> 1;
      kxl = kt * C + cc;
      ky = kyi == 1 ? hy : ((kyi & 1) ? d.Ly - kyh : kyh);
    }
  };
  // offset of global plane z; slabs: R[r][c][zl] blocks, r = z / nzl (exact in fp32, z < 1024)
  auto zoff = [&](int z) -> unsigned {
    unsigned a = (unsigned)z * plane;
    if constexpr (SPLIT) a += (unsigned)(2 * nzl * __float2int_rz(((float)z + 0.5f) * inv_nzl)) * plane;
    return a;
  };
  float2* const reg0 = buf + ch * LINE;              // component 0, this thread's channel
  float2* const reg1 = buf + (NCH + ch) * LINE;      // component 1
  float2* const reg2 = buf + (2 * NCH + ch) * LINE;  // component 2 (exchange only)
  float2 pf[TMA ? 1 : EN];  // (LDG path) the next inputs in flight: component g+1 or the next tile's 0
  __shared__ __align__(8) uint64_t bars[3];  // (TMA path) one per component region
  const int t0 = tfirst + blockIdx.x;
  // TMA: box (C columns, 1 row ky, nz planes) of component g at tile `tl` into region `reg`
  auto issue = [&](int tl, int g, float2* dst, uint64_t* bar) {
    int k0, ky0;
    lane_col(tl, 0, k0, ky0);
    mbar_arrive_expect_tx(bar, (uint32_t)(C * nz * sizeof(float2)));
    tma_load_3d(dst, &tm, k0, ky0, g * nz, bar);
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
      if (t0 < ntiles) {
        issue(t0, 0, reg2 - ch * LINE, &bars[2]);  // (reg2 of channel 0)
        issue(t0, 1, reg1 - ch * LINE, &bars[1]);
      }
    }
    __syncthreads();
  } else {
    int kxl, ky;
    lane_col(t0, c, kxl, ky);
    const bool ok = kxl < d.kxw && ky < d.Ly && t0 < ntiles;
    const unsigned col = (unsigned)min(ky, d.Ly - 1) * row + min(kxl, d.kxw - 1);
#pragma unroll
    for (int i = 0; i < EN; ++i) {
      const int z = t + 16 * i;
      pf[i] = (ok && z < nz) ? Y[col + zoff(z)] : make_float2(0.f, 0.f);
    }
  }
  uint32_t ph1 = 0, ph2 = 0;  // mbarrier phase parities (TMA path)
  for (int tile = t0; tile < ntiles; tile += gridDim.x) {
    const int nxt = tile + gridDim.x;
    if (!TMA && !MCQ_Z2NEXT && tile != t0) {  // component 0 of this tile (L2-prefetched)
      int kxl, ky;
      lane_col(tile, c, kxl, ky);
      const bool ok = kxl < d.kxw && ky < d.Ly;
      const unsigned col = (unsigned)min(ky, d.Ly - 1) * row + min(kxl, d.kxw - 1);
#pragma unroll
      for (int i = 0; i < EN; ++i) {
        const int z = t + 16 * i;
        pf[i] = (ok && z < nz) ? Y[col + zoff(z)] : make_float2(0.f, 0.f);
      }
    }
    // ---- L2 prefetch of the next (normal) tile: its 3 nz row segments of Y (C x 8 bytes, within
    // one 128-byte line) and its L/2 + 1 Khat row segments (C x 24 bytes: 2-3 lines), one
    // line per thread and instruction
    if (nxt < ntiles && nxt >= nlone) {
      int pk, pky;
      lane_col(nxt, 0, pk, pky);
      const int pkyf = pky <= hy ? pky : d.Ly - pky;
      const float2* py = Y + (unsigned)pky * row + pk;
      if (!TMA) {  // (the TMA path loads the inputs itself)
#pragma unroll 1
        for (int g = 0; g < 3; ++g)
          for (int z = threadIdx.x; z < nz; z += NT) prefetch_l2(py + g * cstr + zoff(z));
      }
      const float* pkh = khat + ((unsigned)pkyf * d.kpitch + d.kx0 - d.kxoff + pk) * 6;
      const unsigned kstride = (unsigned)(hy + 1) * d.kpitch * 6;
      for (int j = threadIdx.x; j < (L / 2 + 1) * KLN; j += NT) {  // C x 24 B: <= KLN lines
        const int kzf = j / KLN, q = j - kzf * KLN;
        prefetch_l2(pkh + kzf * kstride + q * 32);
      }
    }
    int kxl, ky;
    lane_col(tile, c, kxl, ky);
    const bool ok = kxl < d.kxw && ky < d.Ly;
    const unsigned col = (unsigned)min(ky, d.Ly - 1) * row + min(kxl, d.kxw - 1);
    if (tile == t0 && tile >= nlone) {  // this tile's Khat rows into L2 (needed after 3 transforms)
      const int pkyf = ky <= hy ? ky : d.Ly - ky;
      int k0, ky0;
      lane_col(tile, 0, k0, ky0);
      const int kyf0 = ky0 <= hy ? ky0 : d.Ly - ky0;
      const float* pkh = khat + ((unsigned)kyf0 * d.kpitch + d.kx0 - d.kxoff + k0) * 6;
      const unsigned kstride = (unsigned)(hy + 1) * d.kpitch * 6;
      (void)pkyf;
      for (int j = threadIdx.x; j < (L / 2 + 1) * KLN; j += NT) {
        const int kzf = j / KLN, q = j - kzf * KLN;
        prefetch_l2(pkh + kzf * kstride + q * 32);
      }
    }
    __syncthreads();  // the previous tile's shared-memory reads are done
    if (TMA && threadIdx.x == 0 && tile != t0) {  // component 1 into region 1 (free again)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile, 1, reg1 - ch * LINE, &bars[1]);
    }

    // ---- forward: component g in registers, 16 x 16 with one exchange; park g = 0, 1
    float2 v[E];
#pragma unroll 1
    for (int g = 0; g < 3; ++g) {
      if constexpr (TMA) {  // the staged box [z][c]: component 1 in region 1, 0 and 2 in region 2
        uint64_t* bar = g == 1 ? &bars[1] : &bars[2];
        mbar_wait(bar, g == 1 ? ph1 : ph2);
        if (g == 1) ph1 ^= 1u; else ph2 ^= 1u;
        const float2* box = (g == 1 ? reg1 : reg2) - ch * LINE;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int z = t + 16 * i;
          v[i] = (i < EN && z < nz) ? box[z * C + c] : make_float2(0.f, 0.f);
        }
        __syncthreads();  // every input read before the box is overwritten
        if (g == 0 && threadIdx.x == 0) {  // component 2 into region 2 (its box is consumed)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(tile, 2, reg2 - ch * LINE, &bars[2]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = i < EN ? pf[i] : make_float2(0.f, 0.f);
      }
      if (!TMA && g < 2) {
#pragma unroll
        for (int i = 0; i < EN; ++i) {
          const int z = t + 16 * i;
          pf[i] = (ok && z < nz) ? Y[col + (g + 1) * cstr + zoff(z)] : make_float2(0.f, 0.f);
        }
      }
      if (NCH == 2 && ch) {
#pragma unroll
        for (int i = 1; i < E; ++i) v[i] = cmul(v[i], w32c(i));
      }
      float2* R = g == 0 ? reg0 : (g == 1 ? reg1 : reg2);
      dft16<false>(v);
#pragma unroll
      for (int r = 0; r < 16; ++r) R[z2a<C>(16 * t + r, c)] = v[r];
      __syncthreads();
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = R[z2a<C>(t + 16 * i, c)];
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
        for (int i = 0; i < E; ++i) R[z2a<C>(t + 16 * i, c)] = v[i];  // own positions: no barrier
      }
    }

    // ---- Khat multiply at the own positions (kz = NCH (t + 16 i) + ch), component 2 in v; the
    // Khat loads of KB points are issued together (one L2 latency per batch, not per point)
    if (ok) {
      const int kx = d.kx0 + kxl;
      const int kyf = ky <= hy ? ky : d.Ly - ky;
      const float sy = ky <= hy ? 1.f : -1.f;
      const float2* kb = reinterpret_cast<const float2*>(khat) + ((unsigned)kyf * d.kpitch + kx - d.kxoff) * 3;
      constexpr int KB = MCQ_Z2KB > 0 ? MCQ_Z2KB : (NCH == 2 ? 4 : 8);
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
          const int a = z2a<C>(t + 16 * i, c);
          const float2 mx = reg0[a], my = reg1[a], mz = v[i];
          reg0[a] = fma2(bc2(kxz), mz, fma2(bc2(kxy), my, mul2(bc2(k01.x), mx)));
          reg1[a] = fma2(bc2(kyz), mz, fma2(bc2(k01.y), my, mul2(bc2(kxy), mx)));
          v[i] = fma2(bc2(k23.x), mz, fma2(bc2(kyz), my, mul2(bc2(kxz), mx)));
        }
      }
    }

    // ---- the next tile's component-0 inputs (in flight during the inverse phase)
    if (!TMA && MCQ_Z2NEXT && nxt < ntiles) {
      int nk, nky;
      lane_col(nxt, c, nk, nky);
      const bool nok = nk < d.kxw && nky < d.Ly;
      const unsigned ncol = (unsigned)min(nky, d.Ly - 1) * row + min(nk, d.kxw - 1);
#pragma unroll
      for (int i = 0; i < EN; ++i) {
        const int z = t + 16 * i;
        pf[i] = (nok && z < nz) ? Y[ncol + zoff(z)] : make_float2(0.f, 0.f);
      }
    }

    // ---- inverse: components 2, 1, 0; channel sum; store the nz real planes
#pragma unroll 1
    for (int g = 2; g >= 0; --g) {
      float2* R = g == 0 ? reg0 : (g == 1 ? reg1 : reg2);
      if (g < 2) {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = R[z2a<C>(t + 16 * i, c)];
      }
      __syncthreads();  // every own-position read of region g is done before the exchange
      if (TMA && g == 1 && threadIdx.x == 0 && nxt < ntiles) {  // region 2 is done with this tile
        if (MCQ_Z2TMAST) tma_store_wait_read();  // (and the TMA store of component 2 has read it)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(nxt, 0, reg2 - ch * LINE, &bars[2]);
      }
      dft16<true>(v);
#pragma unroll
      for (int r = 0; r < 16; ++r) R[z2a<C>(16 * t + r, c)] = v[r];
      __syncthreads();
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = R[z2a<C>(t + 16 * i, c)];
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
          if ((i < 8) == (ch == 1)) R[z2a<C>(t + 16 * i, c)] = v[i];
        __syncthreads();
        const float2* Pr = ch ? R - LINE : R + LINE;  // the partner channel's block
#pragma unroll
        for (int i = 0; i < E; ++i)
          if ((i < 8) == (ch == 0)) v[i] = add2(v[i], Pr[z2a<C>(t + 16 * i, c)]);
      }
      if constexpr (TMA && MCQ_Z2TMAST) {
        // the finished planes into the component's box [z][c] (channel-0 block of region g, read
        // by nobody any more once every thread has passed the barrier), one TMA tensor store
        __syncthreads();
        float2* box = R - ch * LINE;
#pragma unroll
        for (int i = 0; i < EN; ++i) {
          const int z = t + 16 * i;
          if ((NCH == 1 || (i < 8) == (ch == 0)) && z < nz) box[z * C + c] = v[i];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
          int k0, ky0;
          lane_col(tile, 0, k0, ky0);
          tma_store_3d(&tm, box, k0, ky0, g * nz);
        }
      } else if (ok) {
#pragma unroll
        for (int i = 0; i < EN; ++i) {
          const int z = t + 16 * i;
          if ((NCH == 1 || (i < 8) == (ch == 0)) && z < nz) Y[col + g * cstr + zoff(z)] = v[i];
        }
      }
    }
    if (TMA && MCQ_Z2TMAST && threadIdx.x == 0) tma_store_wait_read();  // boxes reusable next tile
  }
  if (TMA && MCQ_Z2TMAST && threadIdx.x == 0) tma_store_wait_all();
}

}  // namespace mcq
