// zconv3.cuh — K-Z for Lz = 256 / 512 with the column slice held in registers (a3 of SURVEY §8(a):
// forward z FFT, Khat multiply, inverse z FFT).  Included by passes.cu; MCQ_Z3 selects it.
//
// Same arithmetic as K-Z v2 (zconv2.cuh: frequency channels X[2k + ch] = DFT_256(x[n] w_512^{n ch}),
// 16 x 16 transforms, the same twiddle tables, the same Khat fold), redistributed so that
// shared memory carries only the 16 x 16 exchanges.  The ncu evidence for v2 (profiles/
// r2_final_ncu.md): 27.5 eight-byte shared-memory passes per column element — 1.97 ms of its
// 3.55 ms at configs[4] — of which 15.5 are parking components 0 / 1 around the multiply, the
// channel hand-over, the reads of the staged input boxes by both channels and the output boxes.
//  * A thread owns one column position set (t + 16 i, i < 16) for BOTH channels and ALL three
//    components: X[3][2][16] complex = 192 registers through the Khat multiply, which then runs
//    in registers in place; the two channel halves of an inverse output are summed in registers.
//    Shared passes per element: 12 (two per 16 x 16 exchange, six transforms) + 1 (input box).
//  * 256 threads = 16 columns x 16 positions per CTA, one CTA per SM (launch bounds (256, 1): up
//    to 255 registers), persistent over the (16-column, ky) tiles; 16 columns = 128-byte rows.
//  * Two shared regions alternate roles.  Tile j's inputs (TMA tensor boxes, 16 columns x 1 row
//    x nz planes per component) arrive in region b; once they are in registers, region b is the
//    exchange area.  Tile j's Khat rows are copied into region b^1 (TMA, [kz][C][3])
//    during the forward transforms — with one CTA per SM nothing else would hide the Khat load
//    latency (ncu r2t: 24 % of the stall samples on the multiply when it loaded from L2); after
//    the multiply, region b^1 receives tile j+1's input boxes during the inverse transforms.
//    Outputs: plain coalesced stores from registers.
//  * The lone Nyquist column (NKX = 16 q + 1) keeps v2's lone-tile launch.
#pragma once

namespace mcq {

#ifndef MCQ_Z3MINB256
#define MCQ_Z3MINB256 2  // Lz = 256: CTAs per SM asked of ptxas (2: the 128-register cap)
#endif
template <int L_>
struct Z3Cfg {
  static_assert(L_ == 256 || L_ == 512, "K-Z v3: Lz = 256 or 512");
  static constexpr int L = L_, NCH = L / 256, C = 16, TL = 16, NT = C * TL;  // 256 threads
  static constexpr int TWP = 18;                                              // as Z2Cfg
  static constexpr int TWN = 2 * NCH * 16 * TWP;                              // twf + twi (complex)
  static constexpr int LINE = 256 * C;                                        // one (channel) exchange block
  static constexpr int BOX = 3 * (L / 2) * C;                                 // one tile's inputs (nz <= L/2)
  static constexpr int NKB = (L / 2 + 1 + 128) / 129;                         // Khat boxes of 129 kz rows
  static constexpr int KH = NKB * 129 * 3 * C;                                // one tile's Khat ([kz][C][3] float2)
  static constexpr int XCH = NCH * LINE;                                      // one component's exchange
  static constexpr int REG0 = BOX > KH ? BOX : KH;
  static constexpr int REG = REG0 > XCH ? REG0 : XCH;                         // a region holds any of them
  static constexpr size_t SMEM = (size_t)(TWN + 2 * REG) * sizeof(float2);   // 207 KB (512), 104 KB (256)
  static constexpr int MINB = L == 256 ? MCQ_Z3MINB256 : 1;  // 512: up to 255 registers
};

// SPLIT (z slabs): the received kx-slab blocks R[source rank][component][zl][ky][KXS]; tm is then a
// 4D map (KXS, Ly, nzl, 3 NS) read with element stride 3 along its last dimension from q = g, so a
// component's box still lands as [z][c] (z = rank * nzl + zl); stores use zconv2.cuh's zoff.
template <int L_, bool SPLIT = false>
__global__ void __launch_bounds__(Z3Cfg<L_>::NT, Z3Cfg<L_>::MINB) k_zconv3(float2* __restrict__ Y, const float* __restrict__ khat,
                                                         Dims d, const float2* __restrict__ gtw, int nkt, int ntiles,
                                                         const __grid_constant__ CUtensorMap tm,
                                                         const __grid_constant__ CUtensorMap tmk) {
  using Z = Z3Cfg<L_>;
  constexpr int L = Z::L, NCH = Z::NCH, C = Z::C, NT = Z::NT, TWP = Z::TWP, LINE = Z::LINE, REG = Z::REG;
  extern __shared__ __align__(128) float2 sm[];
  float2* twf = sm;                   // [ch][k][TWP]: w_L^{r (NCH k + ch)}
  float2* twi = sm + NCH * 16 * TWP;  // [ch][k][TWP]: w_L^{-k (NCH r + ch)}
  float2* bufs = sm + Z::TWN;         // [2][REG]: regions that alternate between the roles below
  __shared__ __align__(8) uint64_t bars[3];  // input boxes of regions 0 / 1, Khat
  pdl_trigger();
  {  // twiddle tables (zconv2.cuh's, every load in flight at once)
    constexpr int NE = (NCH * 256 + NT - 1) / NT;
    float2 wf[NE], wi[NE];
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int e = threadIdx.x + j * NT, ch = e >> 8, k = (e >> 4) & 15, r = e & 15;
      wf[j] = __ldg(gtw + ((r * (NCH * k + ch)) % L) * (kTwMax / L));
      wi[j] = __ldg(gtw + ((k * (NCH * r + ch)) % L) * (kTwMax / L));
    }
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int e = threadIdx.x + j * NT, ch = e >> 8, k = (e >> 4) & 15, r = e & 15;
      twf[(ch * 16 + k) * TWP + r] = wf[j];
      twi[(ch * 16 + k) * TWP + r] = cconj(wi[j]);
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  const int c = threadIdx.x % C, t = threadIdx.x / C;
  const int nz = d.nzg, nzl = d.nz, hy = d.Ly / 2;  // global planes (the transform's inputs), this slab's
  const unsigned row = d.KXS, plane = (unsigned)d.Ly * row, cstr = (unsigned)nzl * plane;
  const float inv_nzl = 1.f / (float)nzl;
  auto zoff = [&](int z) -> unsigned {  // offset of global plane z (zconv2.cuh)
    unsigned a = (unsigned)z * plane;
    if constexpr (SPLIT) a += (unsigned)(2 * nzl * __float2int_rz(((float)z + 0.5f) * inv_nzl)) * plane;
    return a;
  };
  const unsigned kzs = (unsigned)(hy + 1) * d.kpitch * 3;  // Khat stride between kz rows (float2 units)
  const float inv_nkt = 1.f / (float)nkt;
  // first column and row of tile j: rows ky and Ly - ky back to back (same folded Khat rows);
  // j / nkt in fp32 is exact here (zconv2.cuh lane_col)
  auto tile_pos = [&](int j, int& kx0, int& ky) {
    const int kyi = __float2int_rz(((float)j + 0.5f) * inv_nkt), kt = j - kyi * nkt, kyh = kyi >> 1;
    kx0 = kt * C;
    ky = kyi == 1 ? hy : ((kyi & 1) ? d.Ly - kyh : kyh);
  };
  auto issue = [&](int j, int b) {  // thread 0: the three component boxes of tile j into buffer b
    int kx0, ky;
    tile_pos(j, kx0, ky);
    mbar_arrive_expect_tx(&bars[b], (uint32_t)(3 * C * nz * sizeof(float2)));
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      if constexpr (SPLIT)
        tma_load_4d(bufs + b * REG + g * (L / 2) * C, &tm, kx0, ky, 0, g, &bars[b]);
      else
        tma_load_3d(bufs + b * REG + g * (L / 2) * C, &tm, kx0, ky, g * nz, &bars[b]);
    }
  };
  // tile j's Khat rows into region Ks as [kz][C][3] float2 by two TMA tensor copies (tmk: Khat
  // viewed as (6 kpitch floats, Ly/2 + 1, Lz/2 + 1), box (6 C, 1, 129): kz rows 0-128 and 129-257,
  // the last one out of bounds and zero-filled).  (Per-thread 8-byte cp.async measured 2823 us
  // with 14 % of the samples on its loop; 257 1D bulk copies per tile 3856 us: the copy engine
  // serialises small requests.)
  auto khat_stage = [&](int j, float2* Ks) {
    if (threadIdx.x != 0) return;
    int kx0, ky;
    tile_pos(j, kx0, ky);
    const int kyf = ky <= hy ? ky : d.Ly - ky;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic accesses of the region
    mbar_arrive_expect_tx(&bars[2], (uint32_t)(Z::NKB * 129 * 6 * C * sizeof(float)));
#pragma unroll
    for (int q = 0; q < Z::NKB; ++q) tma_load_3d(Ks + q * 129 * 3 * C, &tmk, (d.kx0 - d.kxoff + kx0) * 6, kyf, 129 * q, &bars[2]);
  };
  // Per tile j with its inputs in region b: Khat(j) is staged into region b^1 (free: the previous
  // tile's exchange area) during the forward transforms; once the multiply has read it, the next
  // tile's input boxes go into region b^1 by TMA during the inverse transforms.
  const int t0 = blockIdx.x;
  if (t0 < ntiles && threadIdx.x == 0) issue(t0, 0);
  uint32_t ph0 = 0, ph1 = 0, phk = 0;
  int b = 0;
  for (int j = t0; j < ntiles; j += gridDim.x, b ^= 1) {
    const int jn = j + gridDim.x;
    __syncthreads();  // region b^1 (the previous tile's exchange area) is no longer read
    float2* Ks = bufs + (b ^ 1) * REG;
    khat_stage(j, Ks);
    mbar_wait(&bars[b], b ? ph1 : ph0);
    if (b) ph1 ^= 1u; else ph0 ^= 1u;
    float2* B = bufs + b * REG;
    int kx0, ky;
    tile_pos(j, kx0, ky);
    const int kxl = kx0 + c;
    const bool ok = kxl < d.kxw;

    // ---- inputs (z = t + 16 i < nz) into registers; then the buffer is the exchange area
    constexpr int EN = 8 * NCH;  // slots that can carry inputs / outputs (z = t + 16 i < nz <= L/2)
    float2 X[3][NCH][16];
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int z = t + 16 * i;
        X[g][0][i] = (i < EN && z < nz) ? B[g * (L / 2) * C + z * C + c] : make_float2(0.f, 0.f);
      }
    __syncthreads();

    // ---- forward, per component: both channels, one 16 x 16 exchange
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      if constexpr (NCH == 2) {
        X[g][NCH - 1][0] = X[g][0][0];
#pragma unroll
        for (int i = 1; i < 16; ++i) X[g][NCH - 1][i] = cmul(X[g][0][i], w32c(i));
      }
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) dft16<false>(X[g][ch]);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int r = 0; r < 16; ++r) B[ch * LINE + (16 * t + r) * C + c] = X[g][ch][r];
      __syncthreads();
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
        for (int i = 0; i < 16; ++i) X[g][ch][i] = B[ch * LINE + (t + 16 * i) * C + c];
        const float4* w4 = reinterpret_cast<const float4*>(twf + (ch * 16 + t) * TWP);
#pragma unroll
        for (int r2 = 0; r2 < 8; ++r2) {
          const float4 p = w4[r2];
          if (r2 > 0) X[g][ch][2 * r2] = cmul(X[g][ch][2 * r2], make_float2(p.x, p.y));
          X[g][ch][2 * r2 + 1] = cmul(X[g][ch][2 * r2 + 1], make_float2(p.z, p.w));
        }
        dft16<false>(X[g][ch]);
      }
      __syncthreads();  // the block is rewritten by the next component
    }

    // ---- Khat multiply in place at kz = 2 (t + 16 i) + ch, Khat from region b^1
    mbar_wait(&bars[2], phk);
    phk ^= 1u;
    if (ok) {
      const float sy = ky <= hy ? 1.f : -1.f;
#pragma unroll
      for (int i = 0; i < 16; ++i)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int kz = NCH * (t + 16 * i) + ch;
          const int kzf = i < 8 ? kz : L - kz;  // kz = L/2 (i = 8, t = ch = 0) folds to itself
          const float2* k2 = Ks + (kzf * C + c) * 3;
          const float2 k01 = k2[0], k23 = k2[1], k45 = k2[2];
          const float sz = i < 8 ? 1.f : -1.f;  // (the odd components vanish at kz = L/2)
          const float kxy = sy * k23.y, kxz = sz * k45.x, kyz = sy * sz * k45.y;
          const float2 mx = X[0][ch][i], my = X[1][ch][i], mz = X[2][ch][i];
          X[0][ch][i] = fma2(bc2(kxz), mz, fma2(bc2(kxy), my, mul2(bc2(k01.x), mx)));
          X[1][ch][i] = fma2(bc2(kyz), mz, fma2(bc2(k01.y), my, mul2(bc2(kxy), mx)));
          X[2][ch][i] = fma2(bc2(k23.x), mz, fma2(bc2(kyz), my, mul2(bc2(kxz), mx)));
        }
    }
    __syncthreads();  // Khat read: region b^1 takes the next tile's inputs
    if (jn < ntiles && threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(jn, b ^ 1);
    }

    // ---- inverse, per component: both channels, one exchange, the channel sum in registers
    const unsigned col = (unsigned)ky * row + (unsigned)min(kxl, d.kxw - 1);
#pragma unroll
    for (int g = 0; g < 3; ++g) {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) dft16<true>(X[g][ch]);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int r = 0; r < 16; ++r) B[ch * LINE + (16 * t + r) * C + c] = X[g][ch][r];
      __syncthreads();
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
        for (int i = 0; i < 16; ++i) X[g][ch][i] = B[ch * LINE + (t + 16 * i) * C + c];
        const float4* w4 = reinterpret_cast<const float4*>(twi + (ch * 16 + t) * TWP);
#pragma unroll
        for (int r2 = 0; r2 < 8; ++r2) {
          const float4 p = w4[r2];
          if (NCH == 2 || r2 > 0) X[g][ch][2 * r2] = cmul(X[g][ch][2 * r2], make_float2(p.x, p.y));
          X[g][ch][2 * r2 + 1] = cmul(X[g][ch][2 * r2 + 1], make_float2(p.z, p.w));
        }
        dft16<true>(X[g][ch]);
      }
      __syncthreads();  // the block is rewritten by the next component
      if constexpr (NCH == 2) {
#pragma unroll
        for (int i = 1; i < 16; ++i) X[g][NCH - 1][i] = cmul(X[g][NCH - 1][i], cconj(w32c(i)));
      }
      if (ok) {
#pragma unroll
        for (int i = 0; i < EN; ++i) {
          const int z = t + 16 * i;
          if (z < nz) Y[col + g * cstr + zoff(z)] = NCH == 2 ? add2(X[g][0][i], X[g][NCH - 1][i]) : X[g][0][i];
        }
      }
    }
  }
}

}  // namespace mcq
