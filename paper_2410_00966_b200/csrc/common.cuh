// common.cuh — shared device-side structures of the mcq library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <utility>

namespace mcq {

// ---------------------------------------------------------------- programmatic dependent launch
// The hot-path kernels can be launched with programmatic stream serialization: each CTA signals
// griddepcontrol.launch_dependents on entry (so the next kernel's CTAs may start on SMs freed by
// this kernel's last wave), runs its prologue (twiddle tables, barrier init) and only then waits
// with griddepcontrol.wait for the previous kernel's completion and memory before touching any
// buffer the previous kernels read or write.  Without the launch attribute both instructions are
// no-ops.  The runtime enables it per context (Dims::pdl) only where it measured faster: single
// slab, small grids (latency-bound; configs[0] 56.1 vs 59.5 us/step; configs[1] 1.067 vs 1.031
// ms/step slower) — never with device copies or NCCL calls between kernels.
#ifndef MCQ_PDL
#define MCQ_PDL 0  // off: 6 % on the latency-bound configs[0] only, slower on configs[1]
#endif
__device__ __forceinline__ void pdl_trigger() {
#if MCQ_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if MCQ_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // order the previous grid's generic-proxy writes before this thread's TMA (async-proxy) reads
  asm volatile("fence.proxy.async.global;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (MCQ_PDL && pdl) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr double kGamma = 1.7595e11;             // rad s^-1 T^-1 (reading C8)
constexpr double kMu0 = 4e-7 * 3.14159265358979323846;
constexpr double kHbar = 1.05457182e-34;         // J s
constexpr double kKB = 1.380649e-23;             // J K^-1, SI exact (thermal field, reading C-TH)
constexpr int kTwMax = 1024;                     // global twiddle table length (max FFT length)

// Sizes of one context's padded spectral layout.  Row layout, kx fastest:
//   X[c][z][y][P]    complex64 (x-spectrum of m; the demag spectrum in place), rows 16-byte aligned
//   Y[c][z][ky][P]   complex64 (after the y transform; only the nz real z planes)
//   Khat[kz][ky][kpitch][g] fp32, kz <= Lz/2, ky <= Ly/2 (real, folded; g = XX,YY,ZZ,XY,XZ,YZ
//                       interleaved: one multiply reads 24 contiguous bytes, three 8-byte loads)
//
// z-slab decomposition over NS ranks: nz below is the rank's number of planes,
// nzg the global one, zg0 the global index of local plane 0.  State arrays carry zoff (0 or 1)
// halo planes on each side: cell (x, y, z) of component c sits at c*cs + ((z+zoff)*ny + y)*nx + x.
// Y is kx-slab-major: Y[q][c][z][ky][KXS] with q = kx_owner(kx) the rank owning column kx in the
// z pass (columns [kx_first(q), kx_first(q+1)), KXS >= every rank's width); for NS == 1 this is
// exactly Y[c][z][ky][P] (KXS == P).  After the forward all-to-all a rank holds
// R[r][c][zl][ky][KXS] (r = source rank, z = r*nz + zl) for its kxw columns.
// kx split: blocks of KG columns (KG = 16 when NKX >= 16 NS, else the largest power of two with
// NKX / KG >= NS), KB = NKX / KG blocks spread evenly, the last rank also takes the tail columns.
struct Dims {
  int nx, ny, nz;     // grid (nz: local planes)
  int Lx, Ly, Lz;     // zero-padded FFT lengths (next pow2 >= 2n; 1 if n == 1), Lz from nzg
  int N2;             // Lx / 2: complex length of the packed real x-transform
  int NKX;            // Lx / 2 + 1: x-spectrum columns (Hermitian half)
  int P;              // row pitch of the spectra (complex), NKX rounded up to 16 (128-byte rows)
  long long N;        // nx * ny * nz (local cells)
  int nzg, zg0, zoff; // global planes, global z of local plane 0, halo planes per side
  long long cs;       // component stride of the state arrays: nx * ny * (nz + 2 zoff)
  int NS, KXS;        // kx slabs (ranks) and their storage width (KXS >= every slab's width)
  int kx0, kxw;       // first kx column and width of this rank's slab in the z pass
  int KG, KB;         // kx split: block size (power of two) and number of whole blocks
  int kpitch, kxoff;  // Khat storage: row pitch (columns) and first stored column — P and 0 unless
                      // a z-slab rank keeps only its kx slab [kxoff, kxoff + kpitch) (NCCL mode)
  int pdl;            // launch the passes with programmatic dependent launch (see above)
};

// owner of column kx and first column of rank q under the kx split above
__host__ __device__ __forceinline__ int kx_first(const Dims& d, int q) {
  return q >= d.NS ? d.NKX : d.KG * ((q * d.KB) / d.NS);
}
__host__ __device__ __forceinline__ int kx_owner(const Dims& d, int kx) {
  if (d.NS == 1) return 0;
  const int blk = kx / d.KG;
  if (blk >= d.KB) return d.NS - 1;
  const int q = ((blk + 1) * d.NS - 1) / d.KB;
  return q < d.NS - 1 ? q : d.NS - 1;
}

// Cavity modes (reading C-MM): mode 0 is the paper's single mode; extra
// modes are independent oscillators driven by their own overlaps, their fields add.
constexpr int kMaxModes = 4;

// Cavity state on the device (fp64), advanced once per step by k_cavity (a13).
struct CavState {
  double re[kMaxModes], im[kMaxModes];  // alpha_n per mode
  double t;                             // cavity clock t_n (shared)
  double W[kMaxModes];                  // overlaps of the last completed step
  long long step;
  float gc[kMaxModes][8];  // Gamma_k(t_n + c_s dt) = 2 Re(e^{-(kappa_k+iw_k) c_s dt} alpha_k,n) per stage s
  float ge[kMaxModes][8];  // a_k sinc(w_cut,k (t_n + c_s dt))
  long long trace_rows;    // trace rows recorded since the last reset (may exceed the capacity)
};

// Per-CTA fp64 partials of the stage-4 update, per slab [kNPart][CTA]: W_k = sum B_rms,k . m
// for k < kMaxModes, then sum m_x, m_y, m_z (the trace's spatial mean, NEXT-3)
constexpr int kNPart = kMaxModes + 3;
constexpr int kPartM = kMaxModes;  // index of sum m_x
constexpr int kTraceCols = 8;  // t, <mx>, <my>, <mz>, Re alpha, Im alpha, W, step

// Scalars the cavity kernels need (host precomputed in fp64 for a given dt).
struct CavParams {
  int nst;                                          // integrator stages (4: RK4, 7: Dormand-Prince)
  double cst[8];                                    // stage nodes c_s
  double ec_re[kMaxModes][8], ec_im[kMaxModes][8];  // e^{-(kappa_k + i w_k) c_s dt} per stage
  double ecn_re[kMaxModes], ecn_im[kMaxModes];      // e^{-(kappa_k + i w_k) dt}: the step advance
  double vc_over_hbar;        // V_c / hbar
  double Ms;
  double dt;
  double exc_amp[kMaxModes], exc_omega[kMaxModes];
  int cav_on[kMaxModes];      // B_rms,k nonzero (C14)
  int nmodes;
  int pdl;                    // launch K-CAV with programmatic dependent launch
  double* trace;              // [trace_cap][kTraceCols] or nullptr
  long long trace_cap;
  int trace_every;            // record after every trace_every-th step
  double inv_nmag;            // 1 / number of magnetic cells (spatial mean)
  long long* thstep;          // thermal noise step (reading C-TH): advanced by K-CAV iff th_count
  int th_count;               // 1 on the RK4 path (mcq_run), 0 for Dormand-Prince commits
};

enum UpdateMode : int { MODE_LLG = 0, MODE_RELAX = 1, MODE_FIELD = 2, MODE_MAXTORQUE = 3, MODE_X0 = 4, MODE_DP = 5 };

// Arguments of the fused update kernel K-U.
struct UpdateArgs {
  Dims d;
  int stage;          // 1..4 (MODE_LLG / MODE_RELAX)
  int mode;
  unsigned terms;     // MCQ_TERM_* mask
  const float* mS;    // stage state (SoA [3][N])
  const float* mN;    // m_n (SoA)
  float* mOut;        // m_{s+1} (stages 1-3) or m_{n+1} (stage 4, may alias mN)
  // z-slab halos as remote stores (SURVEY §8(e) "halos move P2P over NVLink"): the same-role
  // buffer of the z-neighbour slab — another slab of this context (loopback) or a peer rank's
  // buffer mapped over NVLink with CUDA IPC (NCCL mode) — or nullptr.  A CTA writing local plane
  // 0 also writes it into halo_lo's top halo plane (storage plane nz + 1); local plane nz - 1 goes
  // into halo_hi's bottom halo plane (storage plane 0).
  float* halo_lo;
  float* halo_hi;
  float* acc;         // RK4 accumulator k1 + 2k2 + 2k3 (SoA)
  float2* X;          // x-spectrum rows [3][nz][ny][P]: demag in, FFT(m_{s+1}) out
  const float* brms[kMaxModes];  // SoA map per mode or nullptr (then the uniform value)
  float brms_u[kMaxModes][3];
  int nmodes;
  float bext[3];
  float ex[3];        // 2A / (Ms d_axis^2)
  float ku, u[3];     // 2 K_u1 / Ms, axis
  float kc, c1[3], c2[3], c3[3];  // 2 K_c1 / Ms, axes
  float dmi[2];       // interfacial DMI: D / (Ms dx), D / (Ms dy) (0: off), reading C-DMI
  float gl;           // gamma / (1 + alpha^2)
  float alpha;
  float gamma;
  float h;            // c_{s+1} dt for stages 1..3
  float dt6;          // dt / 6
  const CavState* cav;
  double* partials;   // per-CTA overlap partials (stage 4)
  float* bout;        // MODE_FIELD output (SoA)
  unsigned* maxbits;  // MODE_MAXTORQUE output (float bits, >= 0)
  int* nonfinite;     // set to 1 by the step's last stage when some m_{n+1} is not finite
  // thermal field (reading C-TH): B_th = th * eta(th_seed, n, global cell), th = sqrt(2 alpha
  // k_B T / (gamma M_s V dt)) for the run's dt (0: off); eta from SplitMix64 + Box-Muller, drawn
  // once per step (n = *thstep, the noise step) and held for all its stages
  float th;
  unsigned long long th_seed;
  float* eta;         // MODE_LLG: the step's draw [3][cs], written by stage 1, read by 2-4 (or nullptr)
  const long long* thstep;  // noise step n of the draw (device word; not the cavity step count)
  int demag;          // run the x-C2R demag phase
  int trace;          // stage 4: also accumulate sum m for the trace
  // MODE_DP (Dormand-Prince, reading C-DP), stage s = 1..7 with h = dt: K[j] = k_{j+1} ([3][cs]
  // each), comb[j] (j < s) the weights of k_1..k_s: stages 1-6 write
  // m_{s+1} = norm(m_n + h sum_j comb[j] k_{j+1}) and K[s-1] = k_s; stage 7 reduces
  // max |h sum_j comb[j] k_{j+1}| (comb = b5 - b4) into maxbits and takes W of its own state
  float* K;
  float comb[8];
};

// ---------------------------------------------------------------- launchers
// passes.cu
void configure_pass_kernels();
// (pass launchers return the number of kernels they launched: a narrow tail launch covers the
// last kx columns beyond the final full column tile)
// comp < 0: all three components in one launch; 0..2: that component only
int launch_yfwd(const Dims& d, const float2* X, float2* Y, const float2* tw, cudaStream_t s, int comp = -1);
int launch_zconv(const Dims& d, float2* Y, const float* khat, const float2* tw, cudaStream_t s);
// tmap2: CUtensorMaps for the TMA-staged K-Z: Y with boxes (zconv2_box_c(Lz), 1, nz) for v2 and
// (16, 1, nz) for v3 at Lz = 512, then Khat for v3 (valid iff khat_map), or nullptr
int launch_zconv_seq(const Dims& d, float2* Y, const float* khat, const float2* tw, cudaStream_t s,
                     const void* tmap2 = nullptr, bool khat_map = false);
int zconv2_box_c(int Lz);
int zconv_tma_box_c(int Lz);  // kx columns per K-Z tile of the TMA-pipelined variant
int launch_zconv_tma(const Dims& d, const void* tmap /* CUtensorMap over Y */, float2* Y, const float* khat,
                     const float2* tw, cudaStream_t s);
int launch_yinv(const Dims& d, const float2* Y, float2* X, const float2* tw, cudaStream_t s, int comp = -1);
int launch_y2d(const Dims& d, float2* X, const float* khat, const float2* tw, cudaStream_t s);
// update.cu
void configure_update_kernels();
void launch_update(const UpdateArgs& a, const float2* tw, cudaStream_t s);
int update_grid_blocks(const Dims& d);
// persistent cooperative kernel for nz == 1 grids (plain RK4, one mode): `steps` steps in one launch;
// returns 0, or -1 when this (N2, Ly) has no instance / the cooperative launch failed
int launch_persist2d(const UpdateArgs u[4], const CavParams& cp, CavState* cav, const float* khat, int steps,
                     const float2* tw, cudaStream_t s);
void launch_cavity(const CavParams& p, CavState* st, const double* partials, int nps, int nbx, int nzl, int nzg,
                   const double* psum_in, cudaStream_t s);
void launch_plane_sums(const CavParams& p, const double* partials, int nps, int nbx, int nzl, double* psum,
                       cudaStream_t s);
void launch_cav_prepare(const CavParams& p, CavState* st, cudaStream_t s);
void launch_aos_to_soa(const float* in, float* out, const uint8_t* mask, long long N, long long cs, long long off,
                       int* bad, cudaStream_t s);
void launch_soa_to_aos(const float* in, float* out, long long N, long long cs, long long off, cudaStream_t s);
void launch_deinterleave(const float* in, float* out, long long N, long long cs, long long off, cudaStream_t s);
// spectro.cu (NEXT-3: spectra, peaks and the anticrossing fit on the device)
int spectrum_peaks_device(int nb, const double* const* d_sig, const long long* d_n, const int* d_stride,
                          const double* d_dt, long long nmax, int pad, int window, double fmin, int npeaks,
                          double* f_out, double* a_out, int* nfound, cudaStream_t s);
int fit_anticrossing_device(int n, const double* w_mag, const double* lo, const double* hi, double wc0, double g0,
                            double* wc, double* g);
void launch_sp_dt(const double* const* d_trace, const long long* d_rows, double* d_dt, int nb, cudaStream_t s);
// tensor.cu
void launch_tensor_octant(double* oct, const Dims& d, double dx, double dy, double dz,
                          cudaStream_t s);
void launch_axis_transform(const double* in, double* out, int m0, int m1, int m2, int axis,
                           const double* Tcos, const double* Tsin, cudaStream_t s);
void launch_khat_finalize(const double* in, float* khat, const Dims& d, int kxoff, int kpitch, double scale,
                          cudaStream_t s);

}  // namespace mcq
