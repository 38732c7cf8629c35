// mcq.cu — host runtime and C ABI (include/mcq.h) of the B200-native Mumax3-cQED hot path.
//
// One step: for each RK4 stage s = 1..4
//     [3D] K-Y (X->Y), K-Z (Y, Khat), K-YI (Y->X)   |   [nz == 1] K-Y2D (X, Khat)
//     K-U(stage s): x-C2R demag + fields + torque + RK4 combine + x-R2C of m_{s+1} (+ W partials)
// then K-CAV: fixed-order W sum, alpha_{n+1}, t_{n+1}, stage factors of the next step.
// Steps are captured once into CUDA graphs and replayed; the host never synchronises inside
// mcq_run.  Device memory is owned by the context (cudaMalloc); work runs on the context
// stream (library-owned, or the caller's via mcq_set_stream).
#include <cuda.h>  // CUtensorMap; cuTensorMapEncodeTiled is fetched with cudaGetDriverEntryPoint
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/mcq.h"
#include "common.cuh"

using namespace mcq;

struct mcq_ctx {
  Dims d{};
  double dx = 0, dy = 0, dz = 0, Ms = 0, Aex = 0, alpha = 0;
  mcq_aniso K{};
  int device = 0;
  cudaStream_t stream = nullptr;  // work stream (user's or own)
  cudaStream_t own = nullptr;
  cudaStream_t cap = nullptr;     // capture stream
  float *mN = nullptr, *mA = nullptr, *mB = nullptr, *acc = nullptr;
  float2 *X = nullptr, *Y = nullptr, *tw = nullptr;
  float* khat = nullptr;
  float* brms = nullptr;
  double brms_u[3] = {0, 0, 0};
  bool cav_on = false;
  uint8_t* mask = nullptr;
  double bext[3] = {0, 0, 0};
  double fc = 1e9, kappa = 0, x0 = 0, p0 = 0, exc_amp = 0, exc_omega = 0;
  CavState* cav = nullptr;
  double* partials = nullptr;
  int nparts = 0;
  float* fieldbuf = nullptr;
  unsigned* maxbits = nullptr;
  int* bad = nullptr;
  float* io = nullptr;
  bool m_set = false;
  // graphs: [0] = 1 LLG step, [1] = kGraphSteps LLG steps, [2] = 1 relax step, [3] = relax chunk
  cudaGraphExec_t g[4] = {nullptr, nullptr, nullptr, nullptr};
  double g_dt[4] = {0, 0, 0, 0};
  long long launches = 0;
  alignas(64) CUtensorMap tmz;  // TMA descriptor of Y for the pipelined K-Z kernel
  bool have_tmz = false;
  std::string err;
};

namespace {

constexpr int kGraphSteps = 8;
constexpr int kRelaxCheck = 50;

int fail(mcq_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(ctx, call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? MCQ_ENOMEM : MCQ_ECUDA,           \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}
int padded(int n) { return n == 1 ? 1 : next_pow2(2 * n); }

void invalidate_graphs(mcq_ctx* c) {
  for (int i = 0; i < 4; ++i) {
    if (c->g[i]) cudaGraphExecDestroy(c->g[i]);
    c->g[i] = nullptr;
  }
}

CavParams cav_params(const mcq_ctx* c, double dt) {
  CavParams p{};
  const double w = 2.0 * M_PI * c->fc;
  const double cs[3] = {0.0, 0.5, 1.0};
  for (int i = 0; i < 3; ++i) {
    const double a = cs[i] * dt;
    const double dec = std::exp(-c->kappa * a);
    p.ec_re[i] = dec * std::cos(w * a);
    p.ec_im[i] = -dec * std::sin(w * a);
  }
  p.vc_over_hbar = c->dx * c->dy * c->dz / kHbar;
  p.Ms = c->Ms;
  p.dt = dt;
  p.exc_amp = c->exc_amp;
  p.exc_omega = c->exc_omega;
  p.cav_on = c->cav_on ? 1 : 0;
  return p;
}

UpdateArgs base_args(const mcq_ctx* c) {
  UpdateArgs a{};
  a.d = c->d;
  a.terms = MCQ_TERM_ALL;
  a.brms = c->brms;
  for (int i = 0; i < 3; ++i) {
    a.brms_u[i] = (float)c->brms_u[i];
    a.bext[i] = (float)c->bext[i];
  }
  a.ex[0] = (float)(2.0 * c->Aex / (c->Ms * c->dx * c->dx));
  a.ex[1] = (float)(2.0 * c->Aex / (c->Ms * c->dy * c->dy));
  a.ex[2] = (float)(2.0 * c->Aex / (c->Ms * c->dz * c->dz));
  auto unit = [](const double* v, float* o) {
    const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int i = 0; i < 3; ++i) o[i] = n > 0 ? (float)(v[i] / n) : 0.f;
  };
  a.ku = (float)(2.0 * c->K.ku1 / c->Ms);
  unit(c->K.u, a.u);
  a.kc = (float)(2.0 * c->K.kc1 / c->Ms);
  {
    double c1[3], c2[3], n1, n2;
    n1 = std::sqrt(c->K.c1[0] * c->K.c1[0] + c->K.c1[1] * c->K.c1[1] + c->K.c1[2] * c->K.c1[2]);
    n2 = std::sqrt(c->K.c2[0] * c->K.c2[0] + c->K.c2[1] * c->K.c2[1] + c->K.c2[2] * c->K.c2[2]);
    for (int i = 0; i < 3; ++i) {
      c1[i] = n1 > 0 ? c->K.c1[i] / n1 : 0;
      c2[i] = n2 > 0 ? c->K.c2[i] / n2 : 0;
    }
    const double c3[3] = {c1[1] * c2[2] - c1[2] * c2[1], c1[2] * c2[0] - c1[0] * c2[2], c1[0] * c2[1] - c1[1] * c2[0]};
    for (int i = 0; i < 3; ++i) {
      a.c1[i] = (float)c1[i];
      a.c2[i] = (float)c2[i];
      a.c3[i] = (float)c3[i];
    }
  }
  a.gl = (float)(kGamma / (1.0 + c->alpha * c->alpha));
  a.alpha = (float)c->alpha;
  a.gamma = (float)kGamma;
  a.cav = c->cav;
  a.partials = c->partials;
  a.bout = c->fieldbuf;
  a.maxbits = c->maxbits;
  a.X = c->X;
  a.acc = c->acc;
  a.demag = 1;
  return a;
}

// ---------------------------------------------------------------- enqueue helpers
typedef void (*KernelHook)(void* user, int kclass, bool begin);

struct Enq {
  mcq_ctx* c;
  cudaStream_t s;
  KernelHook hook = nullptr;
  void* user = nullptr;
  long long count = 0;
  void pre(int k) {
    if (hook) hook(user, k, true);
  }
  void post(int k) {
    ++count;
    if (hook) hook(user, k, false);
  }
  void demag() {
    const Dims& d = c->d;
    if (d.nz > 1) {
      pre(MCQ_K_YFWD);
      launch_yfwd(d, c->X, c->Y, c->tw, s);
      post(MCQ_K_YFWD);
      pre(MCQ_K_ZCONV);
      // K-Z variant (measured on configs[1], 1x B200: seq 170 us, tma 180 us, plain 206 us per
      // launch); MCQ_ZVARIANT=tma|plain selects the others (experiments / profiling)
      static const char* zv = getenv("MCQ_ZVARIANT");
      if (zv && !strcmp(zv, "tma") && c->have_tmz)
        launch_zconv_tma(d, &c->tmz, c->Y, c->khat, c->tw, s);
      else if (zv && !strcmp(zv, "plain"))
        launch_zconv(d, c->Y, c->khat, c->tw, s);
      else
        launch_zconv_seq(d, c->Y, c->khat, c->tw, s);
      post(MCQ_K_ZCONV);
      pre(MCQ_K_YINV);
      launch_yinv(d, c->Y, c->X, c->tw, s);
      post(MCQ_K_YINV);
    } else {
      pre(MCQ_K_Y2D);
      launch_y2d(d, c->X, c->khat, c->tw, s);
      post(MCQ_K_Y2D);
    }
  }
  void update(UpdateArgs a) {
    pre(MCQ_K_UPDATE);
    launch_update(a, c->tw, s);
    post(MCQ_K_UPDATE);
  }
  void stage(int st, double dt, int mode, unsigned terms) {
    UpdateArgs a = base_args(c);
    a.mode = mode;
    a.stage = st;
    a.terms = terms;
    a.mN = c->mN;
    a.mS = st == 1 ? c->mN : (st == 2 ? c->mA : (st == 3 ? c->mB : c->mA));
    a.mOut = st == 1 ? c->mA : (st == 2 ? c->mB : (st == 3 ? c->mA : c->mN));
    a.h = (float)(st == 3 ? dt : 0.5 * dt);
    a.dt6 = (float)(dt / 6.0);
    demag();
    update(a);
  }
  void llg_step(double dt) {
    for (int st = 1; st <= 4; ++st) stage(st, dt, MODE_LLG, MCQ_TERM_ALL);
    const CavParams p = cav_params(c, dt);
    pre(MCQ_K_CAVITY);
    launch_cavity(p, c->cav, c->partials, c->nparts, s);
    post(MCQ_K_CAVITY);
  }
  void relax_step(double dt) {
    for (int st = 1; st <= 4; ++st)
      stage(st, dt, MODE_RELAX, MCQ_TERM_ALL & ~(MCQ_TERM_CAVITY | MCQ_TERM_EXCITATION));
  }
  void x0() {  // X <- R2C(m_n)
    UpdateArgs a = base_args(c);
    a.mode = MODE_X0;
    a.stage = 1;
    a.mS = c->mN;
    a.mN = c->mN;
    a.mOut = c->mN;
    update(a);
  }
  void eval(int mode, unsigned terms) {  // field / max-torque of m_n at stage 1, then restore X
    UpdateArgs a = base_args(c);
    a.mode = mode;
    a.stage = 1;
    a.terms = terms;
    a.mS = c->mN;
    a.mN = c->mN;
    a.mOut = c->mN;
    demag();
    update(a);
    x0();
  }
};

int capture(mcq_ctx* c, int which, double dt, int steps) {
  if (c->g[which] && c->g_dt[which] == dt) return MCQ_OK;
  if (c->g[which]) {
    cudaGraphExecDestroy(c->g[which]);
    c->g[which] = nullptr;
  }
  CK(c, cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
  Enq q{c, c->cap};
  for (int i = 0; i < steps; ++i) {
    if (which < 2)
      q.llg_step(dt);
    else
      q.relax_step(dt);
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e1 = cudaStreamEndCapture(c->cap, &graph);
  cudaError_t e2 = cudaPeekAtLastError();
  if (e1 != cudaSuccess || e2 != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return fail(c, MCQ_ECUDA, std::string("graph capture failed: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  }
  cudaError_t e3 = cudaGraphInstantiate(&c->g[which], graph, 0);
  cudaGraphDestroy(graph);
  if (e3 != cudaSuccess) return fail(c, MCQ_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e3));
  c->g_dt[which] = dt;
  return MCQ_OK;
}

int demag_kernels(const mcq_ctx* c) {
  return c->d.nz > 1 ? 3 : 1;
}

long long kernels_per_step(const mcq_ctx* c, bool llg) {
  return 4LL * (demag_kernels(c) + 1) + (llg ? 1 : 0);
}

int set_cav_state(mcq_ctx* c, double re, double im, double t, long long step) {
  CavState h{};
  h.re = re;
  h.im = im;
  h.t = t;
  h.step = step;
  CK(c, cudaMemcpyAsync(c->cav, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  const CavParams p = cav_params(c, 1e-12);
  launch_cav_prepare(p, c->cav, c->stream);
  CK(c, cudaGetLastError());
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int reset_memory(mcq_ctx* c) { return set_cav_state(c, 0.5 * c->x0, -0.5 * c->p0, 0.0, 0); }

// cos / sin transform matrices of one axis: T[k][o], k, o in [0, L/2]
void axis_matrices(int L, std::vector<double>& Tc, std::vector<double>& Ts) {
  const int M = L / 2 + 1;
  Tc.assign((size_t)M * M, 0.0);
  Ts.assign((size_t)M * M, 0.0);
  for (int k = 0; k < M; ++k)
    for (int o = 0; o < M; ++o) {
      const long long ph = ((long long)k * o) % L;  // exact argument reduction
      const double ang = 2.0 * M_PI * (double)ph / (double)L;
      const double w = (o == 0 || 2 * o == L) ? 1.0 : 2.0;
      Tc[(size_t)k * M + o] = (L == 1) ? 1.0 : w * std::cos(ang);
      Ts[(size_t)k * M + o] = (o == 0 || 2 * o == L || L == 1) ? 0.0 : 2.0 * std::sin(ang);
    }
}

// K-TEN: octant -> x, y, z cosine/sine sums -> folded, scaled fp32 Khat
int build_khat(mcq_ctx* c, double* oct_out /* optional host copy of the octant */) {
  const Dims& d = c->d;
  const int m0 = d.Lx / 2 + 1, m1 = d.Ly / 2 + 1, m2 = d.Lz / 2 + 1;
  const size_t n = 6ULL * m0 * m1 * m2;
  double *a = nullptr, *b = nullptr, *T = nullptr;
  CK(c, cudaMalloc(&a, n * sizeof(double)));
  if (cudaMalloc(&b, n * sizeof(double)) != cudaSuccess) {
    cudaFree(a);
    return fail(c, MCQ_ENOMEM, "tensor workspace");
  }
  launch_tensor_octant(a, d, c->dx, c->dy, c->dz, c->stream);
  int rc = MCQ_OK;
  if (oct_out) {
    if (cudaMemcpyAsync(oct_out, a, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
      rc = fail(c, MCQ_ECUDA, "octant copy");
  } else {
    const int Ls[3] = {d.Lx, d.Ly, d.Lz};
    const int ms[3] = {m0, m1, m2};
    size_t tmax = 0;
    for (int ax = 0; ax < 3; ++ax) tmax = std::max(tmax, (size_t)ms[ax] * ms[ax]);
    if (cudaMalloc(&T, 2 * tmax * sizeof(double)) != cudaSuccess) rc = fail(c, MCQ_ENOMEM, "tensor matrices");
    std::vector<double> Tc, Ts;
    double *src = a, *dst = b;
    for (int ax = 0; ax < 3 && rc == MCQ_OK; ++ax) {
      axis_matrices(Ls[ax], Tc, Ts);
      const size_t mm = (size_t)ms[ax] * ms[ax];
      if (cudaMemcpy(T, Tc.data(), mm * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
          cudaMemcpy(T + tmax, Ts.data(), mm * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
        rc = fail(c, MCQ_ECUDA, "tensor matrix upload");
        break;
      }
      launch_axis_transform(src, dst, m0, m1, m2, ax, T, T + tmax, c->stream);
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) rc = fail(c, MCQ_ECUDA, "axis transform");
      std::swap(src, dst);
    }
    if (rc == MCQ_OK) {
      const double scale = -kMu0 * c->Ms / ((double)d.Lx * d.Ly * d.Lz);
      launch_khat_finalize(src, c->khat, d, scale, c->stream);
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) rc = fail(c, MCQ_ECUDA, "khat finalize");
    }
  }
  cudaFree(a);
  cudaFree(b);
  if (T) cudaFree(T);
  return rc;
}

void free_all(mcq_ctx* c) {
  invalidate_graphs(c);
  void* ptrs[] = {c->mN, c->mA, c->mB, c->acc, c->X, c->Y, c->tw, c->khat, c->brms, c->mask,
                  c->cav, c->partials, c->fieldbuf, c->maxbits, c->bad, c->io};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->own) cudaStreamDestroy(c->own);
  if (c->cap) cudaStreamDestroy(c->cap);
}

// TMA descriptor of Y[3][nz][Ly][P] viewed as a 3D tensor (P, Ly, 3 nz) of 8-byte elements;
// box (C, 1, nz) = one component's z column block of a K-Z tile.  Without it (nz > 256, or no
// driver entry point) K-Z falls back to plain loads.
void make_y_tensor_map(mcq_ctx* c) {
  const Dims& d = c->d;
  c->have_tmz = false;
  if (d.nz < 2 || d.nz > 256 || !c->Y) return;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      cudaGetLastError();
      return;
    }
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)d.P, (cuuint64_t)d.Ly, (cuuint64_t)3 * d.nz};
  const cuuint64_t strides[2] = {(cuuint64_t)d.P * 8, (cuuint64_t)d.Ly * d.P * 8};
  const cuuint32_t box[3] = {(cuuint32_t)zconv_tma_box_c(d.Lz), 1, (cuuint32_t)d.nz};
  const cuuint32_t es[3] = {1, 1, 1};
  if (box[0] == 0) return;
  const CUresult r = enc(&c->tmz, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->Y, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  c->have_tmz = (r == CUDA_SUCCESS);
}

std::once_flag g_cfg_once;

}  // namespace

// ====================================================================== C ABI
extern "C" {

int mcq_create(mcq_ctx** out, const int grid[3], const double cell[3], double Ms, double Aex, double alpha,
               const mcq_aniso* K, const mcq_dist* dist) {
  if (!out || !grid || !cell) return MCQ_EINVAL;
  *out = nullptr;
  if (grid[0] < 2 || grid[1] < 2 || grid[2] < 1 || grid[0] > 512 || grid[1] > 512 || grid[2] > 512) return MCQ_EINVAL;
  if (!(cell[0] > 0 && cell[1] > 0 && cell[2] > 0)) return MCQ_EINVAL;
  if (!(Ms > 0) || !(Aex >= 0) || !(alpha >= 0)) return MCQ_EINVAL;
  if (dist && dist->world > 1) return MCQ_EINVAL;  // z-slab decomposition: not in this build
  mcq_ctx* c = new (std::nothrow) mcq_ctx();
  if (!c) return MCQ_ENOMEM;
  c->dx = cell[0];
  c->dy = cell[1];
  c->dz = cell[2];
  c->Ms = Ms;
  c->Aex = Aex;
  c->alpha = alpha;
  if (K) c->K = *K;
  Dims& d = c->d;
  d.nx = grid[0];
  d.ny = grid[1];
  d.nz = grid[2];
  d.Lx = padded(d.nx);
  d.Ly = padded(d.ny);
  d.Lz = padded(d.nz);
  d.N2 = d.Lx / 2;
  d.NKX = d.N2 + 1;
  d.P = (d.NKX + 15) / 16 * 16;  // 128-byte aligned spectrum rows: whole-sector column tiles, TMA rows
  d.N = (long long)d.nx * d.ny * d.nz;
  auto bail = [&](int code) {
    free_all(c);
    delete c;
    return code;
  };
  if (dist && dist->device >= 0) {
    if (cudaSetDevice(dist->device) != cudaSuccess) return bail(MCQ_ECUDA);
  }
  cudaGetDevice(&c->device);
  std::call_once(g_cfg_once, [] {
    configure_pass_kernels();
    configure_update_kernels();
  });
  if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess)
    return bail(MCQ_ECUDA);
  c->stream = (dist && dist->cuda_stream) ? (cudaStream_t)dist->cuda_stream : c->own;
  const size_t N3 = 3ULL * d.N;
  const size_t nX = 3ULL * d.nz * d.ny * d.P;
  const size_t nY = d.nz > 1 ? 3ULL * d.nz * d.Ly * d.P : 0;
  const size_t nK = 6ULL * (d.Lz / 2 + 1) * (d.Ly / 2 + 1) * d.P;
  c->nparts = update_grid_blocks(d);
  bool ok = cudaMalloc(&c->mN, N3 * 4) == cudaSuccess && cudaMalloc(&c->mA, N3 * 4) == cudaSuccess &&
            cudaMalloc(&c->mB, N3 * 4) == cudaSuccess && cudaMalloc(&c->acc, N3 * 4) == cudaSuccess &&
            cudaMalloc(&c->X, nX * 8) == cudaSuccess && (nY == 0 || cudaMalloc(&c->Y, nY * 8) == cudaSuccess) &&
            cudaMalloc(&c->khat, nK * 4) == cudaSuccess && cudaMalloc(&c->tw, kTwMax * 8) == cudaSuccess &&
            cudaMalloc(&c->cav, sizeof(CavState)) == cudaSuccess &&
            cudaMalloc(&c->partials, (size_t)c->nparts * 8) == cudaSuccess &&
            cudaMalloc(&c->maxbits, 4) == cudaSuccess && cudaMalloc(&c->bad, 4) == cudaSuccess &&
            cudaMalloc(&c->io, N3 * 4) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return bail(MCQ_ENOMEM);
  }
  // zero the spectra once (columns beyond NKX are never touched, keep them finite)
  if (cudaMemsetAsync(c->X, 0, nX * 8, c->stream) != cudaSuccess ||
      (nY && cudaMemsetAsync(c->Y, 0, nY * 8, c->stream) != cudaSuccess) ||
      cudaMemsetAsync(c->khat, 0, nK * 4, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->mN, 0, N3 * 4, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->acc, 0, N3 * 4, c->stream) != cudaSuccess)
    return bail(MCQ_ECUDA);
  // twiddles w_1024^m = exp(-2 pi i m / 1024), generated in fp64
  {
    std::vector<float2> h(kTwMax);
    for (int m = 0; m < kTwMax; ++m) {
      const double ang = 2.0 * M_PI * m / kTwMax;
      h[m] = make_float2((float)std::cos(ang), (float)-std::sin(ang));
    }
    if (cudaMemcpy(c->tw, h.data(), kTwMax * 8, cudaMemcpyHostToDevice) != cudaSuccess) return bail(MCQ_ECUDA);
  }
  if (build_khat(c, nullptr) != MCQ_OK) return bail(MCQ_ECUDA);
  make_y_tensor_map(c);
  if (reset_memory(c) != MCQ_OK) return bail(MCQ_ECUDA);
  *out = c;
  return MCQ_OK;
}

int mcq_set_stream(mcq_ctx* c, void* stream) {
  if (!c) return MCQ_EINVAL;
  CK(c, cudaStreamSynchronize(c->stream));
  c->stream = stream ? (cudaStream_t)stream : c->own;
  return MCQ_OK;
}

int mcq_set_geometry(mcq_ctx* c, const unsigned char* mask) {
  if (!c) return MCQ_EINVAL;
  if (!mask) {
    if (c->mask) cudaFree(c->mask);
    c->mask = nullptr;
    return MCQ_OK;
  }
  if (!c->mask) CK(c, cudaMalloc(&c->mask, c->d.N));
  CK(c, cudaMemcpyAsync(c->mask, mask, c->d.N, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (c->m_set) {  // zero m in vacuum now
    const long long N = c->d.N;
    launch_soa_to_aos(c->mN, c->io, N, c->stream);
    CK(c, cudaMemsetAsync(c->bad, 0, 4, c->stream));
    launch_aos_to_soa(c->io, c->mN, c->mask, N, c->bad, c->stream);
    Enq q{c, c->stream};
    q.x0();
    c->launches += q.count + 2;
    CK(c, cudaStreamSynchronize(c->stream));
  }
  return MCQ_OK;
}

static int set_m_common(mcq_ctx* c, const float* src_dev) {
  const long long N = c->d.N;
  CK(c, cudaMemsetAsync(c->bad, 0, 4, c->stream));
  launch_aos_to_soa(src_dev, c->mA, c->mask, N, c->bad, c->stream);
  int bad = 0;
  CK(c, cudaMemcpyAsync(&bad, c->bad, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (bad) return fail(c, MCQ_EINVAL, std::to_string(bad) + " magnetic cells with a zero or non-finite vector");
  CK(c, cudaMemcpyAsync(c->mN, c->mA, 3ULL * N * 4, cudaMemcpyDeviceToDevice, c->stream));
  Enq q{c, c->stream};
  q.x0();
  c->launches += q.count + 1;
  CK(c, cudaGetLastError());
  c->m_set = true;
  return MCQ_OK;
}

int mcq_set_m(mcq_ctx* c, const float* m) {
  if (!c || !m) return MCQ_EINVAL;
  CK(c, cudaMemcpyAsync(c->io, m, 3ULL * c->d.N * 4, cudaMemcpyHostToDevice, c->stream));
  return set_m_common(c, c->io);
}

int mcq_set_m_device(mcq_ctx* c, const float* d_m) {
  if (!c || !d_m) return MCQ_EINVAL;
  return set_m_common(c, d_m);
}

int mcq_set_bext(mcq_ctx* c, const double B[3]) {
  if (!c || !B) return MCQ_EINVAL;
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(B[i])) return fail(c, MCQ_EINVAL, "B_ext not finite");
  for (int i = 0; i < 3; ++i) c->bext[i] = B[i];
  invalidate_graphs(c);
  return MCQ_OK;
}

int mcq_set_brms(mcq_ctx* c, const float* map, const double uniform[3]) {
  if (!c || (!map && !uniform)) return MCQ_EINVAL;
  const long long N = c->d.N;
  if (map) {
    bool nz = false;
    for (long long i = 0; i < 3 * N; ++i) {
      if (!std::isfinite(map[i])) return fail(c, MCQ_EINVAL, "B_rms map not finite");
      nz = nz || map[i] != 0.f;
    }
    if (!c->brms) CK(c, cudaMalloc(&c->brms, 3ULL * N * 4));
    CK(c, cudaMemcpyAsync(c->io, map, 3ULL * N * 4, cudaMemcpyHostToDevice, c->stream));
    launch_deinterleave(c->io, c->brms, N, c->stream);  // AoS -> SoA, no normalisation
    c->launches += 1;
    CK(c, cudaStreamSynchronize(c->stream));
    c->brms_u[0] = c->brms_u[1] = c->brms_u[2] = 0.0;
    c->cav_on = nz;
  } else {
    for (int i = 0; i < 3; ++i)
      if (!std::isfinite(uniform[i])) return fail(c, MCQ_EINVAL, "B_rms not finite");
    if (c->brms) cudaFree(c->brms);
    c->brms = nullptr;
    for (int i = 0; i < 3; ++i) c->brms_u[i] = uniform[i];
    c->cav_on = uniform[0] != 0 || uniform[1] != 0 || uniform[2] != 0;
  }
  invalidate_graphs(c);
  return reset_memory(c) == MCQ_OK ? MCQ_OK : MCQ_ECUDA;
}

int mcq_set_cavity(mcq_ctx* c, double f_c, double kappa, double x0, double p0) {
  if (!c) return MCQ_EINVAL;
  if (!(f_c > 0) || !(kappa >= 0) || !std::isfinite(x0) || !std::isfinite(p0))
    return fail(c, MCQ_EINVAL, "f_c must be > 0, kappa >= 0");
  c->fc = f_c;
  c->kappa = kappa;
  c->x0 = x0;
  c->p0 = p0;
  invalidate_graphs(c);
  return reset_memory(c);
}

int mcq_set_excitation(mcq_ctx* c, double amplitude, double omega_cut) {
  if (!c || !std::isfinite(amplitude) || !std::isfinite(omega_cut)) return MCQ_EINVAL;
  c->exc_amp = amplitude;
  c->exc_omega = omega_cut;
  invalidate_graphs(c);
  return MCQ_OK;
}

int mcq_reset_memory(mcq_ctx* c) {
  if (!c) return MCQ_EINVAL;
  return reset_memory(c);
}

int mcq_run(mcq_ctx* c, double dt, long long steps) {
  if (!c) return MCQ_EINVAL;
  if (!(dt > 0) || steps < 0) return fail(c, MCQ_EINVAL, "dt must be > 0 and steps >= 0");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "mcq_run before mcq_set_m");
  if (steps == 0) return MCQ_OK;
  const CavParams p = cav_params(c, dt);
  launch_cav_prepare(p, c->cav, c->stream);
  c->launches += 1;
  int rc;
  if (steps >= kGraphSteps && (rc = capture(c, 1, dt, kGraphSteps)) != MCQ_OK) return rc;
  if (steps % kGraphSteps && (rc = capture(c, 0, dt, 1)) != MCQ_OK) return rc;
  for (long long i = 0; i < steps / kGraphSteps; ++i) CK(c, cudaGraphLaunch(c->g[1], c->stream));
  for (long long i = 0; i < steps % kGraphSteps; ++i) CK(c, cudaGraphLaunch(c->g[0], c->stream));
  c->launches += steps * kernels_per_step(c, true);
  return MCQ_OK;
}

int mcq_relax(mcq_ctx* c, double dt, double tol, long long max_steps, long long* taken) {
  if (!c) return MCQ_EINVAL;
  if (!(dt > 0) || max_steps < 0 || !(tol >= 0)) return fail(c, MCQ_EINVAL, "relax: dt > 0, tol >= 0");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "mcq_relax before mcq_set_m");
  int rc;
  long long done = 0;
  while (done < max_steps) {
    const long long k = std::min<long long>(kRelaxCheck, max_steps - done);
    if (k == kRelaxCheck) {
      if ((rc = capture(c, 3, dt, kRelaxCheck)) != MCQ_OK) return rc;
      CK(c, cudaGraphLaunch(c->g[3], c->stream));
    } else {
      if ((rc = capture(c, 2, dt, 1)) != MCQ_OK) return rc;
      for (long long i = 0; i < k; ++i) CK(c, cudaGraphLaunch(c->g[2], c->stream));
    }
    c->launches += k * kernels_per_step(c, false);
    done += k;
    CK(c, cudaMemsetAsync(c->maxbits, 0, 4, c->stream));
    Enq q{c, c->stream};
    q.eval(MODE_MAXTORQUE, MCQ_TERM_ALL & ~(MCQ_TERM_CAVITY | MCQ_TERM_EXCITATION));
    c->launches += q.count;
    unsigned bits = 0;
    CK(c, cudaMemcpyAsync(&bits, c->maxbits, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    float tmax;
    std::memcpy(&tmax, &bits, 4);
    if (tmax < tol) break;
  }
  if (taken) *taken = done;
  return reset_memory(c);
}

int mcq_synchronize(mcq_ctx* c) {
  if (!c) return MCQ_EINVAL;
  CK(c, cudaStreamSynchronize(c->stream));
  CK(c, cudaGetLastError());
  return MCQ_OK;
}

int mcq_get_m(mcq_ctx* c, float* m_out) {
  if (!c || !m_out) return MCQ_EINVAL;
  launch_soa_to_aos(c->mN, c->io, c->d.N, c->stream);
  c->launches += 1;
  CK(c, cudaMemcpyAsync(m_out, c->io, 3ULL * c->d.N * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int mcq_get_m_device(mcq_ctx* c, float* d_out) {
  if (!c || !d_out) return MCQ_EINVAL;
  launch_soa_to_aos(c->mN, d_out, c->d.N, c->stream);
  c->launches += 1;
  CK(c, cudaGetLastError());
  return MCQ_OK;
}

int mcq_get_field(mcq_ctx* c, float* b_out, unsigned terms) {
  if (!c || !b_out) return MCQ_EINVAL;
  if (!c->m_set) return fail(c, MCQ_ESTATE, "mcq_get_field before mcq_set_m");
  const long long N = c->d.N;
  if (!c->fieldbuf) CK(c, cudaMalloc(&c->fieldbuf, 3ULL * N * 4));
  const CavParams p = cav_params(c, 1e-12);
  launch_cav_prepare(p, c->cav, c->stream);
  Enq q{c, c->stream};
  q.eval(MODE_FIELD, terms & MCQ_TERM_ALL);
  launch_soa_to_aos(c->fieldbuf, c->io, N, c->stream);
  c->launches += q.count + 2;
  CK(c, cudaMemcpyAsync(b_out, c->io, 3ULL * N * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int mcq_get_cavity(mcq_ctx* c, mcq_cavity_state* out) {
  if (!c || !out) return MCQ_EINVAL;
  CavState h{};
  CK(c, cudaMemcpyAsync(&h, c->cav, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  out->t = h.t;
  out->re_alpha = h.re;
  out->im_alpha = h.im;
  out->gamma = 2.0 * h.re;
  out->W = h.W;
  out->n_photon = h.re * h.re + h.im * h.im;
  out->step = h.step;
  // S - i C = (hbar / V_c)(alpha_0 - e^{(kappa + i w) t} alpha)
  const double w = 2.0 * M_PI * c->fc, vc = c->dx * c->dy * c->dz;
  const double g = std::exp(c->kappa * h.t);
  const double er = g * std::cos(w * h.t), ei = g * std::sin(w * h.t);
  const double ar = er * h.re - ei * h.im, ai = er * h.im + ei * h.re;
  const double dr = 0.5 * c->x0 - ar, di = -0.5 * c->p0 - ai;
  out->S = kHbar / vc * dr;
  out->C = -kHbar / vc * di;
  return MCQ_OK;
}

int mcq_set_cavity_state(mcq_ctx* c, const mcq_cavity_state* in) {
  if (!c || !in) return MCQ_EINVAL;
  if (!std::isfinite(in->t) || !std::isfinite(in->re_alpha) || !std::isfinite(in->im_alpha))
    return fail(c, MCQ_EINVAL, "non-finite cavity state");
  return set_cav_state(c, in->re_alpha, in->im_alpha, in->t, in->step);
}

int mcq_cavity_status(const mcq_ctx* c) {
  if (!c) return MCQ_EINVAL;
  return c->cav_on ? 1 : 0;
}

long long mcq_kernel_launches(const mcq_ctx* c) { return c ? c->launches : -1; }

namespace {
struct Prof {
  cudaStream_t s;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  cudaEvent_t cur = nullptr;
};
void prof_hook(void* u, int k, bool begin) {
  Prof* p = (Prof*)u;
  if (begin) {
    cudaEventCreate(&p->cur);
    cudaEventRecord(p->cur, p->s);
  } else {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, p->s);
    p->ev.push_back({k, {p->cur, e}});
  }
}
}  // namespace

int mcq_profile_run(mcq_ctx* c, double dt, long long steps, double* kernel_ms, int* per_step) {
  if (!c || !kernel_ms) return MCQ_EINVAL;
  if (!(dt > 0) || steps <= 0) return fail(c, MCQ_EINVAL, "profile: dt > 0, steps > 0");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "profile before set_m");
  const CavParams p = cav_params(c, dt);
  launch_cav_prepare(p, c->cav, c->stream);
  Prof pr{c->stream};
  Enq q{c, c->stream, prof_hook, &pr};
  for (long long i = 0; i < steps; ++i) q.llg_step(dt);
  c->launches += q.count + 1;
  CK(c, cudaStreamSynchronize(c->stream));
  double tot[MCQ_NKCLASS] = {0};
  int cnt[MCQ_NKCLASS] = {0};
  for (auto& e : pr.ev) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.second.first, e.second.second);
    tot[e.first] += ms;
    cnt[e.first] += 1;
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  for (int k = 0; k < MCQ_NKCLASS; ++k) {
    kernel_ms[k] = cnt[k] ? tot[k] / cnt[k] : 0.0;
    if (per_step) per_step[k] = (int)(cnt[k] / steps);
  }
  CK(c, cudaGetLastError());
  return MCQ_OK;
}

int mcq_debug_layout(const mcq_ctx* c, long long out[6]) {
  if (!c || !out) return MCQ_EINVAL;
  out[0] = c->d.Lx;
  out[1] = c->d.Ly;
  out[2] = c->d.Lz;
  out[3] = c->d.NKX;
  out[4] = c->d.P;
  out[5] = c->nparts;
  return MCQ_OK;
}

int mcq_debug_tensor_octant(mcq_ctx* c, double* out) {
  if (!c || !out) return MCQ_EINVAL;
  return build_khat(c, out);
}

int mcq_debug_khat(mcq_ctx* c, float* out) {
  if (!c || !out) return MCQ_EINVAL;
  const size_t nK = 6ULL * (c->d.Lz / 2 + 1) * (c->d.Ly / 2 + 1) * c->d.P;
  CK(c, cudaMemcpyAsync(out, c->khat, nK * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

const char* mcq_last_error(const mcq_ctx* c) { return c ? c->err.c_str() : "null context"; }

void mcq_destroy(mcq_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  free_all(c);
  delete c;
}

}  // extern "C"
