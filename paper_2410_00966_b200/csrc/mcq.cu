// mcq.cu — host runtime and C ABI (include/mcq.h) of the B200-native Mumax3-cQED hot path.
//
// One step: for each RK4 stage s = 1..4
//     [z slabs > 1] halo exchange of the stage state (one plane per side)
//     [3D] K-Y (X->Y), [slabs > 1] all-to-all Y -> R, K-Z (Khat), [slabs > 1] all-to-all back,
//          K-YI (Y->X)                                   |   [nz == 1] K-Y2D (X, Khat)
//     K-U(stage s): x-C2R demag + fields + torque + RK4 combine + x-R2C of m_{s+1} (+ W partials)
// then [slabs > 1] all-gather of the W partials and K-CAV: fixed-order W sum, alpha_{n+1},
// t_{n+1}, stage factors of the next step.
// The grid is split into z slabs: one slab per process over NCCL (one GPU each),
// or all slabs inside one process on one GPU ("loopback": the exchanges become device copies —
// the test vehicle of the decomposition, bitwise equal to the undecomposed run).  Steps are
// captured once into CUDA graphs (kernels, copies and NCCL calls) and replayed; the host never
// synchronises inside mcq_run.  Device memory is owned by the context (cudaMalloc).
#include <cuda.h>  // CUtensorMap; cuTensorMapEncodeTiled is fetched with cudaGetDriverEntryPoint
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is dlopen'ed when a multi-process context is created
#include <nvtx3/nvToolsExt.h>  // header-only NVTX: no-ops unless a profiler attaches

#include <algorithm>
#include <cmath>
#include <cstddef>
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

namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool ok = false;
};

Nccl* nccl_api() {
  static Nccl api;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the libnccl already loaded in this process (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen(getenv("MCQ_NCCL_LIB") ? getenv("MCQ_NCCL_LIB") : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define S_(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym))
    S_(getUniqueId, "ncclGetUniqueId");
    S_(commInitRank, "ncclCommInitRank");
    S_(commDestroy, "ncclCommDestroy");
    S_(send, "ncclSend");
    S_(recv, "ncclRecv");
    S_(allGather, "ncclAllGather");
    S_(allReduce, "ncclAllReduce");
    S_(groupStart, "ncclGroupStart");
    S_(groupEnd, "ncclGroupEnd");
    S_(errStr, "ncclGetErrorString");
#undef S_
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv && api.allGather &&
             api.allReduce && api.groupStart && api.groupEnd && api.errStr;
  });
  return api.ok ? &api : nullptr;
}

// One z slab: its planes of the state (with halo planes when split), its spectra and maps.
struct Slab {
  Dims d{};
  float *mN = nullptr, *mA = nullptr, *mB = nullptr, *acc = nullptr;  // [3][cs]
  float2 *X = nullptr, *Y = nullptr, *R = nullptr;  // X [3][nz][ny][P]; Y, R [NS][3][nz][Ly][KXS]
  float* K = nullptr;  // Dormand-Prince slopes k_1..k_6, [6][3][cs] (allocated on first use)
  float* brms[kMaxModes] = {nullptr, nullptr, nullptr, nullptr};  // [3][cs] per mode (maps)
  float* eta = nullptr;    // thermal draw of the current step, [3][cs] (allocated while T > 0)
  float* field = nullptr;                           // [3][cs]
  uint8_t* mask = nullptr;                          // [nz][ny][nx]
  double* partials = nullptr;                       // into ctx partials (loopback) or own (NCCL)
  int nparts = 0;                                   // K-U CTAs of one stage (nbx * nz)
  double* psum = nullptr;                           // NCCL: this rank's plane sums [nz][kNPart]
  // z slabs: TMA descriptors for K-Z v3 in the [v2, v3, Khat] convention of mcq_ctx::tmz2 — [1]:
  // the received blocks R as 4D (KXS, Ly, nzl, 3 NS), [2]: this slab's Khat ([0] unused)
  alignas(64) CUtensorMap tm3[3];
  bool have_tm3 = false;
};

}  // namespace

struct mcq_ctx {
  Dims dg{};  // global dims (nz = global planes; used for the tensor and the layout report)
  double dx = 0, dy = 0, dz = 0, Ms = 0, Aex = 0, alpha = 0;
  mcq_aniso K{};
  int device = 0;
  int NS = 1;       // slabs
  int rank = 0;     // this process's slab (NCCL mode)
  int mode = 0;     // 0 single, 1 loopback (all slabs here), 2 NCCL (one slab per process)
  ncclComm_t comm = nullptr;
  // z-slab halos as remote stores from K-U (loopback: the neighbour slab's buffers; NCCL: the
  // neighbour ranks' buffers mapped with CUDA IPC, P2P over NVLink); false: copy / NCCL halos
  bool remote_halo = false;
  float* peer_lo[3] = {nullptr, nullptr, nullptr};  // NCCL: rank - 1's mN, mA, mB (IPC-mapped)
  float* peer_hi[3] = {nullptr, nullptr, nullptr};  // NCCL: rank + 1's
  cudaStream_t stream = nullptr;  // work stream (user's or own)
  cudaStream_t own = nullptr;
  cudaStream_t cap = nullptr;     // capture stream
  cudaStream_t side = nullptr;    // z-slab transposes, overlapped with the per-component y passes
  cudaEvent_t ev[8] = {};         // fork / join events of the overlapped schedule
  // overlap the slab transposes with the per-component y passes (side stream): on by default
  // under NCCL (the transfers use NVLink, not this GPU's HBM); off in loopback, where the
  // "transfers" are HBM copies competing with the passes (measured: 97.6 vs 65.1 ms/step,
  // configs[4] x 8 slabs) — mcq_set_slab_overlap switches it (the loopback tests run both)
  bool overlap = false;
  // nz == 1 grids: the persistent cooperative kernel (mcq_set_persistent_2d).  Off by default:
  // measured on configs[0] (64 x 64 x 1), one replica: 64.5 us/step vs 55.4 us for the per-step
  // graphs (its 9 grid barriers per step cost more than the graph's kernel boundaries); 32
  // concurrent replicas (a bias sweep): 77.2 vs 89.5 us per step for all 32 (1.70e9 vs 1.46e9
  // cell-updates/s) — the sweep driver and bench.py --batch switch it on
  bool persist2d = false;
  std::vector<Slab> sl;
  float2* tw = nullptr;
  float* khat = nullptr;
  int nmodes = 1;  // cavity modes (mode 0 = the paper's single mode; NEXT-2, reading C-MM)
  double brms_u[kMaxModes][3] = {};
  bool brms_map[kMaxModes] = {};
  bool cav_on[kMaxModes] = {};
  bool have_mask = false;
  double bext[3] = {0, 0, 0};
  double dmi = 0;  // interfacial DMI constant (J/m^2)
  double temperature = 0;           // K (reading C-TH; 0: no thermal field)
  unsigned long long th_seed = 0;   // SplitMix64 start state of the thermal stream
  double th_dt = 0;                 // dt of the last mcq_run: the field getter's thermal scale
  double fc[kMaxModes] = {1e9, 1e9, 1e9, 1e9}, kappa[kMaxModes] = {}, x0[kMaxModes] = {}, p0[kMaxModes] = {};
  double exc_amp[kMaxModes] = {}, exc_omega[kMaxModes] = {};
  CavState* cav = nullptr;
  double* partials = nullptr;  // all slabs' per-CTA partials [CTA][kNPart] in global z order
  int nparts = 0;              // CTAs of one stage-4 update (all slabs)
  double* psums = nullptr;     // NCCL: gathered plane sums [nzg][kNPart] (update.cu, K-CAV)
  double* trace = nullptr;     // NEXT-3 observables [trace_cap][kTraceCols]
  long long trace_cap = 0;
  int trace_every = 1;
  long long n_magnetic = 0;
  unsigned* maxbits = nullptr;
  long long* thstep = nullptr;  // thermal noise step n (reading C-TH), device word
  int* nonfinite = nullptr;  // divergence flag (set by the update kernel, read by mcq_synchronize)
  int* bad = nullptr;
  float* io = nullptr;  // AoS staging for the cells this context holds
  bool m_set = false;
  // graphs: [0] = 1 LLG step, [1] = kGraphSteps LLG steps, [2] = 1 relax step, [3] = relax chunk
  // graphs: [0]/[1] 1 / kGraphSteps LLG (RK4) steps, [2]/[3] 1 / 50 relax steps,
  // [4]/[5] 1 / kGraphSteps fixed Dormand-Prince steps
  cudaGraphExec_t g[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double g_dt[6] = {0, 0, 0, 0, 0, 0};
  long long g_launches[6] = {0, 0, 0, 0, 0, 0};
  long long launches = 0;
  alignas(64) CUtensorMap tmz;  // TMA descriptor of Y for the pipelined K-Z kernel (1 slab)
  bool have_tmz = false;
  alignas(64) CUtensorMap tmz2[3];  // TMA descriptors for K-Z (1 slab): Y with box (zconv2_box_c, 1,
                                    // nz) for v2, (16, 1, nz) for v3 (Lz = 256, 512); Khat for v3
  bool have_tmz2 = false;
  bool have_tmk = false;  // tmz2[2] (K-Z v3 needs it)
  std::string err;
  long long cells_here() const { return (long long)sl.size() * sl[0].d.N; }
  long long first_cell() const { return mode == 2 ? (long long)rank * sl[0].d.N : 0; }
};

namespace {

// NVTX ranges: one per public call that enqueues work, one per kernel class at enqueue time
// (visible in eager paths: mcq_profile_run, relax checks, the adaptive integrator, and the
// graph captures)
struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};
const char* kclass_name(int k) {
  static const char* n[] = {"K-Y", "K-Z", "K-YI", "K-Y2D", "K-U", "K-CAV"};
  return k >= 0 && k < 6 ? n[k] : "?";
}

constexpr int kGraphSteps = 8;
constexpr long long kPdlMaxCells = 1 << 16;  // PDL only where the step is launch-latency bound
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

#define NK(ctx, call)                                                                          \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess) return fail(ctx, MCQ_ENCCL, std::string(#call) + ": " + nccl_api()->errStr(r_)); \
  } while (0)

int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}
int padded(int n) { return n == 1 ? 1 : next_pow2(2 * n); }

void invalidate_graphs(mcq_ctx* c) {
  for (int i = 0; i < 6; ++i) {
    if (c->g[i]) cudaGraphExecDestroy(c->g[i]);
    c->g[i] = nullptr;
  }
}

// stage nodes c_s: classical RK4 (C1) and Dormand-Prince (C-DP)
constexpr double kRK4Nodes[4] = {0.0, 0.5, 0.5, 1.0};
constexpr double kDPNodes[7] = {0.0, 1.0 / 5, 3.0 / 10, 4.0 / 5, 8.0 / 9, 1.0, 1.0};

CavParams cav_params(const mcq_ctx* c, double dt, bool dp = false) {
  CavParams p{};
  p.nst = dp ? 7 : 4;
  for (int s = 0; s < p.nst; ++s) p.cst[s] = dp ? kDPNodes[s] : kRK4Nodes[s];
  for (int k = 0; k < kMaxModes; ++k) {
    const double w = 2.0 * M_PI * c->fc[k];
    auto factor = [&](double a, double& re, double& im) {  // e^{-(kappa + i w) a}
      const double dec = std::exp(-c->kappa[k] * a);
      re = dec * std::cos(w * a);
      im = -dec * std::sin(w * a);
    };
    for (int s = 0; s < p.nst; ++s) factor(p.cst[s] * dt, p.ec_re[k][s], p.ec_im[k][s]);
    factor(dt, p.ecn_re[k], p.ecn_im[k]);
    p.exc_amp[k] = c->exc_amp[k];
    p.exc_omega[k] = c->exc_omega[k];
    p.cav_on[k] = (k < c->nmodes && c->cav_on[k]) ? 1 : 0;
  }
  p.nmodes = c->nmodes;
  p.vc_over_hbar = c->dx * c->dy * c->dz / kHbar;
  p.Ms = c->Ms;
  p.dt = dt;
  p.trace = c->trace_cap > 0 ? c->trace : nullptr;
  p.trace_cap = c->trace_cap;
  p.trace_every = c->trace_every;
  p.inv_nmag = c->n_magnetic > 0 ? 1.0 / (double)c->n_magnetic : 0.0;
  p.pdl = c->sl.empty() ? 0 : c->sl[0].d.pdl;
  p.thstep = c->thstep;
  p.th_count = dp ? 0 : 1;
  return p;
}

// sigma of each B_th component for time step dt (reading C-TH, Mumax3's Brown field)
static double th_sigma(const mcq_ctx* c, double dt) {
  return std::sqrt(2.0 * c->alpha * kKB * c->temperature / (kGamma * c->Ms * c->dx * c->dy * c->dz * dt));
}

UpdateArgs base_args(const mcq_ctx* c, const Slab& s) {
  UpdateArgs a{};
  a.d = s.d;
  a.terms = MCQ_TERM_ALL;
  a.nmodes = c->nmodes;
  for (int k = 0; k < kMaxModes; ++k) {
    const bool on = k < c->nmodes;
    a.brms[k] = (on && c->brms_map[k]) ? s.brms[k] : nullptr;
    for (int i = 0; i < 3; ++i) a.brms_u[k][i] = on ? (float)c->brms_u[k][i] : 0.f;
  }
  for (int i = 0; i < 3; ++i) a.bext[i] = (float)c->bext[i];
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
  a.dmi[0] = (float)(c->dmi / (c->Ms * c->dx));
  a.dmi[1] = (float)(c->dmi / (c->Ms * c->dy));
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
  a.partials = s.partials;
  a.bout = s.field;
  a.maxbits = c->maxbits;
  a.nonfinite = c->nonfinite;
  a.thstep = c->thstep;
  a.X = s.X;
  a.acc = s.acc;
  a.demag = 1;
  a.trace = c->trace_cap > 0 ? 1 : 0;
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
  int rc = MCQ_OK;  // first failure of a copy / NCCL call
  long long halo_calls = 0;
  // same-role buffer (0 mN, 1 mA, 2 mB) of slab i's z-neighbours for K-U's remote halo stores
  float* halo_peer(int i, int role, bool lo) const {
    if (!c->remote_halo) return nullptr;
    auto buf = [&](const Slab& t) { return role == 0 ? t.mN : (role == 1 ? t.mA : t.mB); };
    if (c->mode == 1) {
      const int j = lo ? i - 1 : i + 1;
      return (j >= 0 && j < c->NS) ? buf(c->sl[j]) : nullptr;
    }
    if (c->mode == 2) return lo ? c->peer_lo[role] : c->peer_hi[role];
    return nullptr;
  }
  void pre(int k) {
    nvtxRangePushA(kclass_name(k));
    if (hook) hook(user, k, true);
  }
  void post(int k, int n = 1) {  // n: kernels the launcher issued
    count += n;
    if (hook) hook(user, k, false);
    nvtxRangePop();
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess && rc == MCQ_OK)
      rc = fail(c, MCQ_ECUDA, "slab exchange copy");
  }
  void nk(ncclResult_t r) {
    if (r != ncclSuccess && rc == MCQ_OK) rc = fail(c, MCQ_ENCCL, nccl_api()->errStr(r));
  }
  // one plane per side of the state buffer `which` (0 mN, 1 mA, 2 mB) into the neighbours' halos
  void halo(int which) {
    if (c->NS == 1) return;
    ++halo_calls;
    auto buf = [&](Slab& t) { return which == 0 ? t.mN : (which == 1 ? t.mA : t.mB); };
    const Dims& d = c->sl[0].d;
    const size_t pl = (size_t)d.nx * d.ny;
    const size_t bytes = pl * sizeof(float);
    if (c->mode == 1) {
      for (int r = 0; r < c->NS; ++r)
        for (int cc = 0; cc < 3; ++cc) {
          float* mine = buf(c->sl[r]) + cc * d.cs;
          if (r > 0) copy(buf(c->sl[r - 1]) + cc * d.cs + (d.nz + 1) * pl, mine + 1 * pl, bytes);
          if (r < c->NS - 1) copy(buf(c->sl[r + 1]) + cc * d.cs, mine + d.nz * pl, bytes);
        }
    } else {
      Nccl* n = nccl_api();
      float* b = buf(c->sl[0]);
      nk(n->groupStart());
      for (int cc = 0; cc < 3; ++cc) {
        float* mine = b + cc * d.cs;
        if (c->rank > 0) {
          nk(n->send(mine + pl, pl, ncclFloat, c->rank - 1, c->comm, s));
          nk(n->recv(mine, pl, ncclFloat, c->rank - 1, c->comm, s));
        }
        if (c->rank < c->NS - 1) {
          nk(n->send(mine + d.nz * pl, pl, ncclFloat, c->rank + 1, c->comm, s));
          nk(n->recv(mine + (d.nz + 1) * pl, pl, ncclFloat, c->rank + 1, c->comm, s));
        }
      }
      nk(n->groupEnd());
    }
  }
  // Y[q] of every slab r  <->  R[r] of slab q  (the z-slab <-> kx-slab transpose); comp < 0: the
  // whole (source, destination) block, else that component's contiguous third of it; on stream st
  void alltoall(bool forward, int comp = -1, cudaStream_t st = nullptr) {
    if (!st) st = s;
    const Dims& d = c->sl[0].d;
    const size_t cb = (size_t)d.nz * d.Ly * d.KXS;  // complex per component of a block
    const size_t blk = 3 * cb;                      // complex per (source, destination) block
    const size_t off = comp < 0 ? 0 : comp * cb, len = comp < 0 ? blk : cb;
    if (c->mode == 1) {
      for (int r = 0; r < c->NS; ++r)
        for (int q = 0; q < c->NS; ++q) {
          float2* y = c->sl[r].Y + q * blk + off;
          float2* rr = c->sl[q].R + r * blk + off;
          cudaError_t e = forward ? cudaMemcpyAsync(rr, y, len * sizeof(float2), cudaMemcpyDeviceToDevice, st)
                                  : cudaMemcpyAsync(y, rr, len * sizeof(float2), cudaMemcpyDeviceToDevice, st);
          if (e != cudaSuccess && rc == MCQ_OK) rc = fail(c, MCQ_ECUDA, "slab transpose copy");
        }
    } else {
      Nccl* n = nccl_api();
      Slab& sl = c->sl[0];
      nk(n->groupStart());
      for (int q = 0; q < c->NS; ++q) {
        float2* y = sl.Y + q * blk + off;
        float2* rr = sl.R + q * blk + off;
        nk(n->send(forward ? (const void*)y : (const void*)rr, 2 * len, ncclFloat, q, c->comm, st));
        nk(n->recv(forward ? (void*)rr : (void*)y, 2 * len, ncclFloat, q, c->comm, st));
      }
      nk(n->groupEnd());
    }
  }
  void record(int e, cudaStream_t st) {
    if (cudaEventRecord(c->ev[e], st) != cudaSuccess && rc == MCQ_OK) rc = fail(c, MCQ_ECUDA, "event record");
  }
  void wait(cudaStream_t st, int e) {
    if (cudaStreamWaitEvent(st, c->ev[e], 0) != cudaSuccess && rc == MCQ_OK) rc = fail(c, MCQ_ECUDA, "event wait");
  }
  void demag() {
    const int NS = c->NS;
    const Dims& d0 = c->sl[0].d;
    // z slabs, overlapped schedule: the y pass runs one component at a time and
    // each component's transpose goes out on the side stream while the next one is transformed;
    // after K-Z the transposes back come in component by component ahead of the inverse y pass
    const bool ovl = NS > 1 && c->side && c->overlap;
    if (d0.nzg > 1 && ovl) {
      record(0, s);
      wait(c->side, 0);  // fork: the side stream joins this stream (and an open graph capture)
      for (int g = 0; g < 3; ++g) {
        for (auto& sl : c->sl) {
          pre(MCQ_K_YFWD);
          const int n = launch_yfwd(sl.d, sl.X, sl.Y, c->tw, s, g);
          post(MCQ_K_YFWD, n);
        }
        record(1 + g, s);
        wait(c->side, 1 + g);
        alltoall(true, g, c->side);
      }
      record(4, c->side);
      wait(s, 4);
      for (auto& sl : c->sl) {
        pre(MCQ_K_ZCONV);
        const int n = launch_zconv_seq(sl.d, sl.R, c->khat, c->tw, s, sl.have_tm3 ? sl.tm3 : nullptr, sl.have_tm3);
        post(MCQ_K_ZCONV, n);
      }
      record(5, s);
      wait(c->side, 5);
      for (int g = 0; g < 3; ++g) {
        alltoall(false, g, c->side);
        record(g == 0 ? 6 : (g == 1 ? 7 : 4), c->side);
        wait(s, g == 0 ? 6 : (g == 1 ? 7 : 4));
        for (auto& sl : c->sl) {
          pre(MCQ_K_YINV);
          const int n = launch_yinv(sl.d, sl.Y, sl.X, c->tw, s, g);
          post(MCQ_K_YINV, n);
        }
      }
    } else if (d0.nzg > 1) {
      for (auto& sl : c->sl) {
        pre(MCQ_K_YFWD);
        const int n = launch_yfwd(sl.d, sl.X, sl.Y, c->tw, s);
        post(MCQ_K_YFWD, n);
      }
      if (NS > 1) alltoall(true);
      for (auto& sl : c->sl) {
        float2* Z = NS > 1 ? sl.R : sl.Y;
        pre(MCQ_K_ZCONV);
        // K-Z variant (measured on configs[1], 1x B200: seq 170 us, tma 180 us, plain 206 us per
        // launch); MCQ_ZVARIANT=tma|plain selects the others (single slab only)
        static const char* zv = getenv("MCQ_ZVARIANT");
        int n;
        if (NS == 1 && zv && !strcmp(zv, "tma") && c->have_tmz)
          n = launch_zconv_tma(sl.d, &c->tmz, Z, c->khat, c->tw, s);
        else if (NS == 1 && zv && !strcmp(zv, "plain"))
          n = launch_zconv(sl.d, Z, c->khat, c->tw, s);
        else
          n = NS > 1 ? launch_zconv_seq(sl.d, Z, c->khat, c->tw, s, sl.have_tm3 ? sl.tm3 : nullptr, sl.have_tm3)
                     : launch_zconv_seq(sl.d, Z, c->khat, c->tw, s, c->have_tmz2 ? c->tmz2 : nullptr, c->have_tmk);
        post(MCQ_K_ZCONV, n);
      }
      if (NS > 1) alltoall(false);
      for (auto& sl : c->sl) {
        pre(MCQ_K_YINV);
        const int n = launch_yinv(sl.d, sl.Y, sl.X, c->tw, s);
        post(MCQ_K_YINV, n);
      }
    } else {
      for (auto& sl : c->sl) {
        pre(MCQ_K_Y2D);
        const int n = launch_y2d(sl.d, sl.X, c->khat, c->tw, s);
        post(MCQ_K_Y2D, n);
      }
    }
  }
  void update(const UpdateArgs& a) {
    pre(MCQ_K_UPDATE);
    launch_update(a, c->tw, s);
    post(MCQ_K_UPDATE);
  }
  void stage(int st, double dt, int mode, unsigned terms) {
    const int sin_ = st == 1 ? 0 : (st == 2 ? 1 : (st == 3 ? 2 : 1));  // stage state buffer
    const int sout = st == 1 ? 1 : (st == 2 ? 2 : (st == 3 ? 1 : 0));  // its output buffer
    if (!c->remote_halo) halo(sin_);  // else the previous K-U wrote the halo planes remotely
    demag();
    for (int i = 0; i < (int)c->sl.size(); ++i) {
      UpdateArgs a = stage_args(i, st, dt, mode, terms);
      update(a);
    }
  }
  UpdateArgs stage_args(int i, int st, double dt, int mode, unsigned terms) const {
    Slab& sl = c->sl[i];
    const int sout = st == 1 ? 1 : (st == 2 ? 2 : (st == 3 ? 1 : 0));
    {
      UpdateArgs a = base_args(c, sl);
      a.halo_lo = halo_peer(i, sout, true);
      a.halo_hi = halo_peer(i, sout, false);
      a.mode = mode;
      a.stage = st;
      a.terms = terms;
      a.mN = sl.mN;
      a.mS = st == 1 ? sl.mN : (st == 2 ? sl.mA : (st == 3 ? sl.mB : sl.mA));
      a.mOut = st == 1 ? sl.mA : (st == 2 ? sl.mB : (st == 3 ? sl.mA : sl.mN));
      a.h = (float)(st == 3 ? dt : 0.5 * dt);
      a.dt6 = (float)(dt / 6.0);
      if (mode == MODE_LLG && c->temperature > 0) {  // one draw per step, held for its stages
        a.th = (float)th_sigma(c, dt);
        a.th_seed = c->th_seed;
        a.eta = sl.eta;
      }
      return a;
    }
  }
  // NCCL: this rank's plane sums of the overlap partials, all-gathered in z order (nzg x kNPart
  // doubles); single / loopback: K-CAV sums every slab's partials itself, in the same tree
  void gather_partials(const CavParams& p) {
    if (c->mode != 2) return;
    Slab& sl = c->sl[0];
    launch_plane_sums(p, sl.partials, sl.nparts, sl.nparts / sl.d.nz, sl.d.nz, sl.psum, s);
    ++count;
    nk(nccl_api()->allGather(sl.psum, c->psums, (size_t)sl.d.nz * kNPart, ncclDouble, c->comm, s));
  }
  void cavity(const CavParams& p) {
    gather_partials(p);
    const Slab& s0 = c->sl[0];
    pre(MCQ_K_CAVITY);
    launch_cavity(p, c->cav, c->partials, s0.nparts, s0.nparts / s0.d.nz, s0.d.nz, c->dg.nz,
                  c->mode == 2 ? c->psums : nullptr, s);
    post(MCQ_K_CAVITY);
  }
  void llg_step(double dt) {
    for (int st = 1; st <= 4; ++st) stage(st, dt, MODE_LLG, MCQ_TERM_ALL);
    cavity(cav_params(c, dt));
  }
  void relax_step(double dt) {
    for (int st = 1; st <= 4; ++st)
      stage(st, dt, MODE_RELAX, MCQ_TERM_ALL & ~(MCQ_TERM_CAVITY | MCQ_TERM_EXCITATION));
  }
  // ---------------- Dormand-Prince (reading C-DP): 7 stages, state buffers mN -> mA -> mB -> ...
  // stage s reads the state s-1 wrote (stage 1: m_n) and writes m_{s+1} to mA (s odd) / mB (s
  // even); stage 6 writes the step result y5 to mB, stage 7 evaluates k7 on it for the error
  void dp_stage(int st, double dt) {
    static const double A[7][7] = {
        {1.0 / 5},
        {3.0 / 40, 9.0 / 40},
        {44.0 / 45, -56.0 / 15, 32.0 / 9},
        {19372.0 / 6561, -25360.0 / 2187, 64448.0 / 6561, -212.0 / 729},
        {9017.0 / 3168, -355.0 / 33, 46732.0 / 5247, 49.0 / 176, -5103.0 / 18656},
        {35.0 / 384, 0.0, 500.0 / 1113, 125.0 / 192, -2187.0 / 6784, 11.0 / 84},
        {35.0 / 384 - 5179.0 / 57600, 0.0, 500.0 / 1113 - 7571.0 / 16695, 125.0 / 192 - 393.0 / 640,
         -2187.0 / 6784 + 92097.0 / 339200, 11.0 / 84 - 187.0 / 2100, -1.0 / 40}};  // b5 - b4
    const int in = st == 1 ? 0 : ((st - 1) % 2 == 1 ? 1 : 2);
    if (!c->remote_halo) halo(in);
    demag();
    for (int i = 0; i < (int)c->sl.size(); ++i) {
      Slab& sl = c->sl[i];
      UpdateArgs a = base_args(c, sl);
      if (st < 7) {
        a.halo_lo = halo_peer(i, st % 2 == 1 ? 1 : 2, true);
        a.halo_hi = halo_peer(i, st % 2 == 1 ? 1 : 2, false);
      }
      a.mode = MODE_DP;
      a.stage = st;
      a.mN = sl.mN;
      a.mS = in == 0 ? sl.mN : (in == 1 ? sl.mA : sl.mB);
      a.mOut = st % 2 == 1 ? sl.mA : sl.mB;
      a.h = (float)dt;
      a.K = sl.K;
      for (int j = 0; j < st; ++j) a.comb[j] = (float)A[st - 1][j];
      update(a);
    }
  }
  void dp_attempt(double dt) {
    for (int st = 1; st <= 6; ++st) dp_stage(st, dt);
    if (cudaMemsetAsync(c->maxbits, 0, 4, s) != cudaSuccess && rc == MCQ_OK) rc = fail(c, MCQ_ECUDA, "memset");
    dp_stage(7, dt);
    if (c->mode == 2)  // max over ranks (non-negative floats: the float order is the bit order)
      nk(nccl_api()->allReduce(c->maxbits, c->maxbits, 1, ncclFloat, ncclMax, c->comm, s));
  }
  void dp_commit(double dt) {  // m_n <- y5; every mode's alpha advances by dt on W(y5)
    for (auto& sl : c->sl) copy(sl.mN, sl.mB, 3ULL * sl.d.cs * sizeof(float));
    cavity(cav_params(c, dt, true));
  }
  void x0() {  // X <- R2C(m_n) in every slab
    for (auto& sl : c->sl) {
      UpdateArgs a = base_args(c, sl);
      a.mode = MODE_X0;
      a.stage = 1;
      a.mS = sl.mN;
      a.mN = sl.mN;
      a.mOut = sl.mN;
      update(a);
    }
  }
  void eval(int mode, unsigned terms) {  // field / max-torque of m_n at stage 1, then restore X
    halo(0);
    demag();
    for (auto& sl : c->sl) {
      UpdateArgs a = base_args(c, sl);
      a.mode = mode;
      a.stage = 1;
      a.terms = terms;
      a.mS = sl.mN;
      a.mN = sl.mN;
      a.mOut = sl.mN;
      if (mode == MODE_FIELD && (terms & MCQ_TERM_THERM) && c->temperature > 0 && c->th_dt > 0) {
        a.th = (float)th_sigma(c, c->th_dt);  // the draw the next step will use
        a.th_seed = c->th_seed;
      }
      update(a);
    }
    x0();
  }
};

int capture(mcq_ctx* c, int which, double dt, int steps) {
  if (c->g[which] && c->g_dt[which] == dt) return MCQ_OK;
  if (c->g[which]) {
    cudaGraphExecDestroy(c->g[which]);
    c->g[which] = nullptr;
  }
  // NCCL contexts: relaxed mode (NCCL may make capture-unsafe runtime calls on its own threads)
  CK(c, cudaStreamBeginCapture(c->cap, c->mode == 2 ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal));
  Enq q{c, c->cap};
  for (int i = 0; i < steps; ++i) {
    if (which < 2) {
      q.llg_step(dt);
    } else if (which < 4) {
      q.relax_step(dt);
    } else {
      q.dp_attempt(dt);
      q.dp_commit(dt);
    }
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e1 = cudaStreamEndCapture(c->cap, &graph);
  cudaError_t e2 = cudaPeekAtLastError();
  if (e1 != cudaSuccess || e2 != cudaSuccess || !graph || q.rc != MCQ_OK) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (q.rc != MCQ_OK) return q.rc;
    return fail(c, MCQ_ECUDA, std::string("graph capture failed: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  }
  cudaError_t e3 = cudaGraphInstantiate(&c->g[which], graph, 0);
  cudaGraphDestroy(graph);
  if (e3 != cudaSuccess) return fail(c, MCQ_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e3));
  c->g_dt[which] = dt;
  c->g_launches[which] = q.count;  // kernels one replay launches (the gpu_launches claim)
  return MCQ_OK;
}

int write_cav_state(mcq_ctx* c, const CavState& h) {
  CK(c, cudaMemcpyAsync(c->cav, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  const CavParams p = cav_params(c, 1e-12);
  launch_cav_prepare(p, c->cav, c->stream);
  CK(c, cudaGetLastError());
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int read_cav_state(mcq_ctx* c, CavState& h) {
  CK(c, cudaMemcpyAsync(&h, c->cav, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

// every mode back to alpha_0 = (x0 - i p0)/2 at t = 0 (ResetMemoryTerm; C6)
int reset_memory(mcq_ctx* c) {
  CavState h{};
  for (int k = 0; k < kMaxModes; ++k) {
    h.re[k] = 0.5 * c->x0[k];
    h.im[k] = -0.5 * c->p0[k];
  }
  return write_cav_state(c, h);
}

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

// K-TEN: octant -> x, y, z cosine/sine sums -> folded, scaled fp32 Khat (global grid)
int build_khat(mcq_ctx* c, double* oct_out /* optional host copy of the octant */) {
  const Dims& d = c->dg;
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
      // stream-ordered uploads: a plain cudaMemcpy from pageable memory may return before the
      // data lands and is not ordered with the (non-blocking) work stream — it made Khat
      // nondeterministic (stale matrices read by the transform)
      if (cudaMemcpyAsync(T, Tc.data(), mm * sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
          cudaMemcpyAsync(T + tmax, Ts.data(), mm * sizeof(double), cudaMemcpyHostToDevice, c->stream) !=
              cudaSuccess) {
        rc = fail(c, MCQ_ECUDA, "tensor matrix upload");
        break;
      }
      launch_axis_transform(src, dst, m0, m1, m2, ax, T, T + tmax, c->stream);
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) rc = fail(c, MCQ_ECUDA, "axis transform");
      std::swap(src, dst);
    }
    if (rc == MCQ_OK) {
      const double scale = -kMu0 * c->Ms / ((double)d.Lx * d.Ly * d.Lz);
      // a z-slab rank under NCCL keeps only its kx slab of Khat (1/world of the spectrum)
      const Dims& s0 = c->sl[0].d;
      launch_khat_finalize(src, c->khat, d, s0.kxoff, s0.kpitch, scale, c->stream);
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
  for (int r = 0; r < 3; ++r) {
    if (c->peer_lo[r]) cudaIpcCloseMemHandle(c->peer_lo[r]);
    if (c->peer_hi[r]) cudaIpcCloseMemHandle(c->peer_hi[r]);
    c->peer_lo[r] = c->peer_hi[r] = nullptr;
  }
  for (auto& s : c->sl) {
    void* ptrs[] = {s.mN, s.mA, s.mB, s.acc, s.X, s.Y, s.R, s.K, s.brms[0], s.brms[1], s.brms[2], s.brms[3],
                    s.field, s.mask, s.eta};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (c->mode == 2 && s.partials) cudaFree(s.partials);
    if (s.psum) cudaFree(s.psum);
  }
  c->sl.clear();
  void* ptrs[] = {c->tw, c->khat, c->cav, c->partials, c->psums, c->maxbits, c->bad, c->nonfinite, c->io, c->trace,
                  c->thstep};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->comm) nccl_api()->commDestroy(c->comm);
  c->comm = nullptr;
  if (c->own) cudaStreamDestroy(c->own);
  if (c->cap) cudaStreamDestroy(c->cap);
  if (c->side) cudaStreamDestroy(c->side);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
}

// TMA descriptor of Y[3][nz][Ly][P] viewed as a 3D tensor (P, Ly, 3 nz) of 8-byte elements;
// box (C, 1, nz) = one component's z column block of a K-Z tile (single slab only).
void make_slab_maps(mcq_ctx* c);

void make_y_tensor_map(mcq_ctx* c) {
  c->have_tmz = false;
  if (c->NS != 1) {
    make_slab_maps(c);
    return;
  }
  const Dims& d = c->sl[0].d;
  if (d.nz < 2 || d.nz > 256 || !c->sl[0].Y) return;
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
  const CUresult r = enc(&c->tmz, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->sl[0].Y, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  c->have_tmz = (r == CUDA_SUCCESS);
  const cuuint32_t box2[3] = {(cuuint32_t)zconv2_box_c(d.Lz), 1, (cuuint32_t)d.nz};
  c->have_tmz2 = false;
  if (box2[0] > 0 && d.nz <= 256) {
    const cuuint32_t box3[3] = {16, 1, (cuuint32_t)d.nz};
    const CUresult r2 = enc(&c->tmz2[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->sl[0].Y, dims, strides, box2, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const CUresult r3 = enc(&c->tmz2[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->sl[0].Y, dims, strides, box3, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    // Khat [kz][ky][kpitch][6] fp32 as (6 kpitch, Ly/2 + 1, Lz/2 + 1), box (96, 1, 129)
    const cuuint64_t kd[3] = {(cuuint64_t)6 * d.kpitch, (cuuint64_t)d.Ly / 2 + 1, (cuuint64_t)d.Lz / 2 + 1};
    const cuuint64_t ks[2] = {(cuuint64_t)6 * d.kpitch * 4, (cuuint64_t)6 * d.kpitch * 4 * (d.Ly / 2 + 1)};
    const cuuint32_t kb[3] = {96, 1, 129};
    CUresult rk = CUDA_ERROR_INVALID_VALUE;
    if ((d.Lz == 512 || d.Lz == 256) && c->khat && d.kpitch % 2 == 0)
      rk = enc(&c->tmz2[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->khat, kd, ks, kb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rk != CUDA_SUCCESS) memset(&c->tmz2[2], 0, sizeof(CUtensorMap));
    c->have_tmz2 = (r2 == CUDA_SUCCESS && r3 == CUDA_SUCCESS);
    c->have_tmk = (rk == CUDA_SUCCESS);
  }
}

// z slabs (K-Z v3, SPLIT): per slab, the received blocks R[q][g][zl][ky][KXS] as a 4D tensor
// (KXS, Ly, nzl, 3 NS); box (16, 1, nzl, 3 NS - 2) with element stride 3 along the last dimension
// picks component g of every source rank q, so the box lands as [z][c].  And the slab's Khat.
void make_slab_maps(mcq_ctx* c) {
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
  for (auto& sl : c->sl) {
    sl.have_tm3 = false;
    const Dims& d = sl.d;
    memset(sl.tm3, 0, sizeof(sl.tm3));
    // (a box wider than the tensor — KXS < 16 on small slabs — faulted on the device with an
    // illegal-instruction error: such slabs keep K-Z v2)
    if (!sl.R || !c->khat || (d.Lz != 512 && d.Lz != 256) || d.nzg > d.Lz / 2 || d.kpitch % 2 || c->NS > 85 ||
        d.KXS < 16 || 6 * d.kpitch < 96)
      continue;
    const cuuint64_t dims[4] = {(cuuint64_t)d.KXS, (cuuint64_t)d.Ly, (cuuint64_t)d.nz, (cuuint64_t)3 * c->NS};
    const cuuint64_t strides[3] = {(cuuint64_t)d.KXS * 8, (cuuint64_t)d.Ly * d.KXS * 8,
                                   (cuuint64_t)d.nz * d.Ly * d.KXS * 8};
    const cuuint32_t box[4] = {16, 1, (cuuint32_t)d.nz, (cuuint32_t)(3 * c->NS - 2)};
    const cuuint32_t es[4] = {1, 1, 1, 3};
    const CUresult r = enc(&sl.tm3[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, sl.R, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const cuuint64_t kd[3] = {(cuuint64_t)6 * d.kpitch, (cuuint64_t)d.Ly / 2 + 1, (cuuint64_t)d.Lz / 2 + 1};
    const cuuint64_t ks[2] = {(cuuint64_t)6 * d.kpitch * 4, (cuuint64_t)6 * d.kpitch * 4 * (d.Ly / 2 + 1)};
    const cuuint32_t kb[3] = {96, 1, 129};
    const cuuint32_t kes[3] = {1, 1, 1};
    const CUresult rk = enc(&sl.tm3[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->khat, kd, ks, kb, kes,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    sl.have_tm3 = (r == CUDA_SUCCESS && rk == CUDA_SUCCESS);
  }
}

int alloc_slab(mcq_ctx* c, Slab& s) {
  const Dims& d = s.d;
  const size_t st = 3ULL * d.cs;
  const size_t nX = 3ULL * d.nz * d.ny * d.P;
  const size_t nY = d.nzg > 1 ? (size_t)d.NS * 3 * d.nz * d.Ly * d.KXS : 0;
  bool ok = cudaMalloc(&s.mN, st * 4) == cudaSuccess && cudaMalloc(&s.mA, st * 4) == cudaSuccess &&
            cudaMalloc(&s.mB, st * 4) == cudaSuccess && cudaMalloc(&s.acc, st * 4) == cudaSuccess &&
            cudaMalloc(&s.X, nX * 8) == cudaSuccess && (nY == 0 || cudaMalloc(&s.Y, nY * 8) == cudaSuccess) &&
            (nY == 0 || d.NS == 1 || cudaMalloc(&s.R, nY * 8) == cudaSuccess);
  if (!ok) {
    cudaGetLastError();
    return fail(c, MCQ_ENOMEM, "slab buffers");
  }
  // zero everything once (halo planes at the global boundary and padding columns stay finite)
  CK(c, cudaMemsetAsync(s.mN, 0, st * 4, c->stream));
  CK(c, cudaMemsetAsync(s.mA, 0, st * 4, c->stream));
  CK(c, cudaMemsetAsync(s.mB, 0, st * 4, c->stream));
  CK(c, cudaMemsetAsync(s.acc, 0, st * 4, c->stream));
  CK(c, cudaMemsetAsync(s.X, 0, nX * 8, c->stream));
  if (nY) CK(c, cudaMemsetAsync(s.Y, 0, nY * 8, c->stream));
  if (s.R) CK(c, cudaMemsetAsync(s.R, 0, nY * 8, c->stream));
  return MCQ_OK;
}

std::once_flag g_cfg_once;

// NCCL mode: map the z-neighbour ranks' state buffers (mN, mA, mB) into this process with CUDA IPC
// (handles all-gathered over the context's communicator) so K-U can store its boundary planes
// straight into their halo planes over NVLink.  Any failure leaves the NCCL halos in place.
int setup_peer_halos(mcq_ctx* c) {
  Nccl* n = nccl_api();
  if (!n) return MCQ_ENCCL;
  Slab& sl = c->sl[0];
  cudaIpcMemHandle_t mine[3];
  float* bufs[3] = {sl.mN, sl.mA, sl.mB};
  for (int r = 0; r < 3; ++r)
    if (cudaIpcGetMemHandle(&mine[r], bufs[r]) != cudaSuccess) {
      cudaGetLastError();
      return MCQ_ECUDA;
    }
  const size_t hb = sizeof(mine);
  char* d = nullptr;
  if (cudaMalloc(&d, hb * (c->NS + 1)) != cudaSuccess) return MCQ_ENOMEM;
  std::vector<cudaIpcMemHandle_t> all(3 * c->NS);
  int rc = MCQ_OK;
  if (cudaMemcpyAsync(d, mine, hb, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
      n->allGather(d, d + hb, hb, ncclChar, c->comm, c->stream) != ncclSuccess ||
      cudaMemcpyAsync(all.data(), d + hb, hb * c->NS, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    rc = MCQ_ENCCL;
  cudaFree(d);
  if (rc != MCQ_OK) return rc;
  for (int side = 0; side < 2; ++side) {
    const int peer = c->rank + (side == 0 ? -1 : 1);
    if (peer < 0 || peer >= c->NS) continue;
    for (int r = 0; r < 3; ++r) {
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, all[3 * peer + r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return MCQ_ECUDA;
      }
      (side == 0 ? c->peer_lo : c->peer_hi)[r] = static_cast<float*>(p);
    }
  }
  return MCQ_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int mcq_nccl_get_unique_id(unsigned char out[128]) {
  if (!out) return MCQ_EINVAL;
  Nccl* n = nccl_api();
  if (!n) return MCQ_ENCCL;
  ncclUniqueId id;
  if (n->getUniqueId(&id) != ncclSuccess) return MCQ_ENCCL;
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
  std::memcpy(out, id.internal, 128);
  return MCQ_OK;
}

int mcq_create(mcq_ctx** out, const int grid[3], const double cell[3], double Ms, double Aex, double alpha,
               const mcq_aniso* K, const mcq_dist* dist) {
  if (!out || !grid || !cell) return MCQ_EINVAL;
  *out = nullptr;
  if (grid[0] < 2 || grid[1] < 2 || grid[2] < 1 || grid[0] > 512 || grid[1] > 512 || grid[2] > 512) return MCQ_EINVAL;
  if (!(cell[0] > 0 && cell[1] > 0 && cell[2] > 0)) return MCQ_EINVAL;
  if (!(Ms > 0) || !(Aex >= 0) || !(alpha >= 0)) return MCQ_EINVAL;
  const int world = dist ? dist->world : 1;
  if (world < 1 || world > 64 || grid[2] % world || (world > 1 && grid[2] / world < 1)) return MCQ_EINVAL;
  if (world > 1 && dist->rank >= 0 && (dist->rank >= world || !dist->nccl_id)) return MCQ_EINVAL;
  mcq_ctx* c = new (std::nothrow) mcq_ctx();
  if (!c) return MCQ_ENOMEM;
  c->dx = cell[0];
  c->dy = cell[1];
  c->dz = cell[2];
  c->Ms = Ms;
  c->Aex = Aex;
  c->alpha = alpha;
  if (K) c->K = *K;
  c->NS = world;
  c->mode = world == 1 ? 0 : (dist->rank < 0 ? 1 : 2);
  c->rank = c->mode == 2 ? dist->rank : 0;
  Dims& g = c->dg;
  g.nx = grid[0];
  g.ny = grid[1];
  g.nz = grid[2];
  g.Lx = padded(g.nx);
  g.Ly = padded(g.ny);
  g.Lz = padded(g.nz);
  g.N2 = g.Lx / 2;
  g.NKX = g.N2 + 1;
  g.P = (g.NKX + 15) / 16 * 16;  // 128-byte aligned spectrum rows: whole-sector column tiles, TMA rows
  g.N = (long long)g.nx * g.ny * g.nz;
  g.nzg = g.nz;
  g.zg0 = 0;
  g.zoff = 0;
  g.cs = g.N;
  c->n_magnetic = g.N;
  g.NS = 1;
  g.KXS = g.P;
  g.kx0 = 0;
  g.kxw = g.NKX;
  g.KG = 16;
  g.KB = g.NKX / 16;
  g.kpitch = g.P;
  g.kxoff = 0;
  g.pdl = 0;
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
  c->overlap = c->mode == 2;
  if (c->mode != 0) {
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) return bail(MCQ_ECUDA);
    for (auto& e : c->ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return bail(MCQ_ECUDA);
  }
  c->stream = (dist && dist->cuda_stream) ? (cudaStream_t)dist->cuda_stream : c->own;
  if (c->mode == 2) {
    Nccl* n = nccl_api();
    if (!n) {
      c->err = "libnccl.so.2 not found";
      return bail(MCQ_ENCCL);
    }
    ncclUniqueId id;
    std::memcpy(id.internal, dist->nccl_id, 128);
    if (n->commInitRank(&c->comm, world, id, c->rank) != ncclSuccess) return bail(MCQ_ENCCL);
  }
  // slabs
  const int nzl = g.nz / world;
  // kx split (common.cuh): the largest block KG <= 16 giving every rank at least one block
  int kg = 16;
  while (kg > 1 && g.NKX / kg < world) kg /= 2;
  Dims split = g;
  split.NS = world;
  split.KG = kg;
  split.KB = g.NKX / kg;
  int kxs = 0;
  for (int q = 0; q < world; ++q) kxs = std::max(kxs, kx_first(split, q + 1) - kx_first(split, q));
  kxs = world == 1 ? g.P : (kxs + 3) / 4 * 4;  // 32-byte rows
  const int first = c->mode == 2 ? c->rank : 0, count = c->mode == 1 ? world : 1;
  c->sl.resize(count);
  Dims probe = g;
  probe.nz = nzl;
  c->nparts = update_grid_blocks(probe) * world;
  for (int i = 0; i < count; ++i) {
    Slab& s = c->sl[i];
    const int r = first + i;
    s.d = g;
    s.d.nz = nzl;
    s.d.N = (long long)g.nx * g.ny * nzl;
    s.d.zg0 = r * nzl;
    s.d.zoff = world > 1 ? 1 : 0;
    s.d.cs = (long long)g.nx * g.ny * (nzl + 2 * s.d.zoff);
    s.d.NS = world;
    s.d.KXS = kxs;
    s.d.KG = split.KG;
    s.d.KB = split.KB;
    s.d.kx0 = kx_first(split, r);
    s.d.kxw = kx_first(split, r + 1) - s.d.kx0;
    if (c->mode == 2) {  // Khat sharded to this rank's kx slab (even pitch: 16-byte Khat rows)
      s.d.kxoff = s.d.kx0;
      s.d.kpitch = std::max(2, (s.d.kxw + 1) & ~1);
    }
    s.d.pdl = (c->mode == 0 && g.N <= kPdlMaxCells) ? 1 : 0;  // see common.cuh
    s.nparts = update_grid_blocks(s.d);
    if (alloc_slab(c, s) != MCQ_OK) return bail(MCQ_ENOMEM);
  }
  const size_t nkhat = 6ULL * (g.Lz / 2 + 1) * (g.Ly / 2 + 1) * c->sl[0].d.kpitch;
  bool ok = cudaMalloc(&c->khat, nkhat * 4) == cudaSuccess &&
            cudaMalloc(&c->tw, kTwMax * 8) == cudaSuccess && cudaMalloc(&c->cav, sizeof(CavState)) == cudaSuccess &&
            cudaMalloc(&c->partials, (size_t)(c->mode == 2 ? 1 : c->nparts) * kNPart * 8) == cudaSuccess &&
            cudaMalloc(&c->psums, (size_t)g.nz * kNPart * 8) == cudaSuccess &&
            cudaMalloc(&c->maxbits, 4) == cudaSuccess && cudaMalloc(&c->bad, 4) == cudaSuccess &&
            cudaMalloc(&c->nonfinite, 4) == cudaSuccess && cudaMalloc(&c->thstep, 8) == cudaSuccess &&
            cudaMalloc(&c->io, 3ULL * c->cells_here() * 4) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return bail(MCQ_ENOMEM);
  }
  for (int i = 0; i < count; ++i) {
    Slab& s = c->sl[i];
    if (c->mode == 2) {
      if (cudaMalloc(&s.partials, (size_t)s.nparts * kNPart * 8) != cudaSuccess ||
          cudaMalloc(&s.psum, (size_t)s.d.nz * kNPart * 8) != cudaSuccess)
        return bail(MCQ_ENOMEM);
      cudaMemsetAsync(s.partials, 0, (size_t)s.nparts * kNPart * 8, c->stream);
      cudaMemsetAsync(s.psum, 0, (size_t)s.d.nz * kNPart * 8, c->stream);
    } else {
      s.partials = c->partials + (size_t)i * s.nparts * kNPart;  // global z order = slab order
    }
  }
  if (cudaMemsetAsync(c->khat, 0, nkhat * 4, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->partials, 0, (size_t)(c->mode == 2 ? 1 : c->nparts) * kNPart * 8, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->psums, 0, (size_t)g.nz * kNPart * 8, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->maxbits, 0, 4, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->nonfinite, 0, 4, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->thstep, 0, 8, c->stream) != cudaSuccess)
    return bail(MCQ_ECUDA);
  // twiddles w_1024^m = exp(-2 pi i m / 1024), generated in fp64
  {
    std::vector<float2> h(kTwMax);
    for (int m = 0; m < kTwMax; ++m) {
      const double ang = 2.0 * M_PI * m / kTwMax;
      h[m] = make_float2((float)std::cos(ang), (float)-std::sin(ang));
    }
    if (cudaMemcpyAsync(c->tw, h.data(), kTwMax * 8, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
      return bail(MCQ_ECUDA);
  }
  if (build_khat(c, nullptr) != MCQ_OK) return bail(MCQ_ECUDA);
  make_y_tensor_map(c);
  {
    static const char* hv = getenv("MCQ_HALO");  // "copy": copy / NCCL halos (comparison)
    const bool want = !(hv && !strcmp(hv, "copy"));
    if (c->mode == 1) c->remote_halo = want;
    if (c->mode == 2 && want) c->remote_halo = setup_peer_halos(c) == MCQ_OK;
  }
  if (c->mode == 2) {
    // one eager round of every exchange (on zeroed buffers): NCCL sets up its peer connections
    // here, outside any graph capture
    Enq q{c, c->stream};
    q.halo(0);
    if (g.nz > 1) {
      q.alltoall(true);
      q.alltoall(false);
    }
    q.nk(nccl_api()->allGather(c->sl[0].psum, c->psums, (size_t)c->sl[0].d.nz * kNPart, ncclDouble, c->comm,
                               c->stream));
    q.nk(nccl_api()->allReduce(c->maxbits, c->maxbits, 1, ncclFloat, ncclMax, c->comm, c->stream));
    if (q.rc != MCQ_OK || cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(MCQ_ENCCL);
  }
  if (reset_memory(c) != MCQ_OK) return bail(MCQ_ECUDA);
  *out = c;
  return MCQ_OK;
}

int mcq_set_persistent_2d(mcq_ctx* c, int on) {
  if (!c) return MCQ_EINVAL;
  c->persist2d = on != 0;
  return MCQ_OK;
}

int mcq_set_slab_overlap(mcq_ctx* c, int on) {
  if (!c) return MCQ_EINVAL;
  c->overlap = on != 0;
  invalidate_graphs(c);
  return MCQ_OK;
}

int mcq_set_stream(mcq_ctx* c, void* stream) {
  if (!c) return MCQ_EINVAL;
  CK(c, cudaStreamSynchronize(c->stream));
  c->stream = stream ? (cudaStream_t)stream : c->own;
  return MCQ_OK;
}

// the cells of slab i inside the global host arrays (x fastest): offset and count
static long long slab_cell0(const mcq_ctx* c, int i) { return (long long)c->sl[i].d.zg0 * c->dg.nx * c->dg.ny; }

// After a geometry change on an installed state: every magnetic cell must hold a vector.  Cells
// the new geometry makes magnetic that were vacuum hold m = 0; aos_to_soa counts them in bad.
// Then the state is unusable until mcq_set_m: mark it and report ESTATE.
static int remask_state(mcq_ctx* c) {
  CK(c, cudaMemsetAsync(c->bad, 0, 4, c->stream));
  for (int i = 0; i < (int)c->sl.size(); ++i) {
    Slab& s = c->sl[i];
    const long long off = (long long)s.d.zoff * s.d.nx * s.d.ny;
    float* io = c->io + 3 * i * s.d.N;
    launch_soa_to_aos(s.mN, io, s.d.N, s.d.cs, off, c->stream);
    launch_aos_to_soa(io, s.mN, s.mask, s.d.N, s.d.cs, off, c->bad, c->stream);
    c->launches += 2;
  }
  Enq q{c, c->stream};
  q.halo(0);
  q.x0();
  c->launches += q.count;
  int bad = 0;
  CK(c, cudaMemcpyAsync(&bad, c->bad, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (bad) {
    c->m_set = false;
    return fail(c, MCQ_ESTATE, "the new geometry makes " + std::to_string(bad) +
                                   " former vacuum cell(s) magnetic with no magnetisation: call mcq_set_m");
  }
  return MCQ_OK;
}

int mcq_set_geometry(mcq_ctx* c, const unsigned char* mask) {
  if (!c) return MCQ_EINVAL;
  invalidate_graphs(c);  // the trace's mean uses the magnetic cell count
  if (!mask) {
    const bool had = c->have_mask;
    for (auto& s : c->sl) {
      if (s.mask) cudaFree(s.mask);
      s.mask = nullptr;
    }
    c->have_mask = false;
    c->n_magnetic = c->dg.N;
    if (had && c->m_set) return remask_state(c);
    return MCQ_OK;
  }
  {
    long long nm = 0;
    for (long long i = 0; i < c->dg.N; ++i) nm += mask[i] != 0;
    c->n_magnetic = nm;
  }
  for (int i = 0; i < (int)c->sl.size(); ++i) {
    Slab& s = c->sl[i];
    if (!s.mask) CK(c, cudaMalloc(&s.mask, s.d.N));
    CK(c, cudaMemcpyAsync(s.mask, mask + slab_cell0(c, i), s.d.N, cudaMemcpyHostToDevice, c->stream));
  }
  CK(c, cudaStreamSynchronize(c->stream));
  c->have_mask = true;
  if (c->m_set) return remask_state(c);  // zero m in vacuum now; new magnetic cells need a state
  return MCQ_OK;
}

// io holds the AoS cells of this context (all slabs in order); convert, validate, commit
static int set_m_from_io(mcq_ctx* c) {
  CK(c, cudaMemsetAsync(c->bad, 0, 4, c->stream));
  for (int i = 0; i < (int)c->sl.size(); ++i) {
    Slab& s = c->sl[i];
    const long long off = (long long)s.d.zoff * s.d.nx * s.d.ny;
    launch_aos_to_soa(c->io + 3 * i * s.d.N, s.mA, s.mask, s.d.N, s.d.cs, off, c->bad, c->stream);
  }
  int bad = 0;
  CK(c, cudaMemcpyAsync(&bad, c->bad, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (bad) return fail(c, MCQ_EINVAL, std::to_string(bad) + " magnetic cells with a zero or non-finite vector");
  for (auto& s : c->sl) CK(c, cudaMemcpyAsync(s.mN, s.mA, 3ULL * s.d.cs * 4, cudaMemcpyDeviceToDevice, c->stream));
  Enq q{c, c->stream};
  q.halo(0);  // a fresh state: its halo planes (later steps keep them current from K-U)
  if (q.rc != MCQ_OK) return q.rc;
  q.x0();
  c->launches += q.count + (long long)c->sl.size();
  CK(c, cudaMemsetAsync(c->nonfinite, 0, 4, c->stream));  // a fresh state clears a divergence
  CK(c, cudaGetLastError());
  c->m_set = true;
  return MCQ_OK;
}

int mcq_set_m(mcq_ctx* c, const float* m) {
  if (!c || !m) return MCQ_EINVAL;
  CK(c, cudaMemcpyAsync(c->io, m + 3 * c->first_cell(), 3ULL * c->cells_here() * 4, cudaMemcpyHostToDevice,
                        c->stream));
  return set_m_from_io(c);
}

int mcq_set_m_device(mcq_ctx* c, const float* d_m) {
  if (!c || !d_m) return MCQ_EINVAL;
  CK(c, cudaMemcpyAsync(c->io, d_m + 3 * c->first_cell(), 3ULL * c->cells_here() * 4, cudaMemcpyDeviceToDevice,
                        c->stream));
  return set_m_from_io(c);
}

int mcq_set_bext(mcq_ctx* c, const double B[3]) {
  if (!c || !B) return MCQ_EINVAL;
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(B[i])) return fail(c, MCQ_EINVAL, "B_ext not finite");
  for (int i = 0; i < 3; ++i) c->bext[i] = B[i];
  invalidate_graphs(c);
  return MCQ_OK;
}

static int valid_mode(mcq_ctx* c, int k) { return k >= 0 && k < c->nmodes; }

int mcq_set_modes(mcq_ctx* c, int nmodes) {
  if (!c) return MCQ_EINVAL;
  if (nmodes < 1 || nmodes > kMaxModes) return fail(c, MCQ_EINVAL, "1 <= nmodes <= MCQ_MAX_MODES");
  CK(c, cudaStreamSynchronize(c->stream));
  for (int k = nmodes; k < kMaxModes; ++k) {  // dropped modes return to their defaults
    for (auto& s : c->sl) {
      if (s.brms[k]) cudaFree(s.brms[k]);
      s.brms[k] = nullptr;
    }
    c->brms_map[k] = c->cav_on[k] = false;
    c->brms_u[k][0] = c->brms_u[k][1] = c->brms_u[k][2] = 0.0;
    c->fc[k] = 1e9;
    c->kappa[k] = c->x0[k] = c->p0[k] = c->exc_amp[k] = c->exc_omega[k] = 0.0;
  }
  c->nmodes = nmodes;
  invalidate_graphs(c);
  return reset_memory(c);
}

int mcq_set_brms_mode(mcq_ctx* c, int k, const float* map, const double uniform[3]) {
  if (!c || (!map && !uniform)) return MCQ_EINVAL;
  if (!valid_mode(c, k)) return fail(c, MCQ_EINVAL, "mode index out of range (mcq_set_modes)");
  const long long Nall = c->dg.N;
  if (map) {
    bool nz = false;
    for (long long i = 0; i < 3 * Nall; ++i) {  // the enable flag is a property of the whole map
      if (!std::isfinite(map[i])) return fail(c, MCQ_EINVAL, "B_rms map not finite");
      nz = nz || map[i] != 0.f;
    }
    CK(c, cudaMemcpyAsync(c->io, map + 3 * c->first_cell(), 3ULL * c->cells_here() * 4, cudaMemcpyHostToDevice,
                          c->stream));
    for (int i = 0; i < (int)c->sl.size(); ++i) {
      Slab& s = c->sl[i];
      if (!s.brms[k]) {
        CK(c, cudaMalloc(&s.brms[k], 3ULL * s.d.cs * 4));
        CK(c, cudaMemsetAsync(s.brms[k], 0, 3ULL * s.d.cs * 4, c->stream));
      }
      launch_deinterleave(c->io + 3 * i * s.d.N, s.brms[k], s.d.N, s.d.cs, (long long)s.d.zoff * s.d.nx * s.d.ny,
                          c->stream);
      c->launches += 1;
    }
    CK(c, cudaStreamSynchronize(c->stream));
    c->brms_u[k][0] = c->brms_u[k][1] = c->brms_u[k][2] = 0.0;
    c->brms_map[k] = true;
    c->cav_on[k] = nz;
  } else {
    for (int i = 0; i < 3; ++i)
      if (!std::isfinite(uniform[i])) return fail(c, MCQ_EINVAL, "B_rms not finite");
    for (auto& s : c->sl) {
      if (s.brms[k]) cudaFree(s.brms[k]);
      s.brms[k] = nullptr;
    }
    c->brms_map[k] = false;
    for (int i = 0; i < 3; ++i) c->brms_u[k][i] = uniform[i];
    c->cav_on[k] = uniform[0] != 0 || uniform[1] != 0 || uniform[2] != 0;
  }
  invalidate_graphs(c);
  return reset_memory(c) == MCQ_OK ? MCQ_OK : MCQ_ECUDA;
}

int mcq_set_brms(mcq_ctx* c, const float* map, const double uniform[3]) {
  return c ? mcq_set_brms_mode(c, 0, map, uniform) : MCQ_EINVAL;
}

int mcq_set_cavity_mode(mcq_ctx* c, int k, double f_c, double kappa, double x0, double p0) {
  if (!c) return MCQ_EINVAL;
  if (!valid_mode(c, k)) return fail(c, MCQ_EINVAL, "mode index out of range (mcq_set_modes)");
  if (!(f_c > 0) || !(kappa >= 0) || !std::isfinite(x0) || !std::isfinite(p0))
    return fail(c, MCQ_EINVAL, "f_c must be > 0, kappa >= 0");
  c->fc[k] = f_c;
  c->kappa[k] = kappa;
  c->x0[k] = x0;
  c->p0[k] = p0;
  invalidate_graphs(c);
  return reset_memory(c);
}

int mcq_set_cavity(mcq_ctx* c, double f_c, double kappa, double x0, double p0) {
  return c ? mcq_set_cavity_mode(c, 0, f_c, kappa, x0, p0) : MCQ_EINVAL;
}

int mcq_set_temperature(mcq_ctx* c, double T, unsigned long long seed) {
  if (!c || !std::isfinite(T) || T < 0) return MCQ_EINVAL;
  CK(c, cudaMemsetAsync(c->thstep, 0, 8, c->stream));  // a new stream starts at noise step 0
  c->temperature = T;
  c->th_seed = seed;
  invalidate_graphs(c);
  return MCQ_OK;
}

int mcq_get_thermal_step(mcq_ctx* c, long long* n) {
  if (!c || !n) return MCQ_EINVAL;
  CK(c, cudaMemcpyAsync(n, c->thstep, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int mcq_set_thermal_step(mcq_ctx* c, long long n) {
  if (!c || n < 0) return MCQ_EINVAL;
  static long long h;  // pageable source: synchronise before it can change
  h = n;
  CK(c, cudaMemcpyAsync(c->thstep, &h, 8, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int mcq_set_dmi(mcq_ctx* c, double D) {
  if (!c || !std::isfinite(D)) return MCQ_EINVAL;
  c->dmi = D;
  invalidate_graphs(c);
  return MCQ_OK;
}

int mcq_set_excitation_mode(mcq_ctx* c, int k, double amplitude, double omega_cut) {
  if (!c || !std::isfinite(amplitude) || !std::isfinite(omega_cut)) return MCQ_EINVAL;
  if (!valid_mode(c, k)) return fail(c, MCQ_EINVAL, "mode index out of range (mcq_set_modes)");
  c->exc_amp[k] = amplitude;
  c->exc_omega[k] = omega_cut;
  invalidate_graphs(c);
  return MCQ_OK;
}

int mcq_set_excitation(mcq_ctx* c, double amplitude, double omega_cut) {
  return c ? mcq_set_excitation_mode(c, 0, amplitude, omega_cut) : MCQ_EINVAL;
}

int mcq_reset_memory(mcq_ctx* c) {
  if (!c) return MCQ_EINVAL;
  return reset_memory(c);
}

int mcq_run(mcq_ctx* c, double dt, long long steps) {
  if (!c) return MCQ_EINVAL;
  NvtxRange nv("mcq_run");
  if (!(dt > 0) || steps < 0) return fail(c, MCQ_EINVAL, "dt must be > 0 and steps >= 0");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "mcq_run before mcq_set_m");
  if (steps == 0) return MCQ_OK;
  c->th_dt = dt;
  if (c->temperature > 0)
    for (auto& s : c->sl)
      if (!s.eta) CK(c, cudaMalloc(&s.eta, 3ULL * s.d.cs * sizeof(float)));
  const CavParams p = cav_params(c, dt);
  launch_cav_prepare(p, c->cav, c->stream);
  c->launches += 1;
  // nz == 1 grids of a few thousand cells (configs[0]): one persistent cooperative kernel per
  // call instead of 9 graph nodes per step (update.cu, K-P2D); same arithmetic, same bits
  static const char* pv = getenv("MCQ_PERSIST2D");  // "0": the graph path (comparison)
  if (c->persist2d && c->mode == 0 && c->dg.nz == 1 && c->dg.N <= (1 << 16) && c->nmodes == 1 && c->dmi == 0 &&
      c->temperature <= 0 && !(pv && pv[0] == '0')) {
    Enq q{c, c->stream};
    UpdateArgs u[4];
    for (int st = 1; st <= 4; ++st) u[st - 1] = q.stage_args(0, st, dt, MODE_LLG, MCQ_TERM_ALL);
    bool ok = true;
    for (long long done = 0; done < steps && ok;) {
      const int k = (int)std::min<long long>(steps - done, 1 << 20);
      ok = launch_persist2d(u, p, c->cav, c->khat, k, c->tw, c->stream) == 0;
      if (ok) {
        done += k;
        c->launches += 1;
      } else if (done > 0) {
        return fail(c, MCQ_ECUDA, "persistent 2D launch failed mid-run");
      }
    }
    if (ok) return MCQ_OK;
    cudaGetLastError();  // no instance for this grid / no co-residency: the graph path below
  }
  int rc;
  if (steps >= kGraphSteps && (rc = capture(c, 1, dt, kGraphSteps)) != MCQ_OK) return rc;
  if (steps % kGraphSteps && (rc = capture(c, 0, dt, 1)) != MCQ_OK) return rc;
  for (long long i = 0; i < steps / kGraphSteps; ++i) CK(c, cudaGraphLaunch(c->g[1], c->stream));
  for (long long i = 0; i < steps % kGraphSteps; ++i) CK(c, cudaGraphLaunch(c->g[0], c->stream));
  c->launches += (steps / kGraphSteps) * c->g_launches[1] + (steps % kGraphSteps) * c->g_launches[0];
  return MCQ_OK;
}

int mcq_relax(mcq_ctx* c, double dt, double tol, long long max_steps, long long* taken) {
  if (!c) return MCQ_EINVAL;
  NvtxRange nv("mcq_relax");
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
    c->launches += k == kRelaxCheck ? c->g_launches[3] : k * c->g_launches[2];
    done += k;
    CK(c, cudaMemsetAsync(c->maxbits, 0, 4, c->stream));
    Enq q{c, c->stream};
    q.eval(MODE_MAXTORQUE, MCQ_TERM_ALL & ~(MCQ_TERM_CAVITY | MCQ_TERM_EXCITATION));
    if (q.rc != MCQ_OK) return q.rc;
    c->launches += q.count;
    if (c->mode == 2)  // max over ranks (non-negative floats: the float order is the bit order)
      NK(c, nccl_api()->allReduce(c->maxbits, c->maxbits, 1, ncclFloat, ncclMax, c->comm, c->stream));
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

static int ensure_dp(mcq_ctx* c) {
  for (auto& s : c->sl)
    if (!s.K) {
      CK(c, cudaMalloc(&s.K, 6ULL * 3 * s.d.cs * sizeof(float)));
      CK(c, cudaMemsetAsync(s.K, 0, 6ULL * 3 * s.d.cs * sizeof(float), c->stream));
    }
  return MCQ_OK;
}

int mcq_run_dp(mcq_ctx* c, double dt, long long steps) {
  if (!c) return MCQ_EINVAL;
  NvtxRange nv("mcq_run_dp");
  if (!(dt > 0) || steps < 0) return fail(c, MCQ_EINVAL, "dt must be > 0 and steps >= 0");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "mcq_run_dp before mcq_set_m");
  if (c->temperature > 0) return fail(c, MCQ_ESTATE, "the thermal field is defined for mcq_run (RK4) only");
  int rc = ensure_dp(c);
  if (rc != MCQ_OK) return rc;
  if (steps == 0) return MCQ_OK;
  // stage factors at the DP nodes for this dt; every step's cavity kernel renews them
  launch_cav_prepare(cav_params(c, dt, true), c->cav, c->stream);
  c->launches += 1;
  if (steps >= kGraphSteps && (rc = capture(c, 5, dt, kGraphSteps)) != MCQ_OK) return rc;
  if (steps % kGraphSteps && (rc = capture(c, 4, dt, 1)) != MCQ_OK) return rc;
  for (long long i = 0; i < steps / kGraphSteps; ++i) CK(c, cudaGraphLaunch(c->g[5], c->stream));
  for (long long i = 0; i < steps % kGraphSteps; ++i) CK(c, cudaGraphLaunch(c->g[4], c->stream));
  c->launches += (steps / kGraphSteps) * c->g_launches[5] + (steps % kGraphSteps) * c->g_launches[4];
  CK(c, cudaGetLastError());
  return MCQ_OK;
}

int mcq_run_adaptive(mcq_ctx* c, double duration, double dt0, double tol, long long max_attempts,
                     long long* accepted, long long* rejected, double* dt_next) {
  if (!c) return MCQ_EINVAL;
  NvtxRange nv("mcq_run_adaptive");
  if (!(duration >= 0) || !(dt0 > 0) || !(tol > 0) || max_attempts < 0)
    return fail(c, MCQ_EINVAL, "adaptive: duration >= 0, dt0 > 0, tol > 0, max_attempts >= 0");
  if (c->temperature > 0) return fail(c, MCQ_ESTATE, "the thermal field is defined for mcq_run (RK4) only");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "mcq_run_adaptive before mcq_set_m");
  int rc = ensure_dp(c);
  if (rc != MCQ_OK) return rc;
  CavState h{};
  if ((rc = read_cav_state(c, h)) != MCQ_OK) return rc;
  const double t_end = h.t + duration;
  double t = h.t, dt = dt0;
  long long acc = 0, rej = 0;
  Enq q{c, c->stream};
  while (t_end - t > 1e-12 * std::max(duration, 1e-30) && acc + rej < max_attempts) {
    const double step = std::min(dt, t_end - t);
    launch_cav_prepare(cav_params(c, step, true), c->cav, c->stream);
    q.dp_attempt(step);
    if (q.rc != MCQ_OK) return q.rc;
    unsigned bits = 0;
    CK(c, cudaMemcpyAsync(&bits, c->maxbits, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    float err;
    std::memcpy(&err, &bits, 4);
    if (!std::isfinite(err)) return fail(c, MCQ_ECUDA, "non-finite error estimate");
    if ((double)err <= tol) {  // accept: state and memory advance by this step
      q.dp_commit(step);
      t += step;
      ++acc;
    } else {  // reject: m_n untouched; restore its spectrum
      q.x0();
      ++rej;
    }
    if (q.rc != MCQ_OK) return q.rc;
    // controller (reading C-DP): safety 0.9, growth in [0.2, 5]
    dt = err > 0 ? step * std::min(5.0, std::max(0.2, 0.9 * std::pow(tol / (double)err, 0.2))) : step * 5.0;
  }
  c->launches += q.count + acc + rej;
  if (accepted) *accepted = acc;
  if (rejected) *rejected = rej;
  if (dt_next) *dt_next = dt;
  CK(c, cudaGetLastError());
  return MCQ_OK;
}

int mcq_synchronize(mcq_ctx* c) {
  if (!c) return MCQ_EINVAL;
  int nf = 0;  // stream-ordered read (no legacy-stream sync with the caller's other work)
  CK(c, cudaMemcpyAsync(&nf, c->nonfinite, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  CK(c, cudaGetLastError());
  if (nf) return fail(c, MCQ_ESTATE, "the integration diverged: a non-finite magnetisation was produced (time step too large?); install a fresh state (mcq_set_m, mcq_reset_memory)");
  return MCQ_OK;
}

// SoA slab contents -> io (AoS, slab order)
static void slabs_to_io(mcq_ctx* c, bool field) {
  for (int i = 0; i < (int)c->sl.size(); ++i) {
    Slab& s = c->sl[i];
    launch_soa_to_aos(field ? s.field : s.mN, c->io + 3 * i * s.d.N, s.d.N, s.d.cs,
                      (long long)s.d.zoff * s.d.nx * s.d.ny, c->stream);
  }
  c->launches += (long long)c->sl.size();
}

int mcq_get_m(mcq_ctx* c, float* m_out) {
  if (!c || !m_out) return MCQ_EINVAL;
  slabs_to_io(c, false);
  CK(c, cudaMemcpyAsync(m_out + 3 * c->first_cell(), c->io, 3ULL * c->cells_here() * 4, cudaMemcpyDeviceToHost,
                        c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int mcq_get_m_device(mcq_ctx* c, float* d_out) {
  if (!c || !d_out) return MCQ_EINVAL;
  slabs_to_io(c, false);
  CK(c, cudaMemcpyAsync(d_out + 3 * c->first_cell(), c->io, 3ULL * c->cells_here() * 4, cudaMemcpyDeviceToDevice,
                        c->stream));
  CK(c, cudaGetLastError());
  return MCQ_OK;
}

int mcq_get_field(mcq_ctx* c, float* b_out, unsigned terms) {
  if (!c || !b_out) return MCQ_EINVAL;
  NvtxRange nv("mcq_get_field");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "mcq_get_field before mcq_set_m");
  if ((terms & MCQ_TERM_THERM) && c->temperature > 0 && !(c->th_dt > 0))
    return fail(c, MCQ_ESTATE, "thermal field before any mcq_run (its scale needs the run's dt)");
  for (auto& s : c->sl) {
    if (!s.field) {
      CK(c, cudaMalloc(&s.field, 3ULL * s.d.cs * 4));
      CK(c, cudaMemsetAsync(s.field, 0, 3ULL * s.d.cs * 4, c->stream));
    }
  }
  const CavParams p = cav_params(c, 1e-12);
  launch_cav_prepare(p, c->cav, c->stream);
  Enq q{c, c->stream};
  q.eval(MODE_FIELD, terms & (MCQ_TERM_ALL | MCQ_TERM_THERM));
  if (q.rc != MCQ_OK) return q.rc;
  c->launches += q.count + 1;
  slabs_to_io(c, true);
  CK(c, cudaMemcpyAsync(b_out + 3 * c->first_cell(), c->io, 3ULL * c->cells_here() * 4, cudaMemcpyDeviceToHost,
                        c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return MCQ_OK;
}

int mcq_get_cavity_mode(mcq_ctx* c, int k, mcq_cavity_state* out) {
  if (!c || !out) return MCQ_EINVAL;
  if (!valid_mode(c, k)) return fail(c, MCQ_EINVAL, "mode index out of range (mcq_set_modes)");
  CavState h{};
  int rc = read_cav_state(c, h);
  if (rc != MCQ_OK) return rc;
  const double re = h.re[k], im = h.im[k];
  out->t = h.t;
  out->re_alpha = re;
  out->im_alpha = im;
  out->gamma = 2.0 * re;
  out->W = h.W[k];
  out->n_photon = re * re + im * im;
  out->step = h.step;
  // S - i C = (hbar / V_c)(alpha_0 - e^{(kappa + i w) t} alpha)
  const double w = 2.0 * M_PI * c->fc[k], vc = c->dx * c->dy * c->dz;
  const double g = std::exp(c->kappa[k] * h.t);
  const double er = g * std::cos(w * h.t), ei = g * std::sin(w * h.t);
  const double ar = er * re - ei * im, ai = er * im + ei * re;
  const double dr = 0.5 * c->x0[k] - ar, di = -0.5 * c->p0[k] - ai;
  out->S = kHbar / vc * dr;
  out->C = -kHbar / vc * di;
  // e^{-kappa t}(S - i C) = (hbar/V_c)(e^{-kappa t} alpha_0 - e^{i w t} alpha): no growing factor
  const double dec = std::exp(-c->kappa[k] * h.t);
  const double br = std::cos(w * h.t) * re - std::sin(w * h.t) * im;
  const double bi = std::cos(w * h.t) * im + std::sin(w * h.t) * re;
  out->S_resc = kHbar / vc * (dec * 0.5 * c->x0[k] - br);
  out->C_resc = -kHbar / vc * (-dec * 0.5 * c->p0[k] - bi);
  return MCQ_OK;
}

int mcq_get_cavity(mcq_ctx* c, mcq_cavity_state* out) { return c ? mcq_get_cavity_mode(c, 0, out) : MCQ_EINVAL; }

long long mcq_cavity_state_bytes(void) { return (long long)sizeof(CavState); }

int mcq_set_cavity_state_mode(mcq_ctx* c, int k, const mcq_cavity_state* in) {
  if (!c || !in) return MCQ_EINVAL;
  if (!valid_mode(c, k)) return fail(c, MCQ_EINVAL, "mode index out of range (mcq_set_modes)");
  if (!std::isfinite(in->t) || !std::isfinite(in->re_alpha) || !std::isfinite(in->im_alpha))
    return fail(c, MCQ_EINVAL, "non-finite cavity state");
  CavState h{};
  int rc = read_cav_state(c, h);
  if (rc != MCQ_OK) return rc;
  h.re[k] = in->re_alpha;
  h.im[k] = in->im_alpha;
  h.t = in->t;  // the clock and the step counter are shared by the modes
  h.step = in->step;
  h.trace_rows = 0;
  return write_cav_state(c, h);
}

int mcq_set_cavity_state(mcq_ctx* c, const mcq_cavity_state* in) {
  return c ? mcq_set_cavity_state_mode(c, 0, in) : MCQ_EINVAL;
}

int mcq_cavity_status(const mcq_ctx* c) {
  if (!c) return MCQ_EINVAL;
  for (int k = 0; k < c->nmodes; ++k)
    if (c->cav_on[k]) return 1;
  return 0;
}

int mcq_set_trace(mcq_ctx* c, long long capacity, int every) {
  if (!c) return MCQ_EINVAL;
  if (capacity < 0 || capacity > (1LL << 28) || every < 1) return fail(c, MCQ_EINVAL, "trace: 0 <= capacity <= 2^28, every >= 1");
  CK(c, cudaStreamSynchronize(c->stream));
  if (c->trace) cudaFree(c->trace);
  c->trace = nullptr;
  c->trace_cap = 0;
  if (capacity > 0) {
    CK(c, cudaMalloc(&c->trace, (size_t)capacity * kTraceCols * 8));
    CK(c, cudaMemsetAsync(c->trace, 0, (size_t)capacity * kTraceCols * 8, c->stream));
  }
  c->trace_cap = capacity;
  c->trace_every = every;
  const long long zero = 0;
  CK(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->cav) + offsetof(CavState, trace_rows), &zero, sizeof(zero),
                        cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  invalidate_graphs(c);
  return MCQ_OK;
}

int mcq_get_trace(mcq_ctx* c, double* out, long long max_rows, long long* rows) {
  if (!c || (!out && max_rows > 0) || max_rows < 0) return MCQ_EINVAL;
  CavState h{};
  CK(c, cudaMemcpyAsync(&h, c->cav, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  const long long stored = std::min(h.trace_rows, c->trace_cap);
  const long long n = std::min(stored, max_rows);
  if (n > 0) {
    CK(c, cudaMemcpyAsync(out, c->trace, (size_t)n * kTraceCols * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
  }
  if (rows) *rows = stored;
  return MCQ_OK;
}

long long mcq_kernel_launches(const mcq_ctx* c) { return c ? c->launches : -1; }

// ---------------------------------------------------------------- NEXT-3: device spectroscopy
int mcq_trace_peaks_batch(mcq_ctx** ctxs, int n, int column, int pad, int window, double fmin, int npeaks,
                          double* f_out, double* a_out, int* nfound) {
  if (!ctxs || n < 1 || n > 1024 || column < 1 || column >= kTraceCols || !f_out || !a_out || !nfound)
    return MCQ_EINVAL;
  std::vector<const double*> ptr(n), tptr(n);
  std::vector<long long> rows(n);
  std::vector<int> stride(n, kTraceCols);
  long long nmax = 0;
  for (int b = 0; b < n; ++b) {
    mcq_ctx* c = ctxs[b];
    if (!c) return MCQ_EINVAL;
    if (c->device != ctxs[0]->device) return fail(ctxs[0], MCQ_EINVAL, "traces on different devices");
    CavState h{};
    CK(c, cudaMemcpyAsync(&h, c->cav, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    rows[b] = std::min(h.trace_rows, c->trace_cap);
    if (rows[b] < 3 || !c->trace) return fail(c, MCQ_ESTATE, "fewer than 3 trace rows recorded (mcq_set_trace)");
    ptr[b] = c->trace + column;
    tptr[b] = c->trace;  // column 0: the clock t
    nmax = std::max(nmax, rows[b]);
  }
  mcq_ctx* c0 = ctxs[0];
  void* dmem = nullptr;
  const size_t bytes = (size_t)n * (8 + 8 + 8 + 8 + 4) + 64;
  CK(c0, cudaMalloc(&dmem, bytes));
  char* p = static_cast<char*>(dmem);
  const double** dptr = reinterpret_cast<const double**>(p);
  long long* drows = reinterpret_cast<long long*>(p + 8 * n);
  double* ddt = reinterpret_cast<double*>(p + 16 * n);
  const double** dtp = reinterpret_cast<const double**>(p + 24 * n);
  int* dstride = reinterpret_cast<int*>(p + 32 * n);
  int rc = MCQ_OK;
  if (cudaMemcpyAsync(dptr, ptr.data(), 8 * n, cudaMemcpyHostToDevice, c0->stream) != cudaSuccess ||
      cudaMemcpyAsync(drows, rows.data(), 8 * n, cudaMemcpyHostToDevice, c0->stream) != cudaSuccess ||
      cudaMemcpyAsync(dtp, tptr.data(), 8 * n, cudaMemcpyHostToDevice, c0->stream) != cudaSuccess ||
      cudaMemcpyAsync(dstride, stride.data(), 4 * n, cudaMemcpyHostToDevice, c0->stream) != cudaSuccess) {
    rc = fail(c0, MCQ_ECUDA, "spectrum setup copy");
  } else {
    launch_sp_dt(reinterpret_cast<const double* const*>(dtp), drows, ddt, n, c0->stream);
    rc = spectrum_peaks_device(n, dptr, drows, dstride, ddt, nmax, pad, window, fmin, npeaks, f_out, a_out, nfound,
                               c0->stream);
    if (rc != MCQ_OK) fail(c0, rc, "device spectrum");
  }
  cudaStreamSynchronize(c0->stream);
  cudaFree(dmem);
  return rc;
}

int mcq_trace_peaks(mcq_ctx* c, int column, int pad, int window, double fmin, int npeaks, double* f_out,
                    double* a_out, int* nfound) {
  return c ? mcq_trace_peaks_batch(&c, 1, column, pad, window, fmin, npeaks, f_out, a_out, nfound) : MCQ_EINVAL;
}

int mcq_spectrum_peaks(const double* signal, long long n, double dt, int pad, int window, double fmin, int npeaks,
                       double* f_out, double* a_out, int* nfound) {
  if (!signal || n < 3 || !(dt > 0) || !f_out || !a_out || !nfound) return MCQ_EINVAL;
  double* d = nullptr;
  void* meta = nullptr;
  if (cudaMalloc(&d, (size_t)n * 8) != cudaSuccess || cudaMalloc(&meta, 64) != cudaSuccess) {
    cudaFree(d);
    cudaGetLastError();
    return MCQ_ENOMEM;
  }
  char* p = static_cast<char*>(meta);
  const double* ptr = d;
  const int stride = 1;
  int rc = MCQ_OK;
  if (cudaMemcpy(d, signal, (size_t)n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p, &ptr, 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p + 8, &n, 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p + 16, &dt, 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p + 24, &stride, 4, cudaMemcpyHostToDevice) != cudaSuccess) {
    rc = MCQ_ECUDA;
  } else {
    rc = spectrum_peaks_device(1, reinterpret_cast<const double* const*>(p), reinterpret_cast<const long long*>(p + 8),
                               reinterpret_cast<const int*>(p + 24), reinterpret_cast<const double*>(p + 16), n, pad,
                               window, fmin, npeaks, f_out, a_out, nfound, 0);
  }
  cudaFree(d);
  cudaFree(meta);
  return rc;
}

int mcq_fit_anticrossing(int n, const double* w_mag, const double* lo, const double* hi, double wc0, double g0,
                         double* wc, double* g) {
  if (!w_mag || !lo || !hi || !wc || !g) return MCQ_EINVAL;
  return fit_anticrossing_device(n, w_mag, lo, hi, wc0, g0, wc, g);
}

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
  NvtxRange nv("mcq_profile_run");
  if (!(dt > 0) || steps <= 0) return fail(c, MCQ_EINVAL, "profile: dt > 0, steps > 0");
  if (!c->m_set) return fail(c, MCQ_ESTATE, "profile before set_m");
  const CavParams p = cav_params(c, dt);
  launch_cav_prepare(p, c->cav, c->stream);
  Prof pr{c->stream};
  Enq q{c, c->stream, prof_hook, &pr};
  for (long long i = 0; i < steps; ++i) q.llg_step(dt);
  if (q.rc != MCQ_OK) return q.rc;
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
  out[0] = c->dg.Lx;
  out[1] = c->dg.Ly;
  out[2] = c->dg.Lz;
  out[3] = c->dg.NKX;
  out[4] = c->dg.P;
  out[5] = c->nparts;
  return MCQ_OK;
}

int mcq_debug_tensor_octant(mcq_ctx* c, double* out) {
  if (!c || !out) return MCQ_EINVAL;
  return build_khat(c, out);
}

int mcq_debug_khat(mcq_ctx* c, float* out) {
  if (!c || !out) return MCQ_EINVAL;
  if (c->sl[0].d.kpitch != c->dg.P) return fail(c, MCQ_ESTATE, "Khat is sharded to this rank's kx slab (NCCL mode)");
  const size_t nK = 6ULL * (c->dg.Lz / 2 + 1) * (c->dg.Ly / 2 + 1) * c->dg.P;
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
