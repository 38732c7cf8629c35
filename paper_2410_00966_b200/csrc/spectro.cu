// spectro.cu — on-device spectroscopy: the paper's spectra are "the
// numerical Fourier transform of the resulting time-dependent spatially-averaged magnetization"
// (P:172), and its couplings are read off the anticrossing of such spectra over a bias sweep
// (P:14-22).  Here the whole analysis of recorded traces runs in CUDA, fp64:
//   K-SP1  mean subtraction, optional Hann window, zero padding to L = pow2 >= pad * n;
//   K-SP2  radix-2 Stockham FFT stages (log2 L launches, batched over traces: grid.y);
//   K-SP3  |X_k| on k <= L/2, local maxima at f >= fmin, the npeaks strongest (ties: lower k),
//          each refined by a parabola through log |X| (reading C23), returned in ascending f;
//   K-FIT  least-squares (omega_c, g) of the two position-coupled oscillators' normal modes
//          (P:419 with lambda -> g, the form spectroscopy.normal_modes documents) to the two
//          branches of a sweep: Levenberg-Marquardt in one thread, fp64.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/mcq.h"
#include "common.cuh"

namespace mcq {

constexpr int kSpThreads = 256;
constexpr int kMaxPeaks = 16;

// mean of sig[0..n) (one block per trace, fixed order)
__global__ void k_sp_mean(const double* const* sig, const long long* n_, const int* stride_, double* mean) {
  const int b = blockIdx.x;
  const double* s = sig[b];
  const long long n = n_[b];
  const int st = stride_[b];
  __shared__ double red[kSpThreads];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += kSpThreads) acc += s[i * st];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kSpThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) mean[b] = n > 0 ? red[0] / (double)n : 0.0;
}

// x = (sig - mean) * window into the complex buffer of length L (zero padded)
__global__ void k_sp_prep(const double* const* sig, const long long* n_, const int* stride_, const double* mean_,
                          int window, long long L, double2* x) {
  const int b = blockIdx.y;
  const double* s = sig[b];
  const long long n = n_[b];
  const int st = stride_[b];
  const double mean = mean_[b];
  double2* xb = x + (size_t)b * L;
  for (long long i = blockIdx.x * (long long)kSpThreads + threadIdx.x; i < L; i += (long long)gridDim.x * kSpThreads) {
    double v = 0.0;
    if (i < n) {
      v = s[i * st] - mean;
      if (window == 1 && n > 1) v *= 0.5 - 0.5 * cospi(2.0 * (double)i / (double)(n - 1));  // numpy.hanning
    }
    xb[i] = make_double2(v, 0.0);
  }
}

// one radix-2 Stockham stage (forward, w = e^{-2 pi i / (2 Ns)}): natural order after log2 L
__global__ void k_sp_stage(const double2* __restrict__ in, double2* __restrict__ out, long long L, long long Ns) {
  const int b = blockIdx.y;
  const double2* ib = in + (size_t)b * L;
  double2* ob = out + (size_t)b * L;
  const long long h = L / 2;
  for (long long j = blockIdx.x * (long long)kSpThreads + threadIdx.x; j < h; j += (long long)gridDim.x * kSpThreads) {
    const long long k = j % Ns;
    double s, c;
    sincospi(-(double)k / (double)Ns, &s, &c);
    const double2 a = ib[j], v = ib[j + h];
    const double2 w = make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
    const long long o = (j - k) * 2 + k;
    ob[o] = make_double2(a.x + w.x, a.y + w.y);
    ob[o + Ns] = make_double2(a.x - w.x, a.y - w.y);
  }
}

// peaks of |X| (one block per trace)
__global__ void k_sp_peaks(const double2* __restrict__ X, long long L, const double* dt_, double fmin, int npeaks,
                           double* fout, double* aout, int* nfound) {
  const int b = blockIdx.x;
  const double2* xb = X + (size_t)b * L;
  const double df = 1.0 / ((double)L * dt_[b]);
  const long long kmax = L / 2;
  // per-thread top-npeaks (amplitude descending, ties: lower k first)
  double ta[kMaxPeaks];
  long long tk[kMaxPeaks];
  for (int i = 0; i < npeaks; ++i) {
    ta[i] = -1.0;
    tk[i] = -1;
  }
  auto amp = [&](long long k) { return hypot(xb[k].x, xb[k].y); };
  for (long long k = 1 + threadIdx.x; k < kmax; k += kSpThreads) {
    if ((double)k * df < fmin) continue;
    const double a = amp(k);
    if (!(a >= amp(k - 1) && a > amp(k + 1))) continue;
    int pos = npeaks;
    while (pos > 0 && (a > ta[pos - 1] || (a == ta[pos - 1] && k < tk[pos - 1]))) --pos;
    if (pos < npeaks) {
      for (int i = npeaks - 1; i > pos; --i) {
        ta[i] = ta[i - 1];
        tk[i] = tk[i - 1];
      }
      ta[pos] = a;
      tk[pos] = k;
    }
  }
  __shared__ double sa[kSpThreads * 4];
  __shared__ long long sk[kSpThreads * 4];
  // merge in rounds of 4 candidates per thread (npeaks <= 16: up to 4 rounds)
  double ba[kMaxPeaks];
  long long bk[kMaxPeaks];
  for (int i = 0; i < npeaks; ++i) {
    ba[i] = -1.0;
    bk[i] = -1;
  }
  for (int r0 = 0; r0 < npeaks; r0 += 4) {
    for (int i = 0; i < 4; ++i) {
      sa[threadIdx.x * 4 + i] = r0 + i < npeaks ? ta[r0 + i] : -1.0;
      sk[threadIdx.x * 4 + i] = r0 + i < npeaks ? tk[r0 + i] : -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int e = 0; e < kSpThreads * 4; ++e) {
        const double a = sa[e];
        const long long k = sk[e];
        if (k < 0) continue;
        int pos = npeaks;
        while (pos > 0 && (a > ba[pos - 1] || (a == ba[pos - 1] && k < bk[pos - 1]))) --pos;
        if (pos < npeaks) {
          for (int i = npeaks - 1; i > pos; --i) {
            ba[i] = ba[i - 1];
            bk[i] = bk[i - 1];
          }
          ba[pos] = a;
          bk[pos] = k;
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int n = 0;
    double f[kMaxPeaks], am[kMaxPeaks];
    for (int i = 0; i < npeaks; ++i) {
      if (bk[i] < 0) break;
      const long long k = bk[i];
      const double y0 = log(amp(k - 1) + 1e-300), y1 = log(ba[i] + 1e-300), y2 = log(amp(k + 1) + 1e-300);
      const double dd = y0 - 2.0 * y1 + y2;
      const double delta = dd != 0.0 ? 0.5 * (y0 - y2) / dd : 0.0;
      f[n] = ((double)k + delta) * df;
      am[n] = ba[i];
      ++n;
    }
    for (int i = 1; i < n; ++i)  // ascending frequency
      for (int j = i; j > 0 && f[j] < f[j - 1]; --j) {
        const double tf = f[j], ta2 = am[j];
        f[j] = f[j - 1];
        am[j] = am[j - 1];
        f[j - 1] = tf;
        am[j - 1] = ta2;
      }
    for (int i = 0; i < n; ++i) {
      fout[b * npeaks + i] = f[i];
      aout[b * npeaks + i] = am[i];
    }
    nfound[b] = n;
  }
}

// trace dt from the recorded clock (column 0): (t_last - t_0) / (rows - 1)
__global__ void k_sp_dt(const double* const* trace, const long long* rows, double* dt) {
  const int b = threadIdx.x;
  if (b < (int)blockDim.x) {
    const double* tr = trace[b];
    const long long n = rows[b];
    dt[b] = n > 1 ? (tr[(n - 1) * kTraceCols] - tr[0]) / (double)(n - 1) : 1.0;
  }
}

// ---------------------------------------------------------------- two-oscillator fit
__device__ void normal_modes(double w1, double w2, double g, double& lo, double& hi) {
  const double a = w1 * w1 + w2 * w2;
  const double bb = sqrt((w1 * w1 - w2 * w2) * (w1 * w1 - w2 * w2) + 16.0 * g * g * w1 * w2);
  lo = sqrt(fmax(0.5 * (a - bb), 0.0));
  hi = sqrt(0.5 * (a + bb));
}

// Levenberg-Marquardt on q = (omega_c / wc0, g / wc0), residuals r = [lo_model - lo, hi_model - hi] / wc0
__global__ void k_fit(int n, const double* __restrict__ wm, const double* __restrict__ lo, const double* __restrict__ hi,
                      double wc0, double g0, double* out) {
  if (threadIdx.x || blockIdx.x) return;
  double q0 = 1.0, q1 = g0 / wc0, lambda = 1e-3;
  auto cost = [&](double a, double b) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
      double l, h;
      normal_modes(wm[i], a * wc0, b * wc0, l, h);
      const double r0 = (l - lo[i]) / wc0, r1 = (h - hi[i]) / wc0;
      s += r0 * r0 + r1 * r1;
    }
    return s;
  };
  double c = cost(q0, q1);
  for (int it = 0; it < 200; ++it) {
    double JtJ00 = 0, JtJ01 = 0, JtJ11 = 0, Jr0 = 0, Jr1 = 0;
    const double e0 = 1e-7 * fmax(1.0, fabs(q0)), e1 = 1e-7 * fmax(1e-3, fabs(q1));
    for (int i = 0; i < n; ++i) {
      double l, h, la, ha, lb, hb;
      normal_modes(wm[i], q0 * wc0, q1 * wc0, l, h);
      normal_modes(wm[i], (q0 + e0) * wc0, q1 * wc0, la, ha);
      normal_modes(wm[i], q0 * wc0, (q1 + e1) * wc0, lb, hb);
      const double r[2] = {(l - lo[i]) / wc0, (h - hi[i]) / wc0};
      const double j0[2] = {(la - l) / (e0 * wc0), (ha - h) / (e0 * wc0)};
      const double j1[2] = {(lb - l) / (e1 * wc0), (hb - h) / (e1 * wc0)};
      for (int k = 0; k < 2; ++k) {
        JtJ00 += j0[k] * j0[k];
        JtJ01 += j0[k] * j1[k];
        JtJ11 += j1[k] * j1[k];
        Jr0 += j0[k] * r[k];
        Jr1 += j1[k] * r[k];
      }
    }
    bool improved = false;
    for (int tries = 0; tries < 30 && !improved; ++tries) {
      const double a00 = JtJ00 * (1 + lambda), a11 = JtJ11 * (1 + lambda), a01 = JtJ01;
      const double det = a00 * a11 - a01 * a01;
      if (det == 0.0) break;
      const double d0 = -(a11 * Jr0 - a01 * Jr1) / det, d1 = -(a00 * Jr1 - a01 * Jr0) / det;
      const double cn = cost(q0 + d0, q1 + d1);
      if (cn < c) {
        q0 += d0;
        q1 += d1;
        const double rel = (c - cn) / fmax(c, 1e-300);
        c = cn;
        lambda = fmax(lambda * 0.3, 1e-12);
        improved = true;
        if (rel < 1e-15 || (fabs(d0) < 1e-14 && fabs(d1) < 1e-14)) it = 1 << 20;
      } else {
        lambda *= 10.0;
      }
    }
    if (!improved) break;
  }
  out[0] = q0 * wc0;
  out[1] = fabs(q1) * wc0;
}

// ---------------------------------------------------------------- host side
static int pow2_at_least(long long v) {
  int e = 0;
  while ((1LL << e) < v) ++e;
  return e;
}

// peaks of `nb` signals (device pointers, element stride, lengths, device dts), results to host
int spectrum_peaks_device(int nb, const double* const* d_sig, const long long* d_n, const int* d_stride,
                          const double* d_dt, long long nmax, int pad, int window, double fmin, int npeaks,
                          double* f_out, double* a_out, int* nfound, cudaStream_t s) {
  if (nb < 1 || npeaks < 1 || npeaks > kMaxPeaks || pad < 1 || nmax < 3) return MCQ_EINVAL;
  const int e = pow2_at_least(nmax * (long long)pad);
  const long long L = 1LL << e;
  double2 *x = nullptr, *y = nullptr;
  double *df = nullptr, *da = nullptr, *dm = nullptr;
  int* dn = nullptr;
  if (cudaMalloc(&dm, (size_t)nb * 8) != cudaSuccess || cudaMalloc(&x, (size_t)nb * L * sizeof(double2)) != cudaSuccess ||
      cudaMalloc(&y, (size_t)nb * L * sizeof(double2)) != cudaSuccess ||
      cudaMalloc(&df, (size_t)nb * npeaks * 8) != cudaSuccess || cudaMalloc(&da, (size_t)nb * npeaks * 8) != cudaSuccess ||
      cudaMalloc(&dn, (size_t)nb * 4) != cudaSuccess) {
    cudaFree(x);
    cudaFree(y);
    cudaFree(df);
    cudaFree(da);
    cudaFree(dn);
    cudaFree(dm);
    cudaGetLastError();
    return MCQ_ENOMEM;
  }
  long long blocks = (L + kSpThreads - 1) / kSpThreads;
  if (blocks > 4096) blocks = 4096;
  k_sp_mean<<<nb, kSpThreads, 0, s>>>(d_sig, d_n, d_stride, dm);
  k_sp_prep<<<dim3((unsigned)blocks, nb), kSpThreads, 0, s>>>(d_sig, d_n, d_stride, dm, window, L, x);
  long long hb = (L / 2 + kSpThreads - 1) / kSpThreads;
  if (hb > 4096) hb = 4096;
  for (long long Ns = 1; Ns < L; Ns *= 2) {
    k_sp_stage<<<dim3((unsigned)hb, nb), kSpThreads, 0, s>>>(x, y, L, Ns);
    std::swap(x, y);
  }
  k_sp_peaks<<<nb, kSpThreads, 0, s>>>(x, L, d_dt, fmin, npeaks, df, da, dn);
  int rc = MCQ_OK;
  if (cudaMemcpyAsync(f_out, df, (size_t)nb * npeaks * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(a_out, da, (size_t)nb * npeaks * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(nfound, dn, (size_t)nb * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    rc = MCQ_ECUDA;
  cudaFree(x);
  cudaFree(y);
  cudaFree(df);
  cudaFree(da);
  cudaFree(dn);
  cudaFree(dm);
  return rc;
}

int fit_anticrossing_device(int n, const double* w_mag, const double* lo, const double* hi, double wc0, double g0,
                            double* wc, double* g) {
  if (n < 2 || !(wc0 > 0)) return MCQ_EINVAL;
  double* d = nullptr;
  if (cudaMalloc(&d, (3 * (size_t)n + 2) * 8) != cudaSuccess) return MCQ_ENOMEM;
  int rc = MCQ_OK;
  if (cudaMemcpy(d, w_mag, n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d + n, lo, n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d + 2 * n, hi, n * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
    rc = MCQ_ECUDA;
  } else {
    k_fit<<<1, 1>>>(n, d, d + n, d + 2 * n, wc0, g0, d + 3 * n);
    double o[2];
    if (cudaMemcpy(o, d + 3 * n, 16, cudaMemcpyDeviceToHost) != cudaSuccess) {
      rc = MCQ_ECUDA;
    } else {
      *wc = o[0];
      *g = o[1];
    }
  }
  cudaFree(d);
  return rc;
}

void launch_sp_dt(const double* const* d_trace, const long long* d_rows, double* d_dt, int nb, cudaStream_t s) {
  k_sp_dt<<<1, nb, 0, s>>>(d_trace, d_rows, d_dt);
}

}  // namespace mcq
