// tensor.cu — K-TEN: the demagnetising kernel spectrum, computed once per context in fp64.
//
// Definition (reading C11; PAPER.md only names the demag term):
//   N_ab(i dx, j dy, k dz) = Newell's cell-averaged tensor (27-point second difference of f, g)
//                            for max(|i|,|j|,|k|) <= 16;
//                          = the point-dipole tensor (V/4 pi r^3)(I - 3 r^ r^) averaged over the
//                            source and target cells with 3-point Gauss-Legendre per axis, beyond.
//   B_demag,i = -mu0 sum_j N(r_i - r_j) Ms m_j.
// The DFT of the zero-padded cyclic tensor is real (each component is even or odd in every
// axis), so it is evaluated on one octant with per-axis cosine / sine sums:
//   even axis: Nhat(k) = sum_o w_o N(o) cos(2 pi k o / L),  w_0 = 1, w_o = 2 (0 < o < L/2)
//   odd  axis: Nhat(k) = -i sum_o 2 N(o) sin(2 pi k o / L)
// and the two factors of -i of an off-diagonal component give its sign -1.  The stored fp32
// spectrum is Khat = -mu0 Ms / (Lx Ly Lz) Nhat (FFT normalisation and Ms folded in).
#include "common.cuh"

namespace mcq {

__device__ __forceinline__ double asinh_ratio(double num, double den) { return den > 0.0 ? asinh(num / den) : 0.0; }
__device__ __forceinline__ double atan_ratio(double num, double den) { return den != 0.0 ? atan(num / den) : 0.0; }

__device__ double newell_f(double x, double y, double z) {
  const double x2 = x * x, y2 = y * y, z2 = z * z;
  const double R = sqrt(x2 + y2 + z2);
  double v = (2.0 * x2 - y2 - z2) * R / 6.0;
  v += 0.5 * y * (z2 - x2) * asinh_ratio(y, sqrt(x2 + z2));
  v += 0.5 * z * (y2 - x2) * asinh_ratio(z, sqrt(x2 + y2));
  v -= x * y * z * atan_ratio(y * z, x * R);
  return v;
}

__device__ double newell_g(double x, double y, double z) {
  const double x2 = x * x, y2 = y * y, z2 = z * z;
  const double R = sqrt(x2 + y2 + z2);
  double v = -x * y * R / 3.0;
  v += x * y * z * asinh_ratio(z, sqrt(x2 + y2));
  v += y / 6.0 * (3.0 * z2 - y2) * asinh_ratio(x, sqrt(y2 + z2));
  v += x / 6.0 * (3.0 * z2 - x2) * asinh_ratio(y, sqrt(x2 + z2));
  v -= z2 * z / 6.0 * atan_ratio(x * y, z * R);
  v -= z * y2 / 2.0 * atan_ratio(x * z, y * R);
  v -= z * x2 / 2.0 * atan_ratio(y * z, x * R);
  return v;
}

// component c of the Newell tensor at offset (X, Y, Z): second difference with weights
// w_0 = 2, w_+-1 = -1 per axis, / (4 pi dx dy dz)
__device__ void newell6(double X, double Y, double Z, double dx, double dy, double dz, double out[6]) {
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b)
      for (int c = -1; c <= 1; ++c) {
        const double w = (a ? -1.0 : 2.0) * (b ? -1.0 : 2.0) * (c ? -1.0 : 2.0);
        const double x = X + a * dx, y = Y + b * dy, z = Z + c * dz;
        acc[0] += w * newell_f(x, y, z);
        acc[1] += w * newell_f(y, x, z);
        acc[2] += w * newell_f(z, y, x);
        acc[3] += w * newell_g(x, y, z);
        acc[4] += w * newell_g(x, z, y);
        acc[5] += w * newell_g(y, z, x);
      }
  const double pre = 1.0 / (4.0 * 3.14159265358979323846 * dx * dy * dz);
  for (int i = 0; i < 6; ++i) out[i] = pre * acc[i];
}

// 3-point Gauss-Legendre on [-1/2, 1/2] for source and target: the node differences
// {-2a, -a, 0, a, 2a}, a = sqrt(3/5)/2, carry weights {25, 80, 114, 80, 25} / 324.
__device__ void far6(double X, double Y, double Z, double dx, double dy, double dz, double out[6]) {
  const double a = 0.5 * sqrt(0.6);
  const double off[5] = {-2.0 * a, -a, 0.0, a, 2.0 * a};
  const double wt[5] = {25.0 / 324.0, 80.0 / 324.0, 114.0 / 324.0, 80.0 / 324.0, 25.0 / 324.0};
  const double V = dx * dy * dz;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int u = 0; u < 5; ++u)
    for (int v = 0; v < 5; ++v)
      for (int s = 0; s < 5; ++s) {
        const double x = X + off[u] * dx, y = Y + off[v] * dy, z = Z + off[s] * dz;
        const double r2 = x * x + y * y + z * z;
        const double r = sqrt(r2);
        const double pre = wt[u] * wt[v] * wt[s] * V / (4.0 * 3.14159265358979323846 * r2 * r);
        const double i2 = 3.0 / r2;
        acc[0] += pre * (1.0 - i2 * x * x);
        acc[1] += pre * (1.0 - i2 * y * y);
        acc[2] += pre * (1.0 - i2 * z * z);
        acc[3] -= pre * i2 * x * y;
        acc[4] -= pre * i2 * x * z;
        acc[5] -= pre * i2 * y * z;
      }
  for (int i = 0; i < 6; ++i) out[i] = acc[i];
}

// octant (6, mz, my, mx) with m = L/2 + 1 per axis; zero outside the grid's offsets
__global__ void k_tensor_octant(double* __restrict__ oct, int mx, int my, int mz, int nx, int ny, int nz, double dx,
                                double dy, double dz) {
  const long long tot = (long long)mx * my * mz;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % mx);
    const int j = (int)((e / mx) % my);
    const int k = (int)(e / ((long long)mx * my));
    double v[6] = {0, 0, 0, 0, 0, 0};
    if (i < nx && j < ny && k < nz) {
      const int mxyz = max(i, max(j, k));
      if (mxyz <= 16)
        newell6(i * dx, j * dy, k * dz, dx, dy, dz, v);
      else
        far6(i * dx, j * dy, k * dz, dx, dy, dz, v);
    }
    for (int c = 0; c < 6; ++c) oct[c * tot + e] = v[c];
  }
}

// parity per component (XX,YY,ZZ,XY,XZ,YZ) along x, y, z: 1 = odd
__constant__ int kOdd[6][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}};

// out[c][..k..] = sum_o T_parity[k][o] in[c][..o..] along `axis` of a (6, m2, m1, m0) array
__global__ void k_axis_transform(const double* __restrict__ in, double* __restrict__ out, int m0, int m1, int m2,
                                 int axis, const double* __restrict__ Tc, const double* __restrict__ Ts) {
  const long long per = (long long)m0 * m1 * m2;
  const long long tot = 6 * per;
  const int M = axis == 0 ? m0 : (axis == 1 ? m1 : m2);
  const long long stride = axis == 0 ? 1 : (axis == 1 ? m0 : (long long)m0 * m1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / per);
    const long long r = e - c * per;
    const int i0 = (int)(r % m0), i1 = (int)((r / m0) % m1), i2 = (int)(r / ((long long)m0 * m1));
    const int kk = axis == 0 ? i0 : (axis == 1 ? i1 : i2);
    const long long base = c * per + r - kk * stride;
    const double* T = (kOdd[c][axis] ? Ts : Tc) + (long long)kk * M;
    double s = 0.0;
    for (int o = 0; o < M; ++o) s += T[o] * in[base + o * stride];
    out[e] = s;
  }
}

// Khat[c][kz][ky][P] (fp32, row layout) = scale * sign_c * Nhat[c][kz][ky][kx]
// columns [kxoff, kxoff + kpitch) of the folded spectrum (all of them: kxoff = 0, kpitch = P)
__global__ void k_khat_finalize(const double* __restrict__ in, float* __restrict__ khat, int m0, int m1, int m2,
                                int kxoff, int kpitch, double scale) {
  const long long per = (long long)m0 * m1 * m2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < 6 * per; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / per);
    const long long r = e - c * per;
    const int i0 = (int)(r % m0) - kxoff;
    if (i0 < 0 || i0 >= kpitch) continue;
    const long long row = r / m0;            // kz * m1 + ky
    const double sgn = c >= 3 ? -1.0 : 1.0;  // (-i)^2 of the two odd axes
    khat[(row * kpitch + i0) * 6 + c] = (float)(scale * sgn * in[e]);  // [kz][ky][kpitch][6]
  }
}

static int grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (int)(b < 1 ? 1 : b);
}

void launch_tensor_octant(double* oct, const Dims& d, double dx, double dy, double dz, cudaStream_t s) {
  const int mx = d.Lx / 2 + 1, my = d.Ly / 2 + 1, mz = d.Lz / 2 + 1;
  k_tensor_octant<<<grid_for((long long)mx * my * mz), 256, 0, s>>>(oct, mx, my, mz, d.nx, d.ny, d.nz, dx, dy, dz);
}

void launch_axis_transform(const double* in, double* out, int m0, int m1, int m2, int axis, const double* Tcos,
                           const double* Tsin, cudaStream_t s) {
  k_axis_transform<<<grid_for(6LL * m0 * m1 * m2), 256, 0, s>>>(in, out, m0, m1, m2, axis, Tcos, Tsin);
}

void launch_khat_finalize(const double* in, float* khat, const Dims& d, int kxoff, int kpitch, double scale,
                          cudaStream_t s) {
  const int m0 = d.Lx / 2 + 1, m1 = d.Ly / 2 + 1, m2 = d.Lz / 2 + 1;
  k_khat_finalize<<<grid_for(6LL * m0 * m1 * m2), 256, 0, s>>>(in, khat, m0, m1, m2, kxoff, kpitch, scale);
}

}  // namespace mcq
