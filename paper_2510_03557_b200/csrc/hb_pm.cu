// hb_pm.cu -- particle-mesh long-range gravity (hb/gravity.py:58-245), the
// step on the other side of the short-range path.
//
//   hb_pm_deposit   cloud-in-cell mass deposition onto cell centres, periodic
//                   (hb/gravity.py:58-82): one thread per particle, 8 float64
//                   atomics; index / fraction / weight arithmetic in the
//                   reference's operation order (u = x / h - 0.5, i0 = floor(u),
//                   f = u - i0, w = ((m wx) wy) wz), then rho /= h^3 in a
//                   separate pass as the reference does.
//   hb_pm_spectral  phi_k = -(4 pi G) rho_k D(k), phi_0 = 0, and the three
//                   ik-differentiated force spectra F_k = -i k_d phi_k
//                   (hb/gravity.py:196-216) in one pass over the half-complex
//                   grid (the FFTs themselves are cuFFT's).
//   hb_pm_interp    trilinear gather with the deposition stencil
//                   (hb/gravity.py:219-241), same 8-term summation order.
#include "hb_common.cuh"

namespace hb {

struct Cic {
  int64_t i0[3], i1[3];
  double f[3];
};

// cell-centred CIC stencil (hb/gravity.py:58-66): floor / mod as numpy does
__device__ __forceinline__ Cic cic_of(const double* p, int64_t n, double spacing) {
  Cic c;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double u = __dsub_rn(__ddiv_rn(p[d], spacing), 0.5);
    double fl = floor(u);
    int64_t i = (int64_t)fl;
    c.f[d] = __dsub_rn(u, fl);
    int64_t m0 = i % n, m1 = (i + 1) % n;
    c.i0[d] = m0 < 0 ? m0 + n : m0;
    c.i1[d] = m1 < 0 ? m1 + n : m1;
  }
  return c;
}

__global__ void k_pm_deposit(int64_t np, const double* pos, const double* mass, int64_t n,
                             double spacing, double* rho) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  Cic c = cic_of(pos + 3 * k, n, spacing);
  double m = mass[k];
  double w0[3], w1[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) { w1[d] = c.f[d]; w0[d] = __dsub_rn(1.0, c.f[d]); }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    int64_t cx = a ? c.i1[0] : c.i0[0];
    double wx = a ? w1[0] : w0[0];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      int64_t cy = b ? c.i1[1] : c.i0[1];
      double wy = b ? w1[1] : w0[1];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int64_t cz = e ? c.i1[2] : c.i0[2];
        double wz = e ? w1[2] : w0[2];
        double v = __dmul_rn(__dmul_rn(__dmul_rn(m, wx), wy), wz);
        atomicAdd(&rho[(cx * n + cy) * n + cz], v);
      }
    }
  }
}

__global__ void k_pm_scale(int64_t m, double* v, double vol) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) v[k] = __ddiv_rn(v[k], vol);
}

// half-complex grid (n, n, n/2+1) row-major; k = 2 pi / L * fftfreq index
__global__ void k_pm_spectral(int64_t n, double L, double four_pi_g, const double2* rho_k,
                              const double* d_k, double2* fx, double2* fy, double2* fz,
                              double2* phi) {
  int64_t nh = n / 2 + 1;
  int64_t m = n * n * nh;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int64_t iz = t % nh, iy = (t / nh) % n, ix = t / (nh * n);
  // 2 pi * np.fft.(r)fftfreq(n, d=L/n): j * (1 / (n * (L / n))) then * 2 pi, with
  // j in [0, (n+1)/2) U [-n/2, 0) on the full axes and [0, n/2] on the half axis
  double val = __ddiv_rn(1.0, __dmul_rn((double)n, __ddiv_rn(L, (double)n)));
  const double two_pi = 6.283185307179586;
  auto kval = [&](int64_t j) {
    int64_t jj = j < (n + 1) / 2 ? j : j - n;
    return __dmul_rn(two_pi, __dmul_rn((double)jj, val));
  };
  double kx = kval(ix), ky = kval(iy), kz = __dmul_rn(two_pi, __dmul_rn((double)iz, val));
  double2 r = rho_k[t];
  double s = -four_pi_g;
  double2 p = make_double2(__dmul_rn(__dmul_rn(s, r.x), d_k[t]), __dmul_rn(__dmul_rn(s, r.y), d_k[t]));
  if (t == 0) p = make_double2(0.0, 0.0);
  if (phi) phi[t] = p;
  // -1j * k * phi = k * phi.y - 1j * k * phi.x
  fx[t] = make_double2(__dmul_rn(kx, p.y), -__dmul_rn(kx, p.x));
  fy[t] = make_double2(__dmul_rn(ky, p.y), -__dmul_rn(ky, p.x));
  fz[t] = make_double2(__dmul_rn(kz, p.y), -__dmul_rn(kz, p.x));
}

__global__ void k_pm_interp(int64_t np, const double* pos, int nf, const double* f0,
                            const double* f1, const double* f2, int64_t n, double spacing,
                            double* out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  Cic c = cic_of(pos + 3 * k, n, spacing);
  double w0[3], w1[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) { w1[d] = c.f[d]; w0[d] = __dsub_rn(1.0, c.f[d]); }
  const double* fld[3] = {f0, f1, f2};
  for (int q = 0; q < nf; ++q) {
    const double* v = fld[q];
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      int64_t cx = a ? c.i1[0] : c.i0[0];
      double wx = a ? w1[0] : w0[0];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        int64_t cy = b ? c.i1[1] : c.i0[1];
        double wy = b ? w1[1] : w0[1];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int64_t cz = e ? c.i1[2] : c.i0[2];
          double wz = e ? w1[2] : w0[2];
          acc = __dadd_rn(acc, __dmul_rn(v[(cx * n + cy) * n + cz],
                                         __dmul_rn(__dmul_rn(wx, wy), wz)));
        }
      }
    }
    out[k * nf + q] = acc;
  }
}

}  // namespace hb

using namespace hb;

extern "C" int hb_pm_deposit(int64_t np, const double* pos, const double* mass, int64_t grid_n,
                             double spacing, double cell_volume, double* rho, void* stream,
                             HbError* err) {
  if (err) *err = HbError{};
  cudaStream_t st = (cudaStream_t)stream;
  int64_t m = grid_n * grid_n * grid_n;
  if (grid_n <= 0) return set_err(err, HB_CONTRACT, "grid_n must be positive");
  HB_CUDA_TRY(cudaMemsetAsync(rho, 0, m * sizeof(double), st));
  if (np > 0) {
    k_pm_deposit<<<grid_for(np, 256), 256, 0, st>>>(np, pos, mass, grid_n, spacing, rho);
    HB_LAUNCH_CHECK();
  }
  k_pm_scale<<<grid_for(m, 256), 256, 0, st>>>(m, rho, cell_volume);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" int hb_pm_spectral(int64_t grid_n, double side_length, double four_pi_g,
                              const void* rho_k, const double* influence, void* fx_k, void* fy_k,
                              void* fz_k, void* phi_k, void* stream, HbError* err) {
  if (err) *err = HbError{};
  int64_t m = grid_n * grid_n * (grid_n / 2 + 1);
  k_pm_spectral<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(
      grid_n, side_length, four_pi_g, (const double2*)rho_k, influence, (double2*)fx_k,
      (double2*)fy_k, (double2*)fz_k, (double2*)phi_k);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" int hb_pm_interp(int64_t np, const double* pos, int32_t n_fields, const double* f0,
                            const double* f1, const double* f2, int64_t grid_n, double spacing,
                            double* out, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (n_fields < 1 || n_fields > 3) return set_err(err, HB_CONTRACT, "n_fields must be 1..3");
  if (np <= 0) return HB_OK;
  k_pm_interp<<<grid_for(np, 256), 256, 0, (cudaStream_t)stream>>>(np, pos, n_fields, f0, f1, f2,
                                                                  grid_n, spacing, out);
  HB_LAUNCH_CHECK();
  return HB_OK;
}
