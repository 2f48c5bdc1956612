// ES-BGK (anisotropic Gaussian) equilibrium on the device (collision.hpp:52-71,
// 84-94): Lambda = theta I + (1 - 1/Pr)/rho sigma with the stress of
// extract_macro (moment_rep.hpp:126-133, sigma_ij = (1 + delta_ij) f_{e_i+e_j}),
// the SPD check min eig(Lambda) > 1e-12 theta (NonSpdTensor otherwise), and the
// Gaussian's coefficients in the cell's own basis by the two-step recurrence
//   g_{mu + e_d} = sum_j C_{dj} g_{mu - e_j} / (mu_d + 1),  C = Lambda - theta I,
// seeded at g_0 = rho, odd degrees zero.  Used by the thread-per-face
// (thread_cell.cuh, M <= 6) and warp-per-cell (momg_cell.cuh, M = 7, 8)
// kernels; the band kernels route ES-BGK sweeps to those (kernels_impl.cuh).
// The eigenvalue check is the cyclic Jacobi of the oracle (the reference uses
// Eigen's SelfAdjointEigenSolver; only the SPD decision depends on it).
#pragma once

#include "types.h"

namespace momg_gpu {
namespace es {

__device__ __forceinline__ double min_eig3(const double (&A)[3][3]) {
  double a[3][3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) a[p][q] = A[p][q];
  for (int sweep = 0; sweep < 60; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    if (off == 0.0) break;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = cs * akp - sn * akq;
          a[k][q] = sn * akp + cs * akq;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = cs * apk - sn * aqk;
          a[q][k] = sn * apk + cs * aqk;
        }
      }
  }
  const double m01 = a[1][1] < a[0][0] ? a[1][1] : a[0][0];
  return a[2][2] < m01 ? a[2][2] : m01;
}

// Lambda of equilibrium_rep (collision.hpp:86-87) from a state S (stride ST)
// centred on its own basis
template <int ST>
__device__ __forceinline__ void lambda(const double* S, double theta, double prandtl, double (&lam)[3][3]) {
  const double rho = S[0];
  const double corr = 1.0 - 1.0 / prandtl;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int k = flat3((i == 0) + (j == 0), (i == 1) + (j == 1), (i == 2) + (j == 2));
      const double sig = (i == j ? 2.0 : 1.0) * S[k * ST];
      lam[i][j] = theta * (i == j ? 1.0 : 0.0) + corr / rho * sig;
    }
}

// the SPD check; W_NON_SPD with *bad = the minimum eigenvalue
template <int ST>
__device__ __forceinline__ int check(const double* S, double theta, double prandtl, double* bad) {
  double lam[3][3];
  lambda<ST>(S, theta, prandtl, lam);
  const double me = min_eig3(lam);
  if (!(me > 1e-12 * theta)) {
    *bad = me;
    return W_NON_SPD;
  }
  return W_NONE;
}

// gaussian_rep (collision.hpp:52-71) into eq (stride ST), every coefficient
template <int M, int ST>
__device__ __forceinline__ void fill(const double* S, double theta, double prandtl, double* eq) {
  double lam[3][3], c[3][3];
  lambda<ST>(S, theta, prandtl, lam);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[i][j] = lam[i][j] - theta * (i == j ? 1.0 : 0.0);
  eq[0] = S[0];
#pragma unroll
  for (int n = 1; n <= M; ++n)
#pragma unroll
    for (int a1 = n; a1 >= 0; --a1)
#pragma unroll
      for (int a2 = n - a1; a2 >= 0; --a2) {
        const int a3 = n - a1 - a2;
        const int k = flat3(a1, a2, a3);
        if (n & 1) {
          eq[k * ST] = 0.0;
          continue;
        }
        const int d = a1 > 0 ? 0 : (a2 > 0 ? 1 : 2);  // first axis with down(k, d) >= 0
        const int m[3] = {a1 - (d == 0), a2 - (d == 1), a3 - (d == 2)};
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (m[j] > 0) acc += c[d][j] * eq[flat3(m[0] - (j == 0), m[1] - (j == 1), m[2] - (j == 2)) * ST];
        eq[k * ST] = acc / (double)(m[d] + 1);
      }
}

}  // namespace es
}  // namespace momg_gpu
