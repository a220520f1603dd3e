// k_kinematics.cu — K5: windowed kinematic fused metric + hybrid-boundary
// decision, one warp per window (lane i = trajectory point i, w <= 32).
//
// Restates kinematics.cpp:38-273 Eigen-free, in fp64:
//   project_window   (:38-76)  mean-centre, 3x3 covariance, Jacobi eigen,
//                               top-2 axes with the canonical sign (:63-69);
//   fit_circle_center(:107-207) spread < 1e-9 -> degenerate; collinear start
//                               along the minor scatter axis; damped
//                               Gauss-Newton (lambda 1e-6, x0.3 / x10, <= 25
//                               attempts, step < 1e-10, <= 100 iterations);
//   curvature_radius (:209-218), cumulative_displacement (:220-230),
//   normalize / fused_metric / classify_segment (:232-259),
//   decide_sd cold start.
// Every reduction is a butterfly all-reduce, so all lanes hold bitwise
// identical values and the data-dependent control flow stays warp-uniform.
#include "common.cuh"
#include "kernels.h"

namespace hsd {
namespace {

// 16 windows per block: a decode round's windows occupy few SMs, which the
// engine keeps free of the similarity kernel so K5 overlaps K1 (api.cu).
constexpr int kThreads = 512;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3 (same as the oracle).
__device__ void eig3_sym(double A[3][3], double w[3], double V[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    const double scale = fabs(A[0][0]) + fabs(A[1][1]) + fabs(A[2][2]);
    if (off == 0.0 || off <= 1e-300 || off <= scale * 1e-18) break;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        const double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
    }
  }
  int idx[3] = {0, 1, 2};
  const double d[3] = {A[0][0], A[1][1], A[2][2]};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (d[idx[j]] < d[idx[i]]) {
        const int t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
      }
  double Vs[3][3];
  for (int c = 0; c < 3; ++c) {
    w[c] = d[idx[c]];
    for (int r = 0; r < 3; ++r) Vs[r][c] = V[r][idx[c]];
  }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) V[r][c] = Vs[r][c];
}

// RadiusObjective::eval (kinematics.cpp:90-103)
__device__ __forceinline__ double objective(bool act, double u, double v, double cx, double cy, double inv_n) {
  const double r = act ? hypot(u - cx, v - cy) : 0.0;
  const double mu = wsum(r) * inv_n;
  const double d = act ? (r - mu) : 0.0;
  return wsum(d * d);
}

__global__ void __launch_bounds__(kThreads) kinematics_kernel(const double* __restrict__ xyz, int W, int n,
                                                              hsd_metric_params mp, hsd_norm_bounds nb,
                                                              const int32_t* __restrict__ history,
                                                              double* __restrict__ Rout, double* __restrict__ Dout,
                                                              double* __restrict__ Fout, int32_t* __restrict__ dec,
                                                              double* __restrict__ vaj) {
  const int lane = threadIdx.x & 31;
  const int win = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (win >= W) return;
  const bool act = lane < n;
  const double* P = xyz + (size_t)win * n * 3;
  const double x = act ? P[lane * 3 + 0] : 0.0, y = act ? P[lane * 3 + 1] : 0.0, z = act ? P[lane * 3 + 2] : 0.0;
  const bool finite = !act || (isfinite(x) && isfinite(y) && isfinite(z));
  if (!__all_sync(0xffffffffu, finite)) {  // InvalidInputError (kinematics.cpp:29-35)
    if (lane == 0) {
      Rout[win] = 0.0;
      Dout[win] = 0.0;
      Fout[win] = 0.0;
      dec[win] = -1;
      if (vaj) vaj[(size_t)win * 3 + 0] = vaj[(size_t)win * 3 + 1] = vaj[(size_t)win * 3 + 2] = 0.0;
    }
    return;
  }
  const double inv_n = 1.0 / (double)n;

  // ---- cumulative displacement (Vec3::norm = sqrt(dot), geometry.hpp:17)
  const double nx = __shfl_down_sync(0xffffffffu, x, 1), ny = __shfl_down_sync(0xffffffffu, y, 1),
               nz = __shfl_down_sync(0xffffffffu, z, 1);
  double seg = 0.0;
  if (lane + 1 < n) {
    const double dx = x - nx, dy = y - ny, dz = z - nz;
    seg = sqrt(dx * dx + dy * dy + dz * dz);
  }
  const double D = wsum(seg);

  // ---- windowed finite-difference kinematics (north-star diagnostics; the
  //      reference pins only R / D / F): mean |velocity|, |acceleration|,
  //      |jerk| per action step, v_i = P_{i+1} - P_i, a_i = v_{i+1} - v_i,
  //      j_i = a_{i+1} - a_i.
  if (vaj) {
    const double vx = nx - x, vy = ny - y, vz = nz - z;  // valid on lanes < n - 1
    const double ax_ = __shfl_down_sync(0xffffffffu, vx, 1) - vx, ay_ = __shfl_down_sync(0xffffffffu, vy, 1) - vy,
                 az_ = __shfl_down_sync(0xffffffffu, vz, 1) - vz;  // lanes < n - 2
    const double jx = __shfl_down_sync(0xffffffffu, ax_, 1) - ax_, jy = __shfl_down_sync(0xffffffffu, ay_, 1) - ay_,
                 jz = __shfl_down_sync(0xffffffffu, az_, 1) - az_;  // lanes < n - 3
    const double sv = wsum(lane + 1 < n ? sqrt(__dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz))) : 0.0);
    const double sa = wsum(lane + 2 < n ? sqrt(__dadd_rn(__dadd_rn(__dmul_rn(ax_, ax_), __dmul_rn(ay_, ay_)), __dmul_rn(az_, az_))) : 0.0);
    const double sj = wsum(lane + 3 < n ? sqrt(__dadd_rn(__dadd_rn(__dmul_rn(jx, jx), __dmul_rn(jy, jy)), __dmul_rn(jz, jz))) : 0.0);
    if (lane == 0) {
      vaj[(size_t)win * 3 + 0] = n > 1 ? sv / (double)(n - 1) : 0.0;
      vaj[(size_t)win * 3 + 1] = n > 2 ? sa / (double)(n - 2) : 0.0;
      vaj[(size_t)win * 3 + 2] = n > 3 ? sj / (double)(n - 3) : 0.0;
    }
  }

  // ---- project_window
  const double mx = wsum(x) * inv_n, my = wsum(y) * inv_n, mz = wsum(z) * inv_n;
  const double cx = act ? x - mx : 0.0, cy = act ? y - my : 0.0, cz = act ? z - mz : 0.0;
  double C[3][3];
  C[0][0] = wsum(cx * cx);
  C[0][1] = C[1][0] = wsum(cx * cy);
  C[0][2] = C[2][0] = wsum(cx * cz);
  C[1][1] = wsum(cy * cy);
  C[1][2] = C[2][1] = wsum(cy * cz);
  C[2][2] = wsum(cz * cz);
  double ev[3], V[3][3];
  eig3_sym(C, ev, V);
  double ax[2][3] = {{V[0][2], V[1][2], V[2][2]}, {V[0][1], V[1][1], V[2][1]}};
  for (int k = 0; k < 2; ++k) {
    int lead = 0;
    for (int j = 1; j < 3; ++j)
      if (fabs(ax[k][j]) > fabs(ax[k][lead])) lead = j;
    if (ax[k][lead] < 0.0)
      for (int j = 0; j < 3; ++j) ax[k][j] = -ax[k][j];
  }
  const double u = act ? cx * ax[0][0] + cy * ax[0][1] + cz * ax[0][2] : 0.0;
  const double v = act ? cx * ax[1][0] + cy * ax[1][1] + cz * ax[1][2] : 0.0;

  // ---- fit_circle_center
  const double gx = wsum(u) * inv_n, gy = wsum(v) * inv_n;
  double spread = 0.0;
  for (int j = 0; j < n; ++j) {
    const double uj = __shfl_sync(0xffffffffu, u, j), vj = __shfl_sync(0xffffffffu, v, j);
    if (act && j > lane) spread = fmax(spread, hypot(u - uj, v - vj));
  }
  spread = wmax(spread);
  double R = 0.0;
  if (!(spread < 1e-9)) {
    const double du = act ? u - gx : 0.0, dv = act ? v - gy : 0.0;
    const double sa = wsum(du * du), sb = wsum(du * dv), sc = wsum(dv * dv);
    const double half_tr = 0.5 * (sa + sc), half_diff = 0.5 * (sa - sc);
    const double rad = sqrt(half_diff * half_diff + sb * sb);
    const double l1 = half_tr + rad, l0 = half_tr - rad;
    double ex, ey;
    if (sb == 0.0) {
      ex = sa <= sc ? 1.0 : 0.0;
      ey = sa <= sc ? 0.0 : 1.0;
    } else if (fabs(l0 - sa) >= fabs(l0 - sc)) {
      ex = sb;
      ey = l0 - sa;
    } else {
      ex = l0 - sc;
      ey = sb;
    }
    const double en = sqrt(ex * ex + ey * ey);
    ex /= en;
    ey /= en;
    double px = gx, py = gy;
    if (l0 <= 1e-12 * l1) {
      px += ex * spread;
      py += ey * spread;
    }
    double lambda = 1e-6;
    double obj = objective(act, u, v, px, py, inv_n);
    for (int iter = 0; iter < 100; ++iter) {
      const double dx = act ? u - px : 0.0, dy = act ? v - py : 0.0;
      const double r = sqrt(dx * dx + dy * dy);
      const double ux = (act && r > 0.0) ? dx / r : 0.0, uy = (act && r > 0.0) ? dy / r : 0.0;
      const double mu = wsum(r) * inv_n;
      const double mux = wsum(ux) * inv_n, muy = wsum(uy) * inv_n;
      const double jx = act ? -ux + mux : 0.0, jy = act ? -uy + muy : 0.0;
      const double f = act ? r - mu : 0.0;
      const double j00 = wsum(jx * jx), j01 = wsum(jx * jy), j11 = wsum(jy * jy);
      const double g0 = wsum(jx * f), g1 = wsum(jy * f);
      bool moved = false, done = false;
      for (int attempt = 0; attempt < 25; ++attempt) {
        // LDLT (diagonal pivoting) solve of (J^T J + lambda I) s = -J^T f
        const double a = j00 + lambda, c = j11 + lambda, b = j01;
        const bool sw = fabs(c) > fabs(a);
        const double A00 = sw ? c : a, A11 = sw ? a : c, q0 = sw ? -g1 : -g0, q1 = sw ? -g0 : -g1;
        const double l = b / A00, d1 = A11 - l * b;
        const double z1 = (q1 - l * q0) / d1, z0 = q0 / A00;
        const double s1v = z1, s0v = z0 - l * s1v;
        const double s0 = sw ? s1v : s0v, s1 = sw ? s0v : s1v;
        if (!isfinite(s0) || !isfinite(s1)) {
          lambda *= 10.0;
          continue;
        }
        const double cand = objective(act, u, v, px + s0, py + s1, inv_n);
        if (cand <= obj) {
          px += s0;
          py += s1;
          obj = cand;
          lambda = fmax(lambda * 0.3, 1e-12);
          moved = sqrt(s0 * s0 + s1 * s1) >= 1e-10;
          if (!moved) done = true;
          break;
        }
        lambda *= 10.0;
      }
      if (done || !moved) break;
    }
    const double dist = act ? hypot(u - px, v - py) : 0.0;
    R = wsum(dist) * inv_n;
    R = R < mp.r_cap ? R : mp.r_cap;
  }
  // ---- normalize / fused metric / classify (kinematics.cpp:232-259)
  auto nrm = [](double xv, double lo, double hi) {
    if (lo == hi) return 0.0;
    const double t = (xv - lo) / (hi - lo);
    return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  };
  const double F = mp.alpha * nrm(R, nb.r_min, nb.r_max95) + (1.0 - mp.alpha) * nrm(D, nb.d_min, nb.d_max95);
  const bool warm = history ? history[win] >= mp.w : true;
  if (lane == 0) {
    Rout[win] = R;
    Dout[win] = D;
    Fout[win] = F;
    dec[win] = (warm && F > mp.threshold) ? 1 : 0;
  }
}

}  // namespace

cudaError_t launch_kinematics(const double* xyz, int W, const hsd_metric_params& mp, const hsd_norm_bounds& nb,
                              const int32_t* history, double* R, double* D, double* F, int32_t* decision,
                              cudaStream_t s, double* vaj) {
  if (W <= 0) return cudaSuccess;
  const int wpb = kThreads / 32;
  kinematics_kernel<<<(W + wpb - 1) / wpb, kThreads, 0, s>>>(xyz, W, mp.w, mp, nb, history, R, D, F, decision, vaj);
  return cudaGetLastError();
}

}  // namespace hsd
