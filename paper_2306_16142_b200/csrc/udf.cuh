// Unsigned distance from the DDF (paper Eq. 5: UDF(x) = min_theta phi(x, theta)):
// field.udf_many (field.py:418-488) and recon.udf_grid (recon.py:61-81).
//
// Stage 1 (scan) is one MLP pass over points x directions (row s -> point
// s / n_dirs, Halton direction s % n_dirs) with QueryOp's exact per-row math
// (field.py:248-258); its value (t on a hit, +inf on a miss) lands in a
// row-major (points, n_dirs) buffer and a warp per point takes the first
// argmin.  Stage 2 (polish) runs the reference's lockstep golden-section
// search per found point: 2 rounds x {polar, azimuth} x 13 probe pairs, every
// pair one MLP pass of 2 rows per point (ProbeOp) followed by a tiny state
// kernel.  All state is float64 and updated with the reference's operation
// order (no FMA contraction), so the only differences from the f64 reference
// are the network's own fp32 / bf16 rounding.
#pragma once
#include "ddf_common.cuh"
#include "field_kernels.cuh"

namespace ddf {
namespace udf {

constexpr double INF = __builtin_huge_val();

// per-row query value (field.py:411-413, 441-442)
__device__ __forceinline__ double query_value(double pred, double delta, double thresh) {
  const double c = fmin(fmax(pred, -delta), delta);
  return c < thresh ? fmax(c, 0.0) : INF;
}

// query_batch's canonicalisation of a direction vector into encoded angles
__device__ __forceinline__ void query_u34(d3 d, double& u3, double& u4) {
  double a0, a1;
  dir_angles(d, a0, a1);                 // field.py:258
  dir_u34(angles_dir(a0, a1), u3, u4);   // field.py:251 re-canonicalise
}

// the encoded angles of a direction do not depend on the point: once per direction
#ifndef DDF_OPS_ONLY
__global__ void dir_u34_kernel(const double* dirs, int n, double* u34) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) query_u34(ld3(dirs, k), u34[2 * k], u34[2 * k + 1]);
}
#endif

struct ScanOp : ListBase {
  static constexpr bool kGrad = false;
  static constexpr bool kRaw = false;
  const double* pts; const double* u34; int n_dirs;
  double* vals; double delta, thresh;
  __device__ double raw(int, int) const { return 0.0; }
  __device__ void load(int s, double* p, double& u3, double& u4) const {
    const int pt = s / n_dirs, k = s - pt * n_dirs;
    const d3 q = ld3(pts, pt);
    p[0] = q.x; p[1] = q.y; p[2] = q.z;
    u3 = u34[2 * k];
    u4 = u34[2 * k + 1];
  }
  __device__ void store_fwd(int s, double pred, int) const { vals[s] = query_value(pred, delta, thresh); }
};

// Golden-section state of the found points, SoA (q = index among found points).
struct Polish {
  const int* pidx;      // q -> point index
  double* ang;          // (nq, 2) current best angles (azimuth, polar)
  double* val;          // current best value
  double* lo; double* hi; double* x1; double* x2; double* f1; double* f2;
};

struct ProbeOp : ListBase {   // rows 2q + e: probe x1 (e = 0) or x2 (e = 1) of point q
  static constexpr bool kGrad = false;
  static constexpr bool kRaw = false;
  const double* pts; Polish P; int axis; double delta, thresh;
  __device__ double raw(int, int) const { return 0.0; }
  __device__ void load(int s, double* p, double& u3, double& u4) const {
    const int q = s >> 1;
    const d3 c = ld3(pts, P.pidx[q]);
    p[0] = c.x; p[1] = c.y; p[2] = c.z;
    const double x = (s & 1) ? P.x2[q] : P.x1[q];
    const double a0 = axis == 0 ? x : P.ang[2 * q];
    const double a1 = axis == 0 ? P.ang[2 * q + 1] : x;
    query_u34(angles_dir(a0, a1), u3, u4);   // field.py:409-413: angles_to_vecs -> query_batch
  }
  __device__ void store_fwd(int s, double pred, int) const {
    ((s & 1) ? P.f2 : P.f1)[s >> 1] = query_value(pred, delta, thresh);
  }
};

// one warp per point: first argmin over its n_dirs values (field.py:438-448)
#ifndef DDF_OPS_ONLY
__global__ void reduce_kernel(const double* vals, int n_pts, int n_dirs, double* best, int* arg, uint8_t* found) {
  const int lane = threadIdx.x & 31;
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n_pts) return;
  const double* v = vals + (int64_t)p * n_dirs;
  double bv = INF;
  int bi = 0x7fffffff;
  for (int k = lane; k < n_dirs; k += 32) {
    const double x = v[k];
    if (x < bv) { bv = x; bi = k; }
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) {
    best[p] = bv;
    arg[p] = bi == 0x7fffffff ? 0 : bi;   // all +inf: np.argmin -> 0
    found[p] = bv < INF;
  }
}
#endif

// found point q: start angles = vecs_to_angles(best direction) (field.py:449)
#ifndef DDF_OPS_ONLY
__global__ void polish_init(Polish P, const int* arg, const double* best, const double* dirs, int nq_max,
                            const int* nq) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq_max || q >= *nq) return;
  const int p = P.pidx[q];
  double a0, a1;
  dir_angles(ld3(dirs, arg[p]), a0, a1);
  P.ang[2 * q] = a0;
  P.ang[2 * q + 1] = a1;
  P.val[q] = best[p];
}
#endif

// field.py:462-470: window about the current angle, first probe pair
#ifndef DDF_OPS_ONLY
__global__ void gs_begin(Polish P, int axis, double half, double golden, int nq_max, const int* nq) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq_max || q >= *nq) return;
  const double c = P.ang[2 * q + axis];
  double a = dsub(c, half), b = dadd(c, half);
  if (axis == 1) {
    const double pi = 3.141592653589793;
    a = fmin(fmax(a, 0.0), pi);
    b = fmin(fmax(b, 0.0), pi);
  }
  P.lo[q] = a; P.hi[q] = b;
  P.x1[q] = dsub(b, dmul(golden, dsub(b, a)));
  P.x2[q] = dadd(a, dmul(golden, dsub(b, a)));
}
#endif

// field.py:477-482: keep the side holding the smaller probe, new probe pair
#ifndef DDF_OPS_ONLY
__global__ void gs_step(Polish P, double golden, int nq_max, const int* nq) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq_max || q >= *nq) return;
  const bool right = P.f1[q] > P.f2[q];
  const double a = right ? P.x1[q] : P.lo[q];
  const double b = right ? P.hi[q] : P.x2[q];
  P.lo[q] = a; P.hi[q] = b;
  P.x1[q] = dsub(b, dmul(golden, dsub(b, a)));
  P.x2[q] = dadd(a, dmul(golden, dsub(b, a)));
}
#endif

// field.py:483-487: accept the better probe if it improves strictly
#ifndef DDF_OPS_ONLY
__global__ void gs_end(Polish P, int axis, int nq_max, const int* nq) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq_max || q >= *nq) return;
  const double f1 = P.f1[q], f2 = P.f2[q];
  const double xs = f1 < f2 ? P.x1[q] : P.x2[q];
  const double fs = fmin(f1, f2);
  if (fs < P.val[q]) {
    P.val[q] = fs;
    P.ang[2 * q + axis] = xs;
  }
}
#endif

#ifndef DDF_OPS_ONLY
__global__ void polish_scatter(Polish P, double* out, int nq_max, const int* nq) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq_max || q >= *nq) return;
  out[P.pidx[q]] = P.val[q];
}
#endif

// recon.py:53-58: np.linspace(lo, hi, res) per axis (i * step + lo, last = hi),
// ij meshgrid, C order (z fastest)
#ifndef DDF_OPS_ONLY
__global__ void grid_points_kernel(double* pts, int res, double lx, double ly, double lz, double hx, double hy,
                                   double hz) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)res * res * res;
  if (i >= n) return;
  const int ix = (int)(i / ((int64_t)res * res)), iy = (int)((i / res) % res), iz = (int)(i % res);
  const double lo[3] = {lx, ly, lz}, hi[3] = {hx, hy, hz};
  const int idx[3] = {ix, iy, iz};
  for (int k = 0; k < 3; ++k) {
    const double step = ddiv(dsub(hi[k], lo[k]), (double)(res - 1));
    pts[3 * i + k] = idx[k] == res - 1 ? hi[k] : dadd(dmul((double)idx[k], step), lo[k]);
  }
}
#endif

}  // namespace udf
}  // namespace ddf
