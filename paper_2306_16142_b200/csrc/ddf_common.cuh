// Shared device-side definitions for the B200 DDF hot path.
//
// Geometry (rays, slab test, normals, cosine sampling, film) stays in float64
// exactly as the reference computes it (ddfield/render.py, ddfield/field.py);
// the explicit __dadd_rn/__dmul_rn helpers keep nvcc from contracting a*b+c
// into an FMA, so the sqrt/mul/add paths round like numpy does.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef DDF_MAX_LAYERS
#define DDF_MAX_LAYERS 12      // weight layers per network (configs use <= 9)
#endif
#define DDF_MAX_OBJECTS 8      // networks per field (config 5 uses 8)
#define DDF_PE_OCTAVES 6
#define DDF_HIT_FRACTION 0.98  // ddfield/field.py:24 MISS_FRACTION

namespace ddf {

// ---------------------------------------------------------------- f64 helpers
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

struct d3 { double x, y, z; };
__device__ __forceinline__ d3 mk3(double x, double y, double z) { return d3{x, y, z}; }
// numpy: sqrt((x*x + y*y) + z*z)  (np.linalg.norm over a length-3 axis)
__device__ __forceinline__ double norm3(d3 v) {
  return __dsqrt_rn(dadd(dadd(dmul(v.x, v.x), dmul(v.y, v.y)), dmul(v.z, v.z)));
}
// numpy einsum("ij,ij->i"): ((x*x' + y*y') + z*z')
__device__ __forceinline__ double dot3(d3 a, d3 b) {
  return dadd(dadd(dmul(a.x, b.x), dmul(a.y, b.y)), dmul(a.z, b.z));
}
// np.cross
__device__ __forceinline__ d3 cross3(d3 a, d3 b) {
  return mk3(dsub(dmul(a.y, b.z), dmul(a.z, b.y)),
             dsub(dmul(a.z, b.x), dmul(a.x, b.z)),
             dsub(dmul(a.x, b.y), dmul(a.y, b.x)));
}

// field.py:77-82 vecs_to_angles: (atan2(y,x) mod 2pi, arccos(clip(z,-1,1)))
__device__ __forceinline__ void dir_angles(d3 d, double& az, double& pol) {
  const double two_pi = 6.283185307179586;
  double zc = fmin(fmax(d.z, -1.0), 1.0);
  pol = acos(zc);
  double a = atan2(d.y, d.x);
  // numpy float mod: result has the sign of the divisor
  double r = fmod(a, two_pi);
  if (r != 0.0 && r < 0.0) r = dadd(r, two_pi);
  az = r;
}
// field.py:69-74 angles_to_vecs
__device__ __forceinline__ d3 angles_dir(double az, double pol) {
  double s = sin(pol);
  return mk3(dmul(cos(az), s), dmul(sin(az), s), cos(pol));
}
// neural.py:36-37 encoded angle inputs
__device__ __forceinline__ void encode_angles(double az, double pol, double& u3, double& u4) {
  const double pi = 3.141592653589793;
  u3 = dsub(ddiv(az, pi), 1.0);
  u4 = dsub(ddiv(dmul(2.0, pol), pi), 1.0);
}

// field.py:323-337 slab test; returns enter > exit on a miss
__device__ __forceinline__ void ray_box(d3 o, d3 d, const double* lo, const double* hi,
                                        double& t_enter, double& t_exit) {
  double oc[3] = {o.x, o.y, o.z}, dc[3] = {d.x, d.y, d.z};
  double a = -INFINITY, b = INFINITY;
  #pragma unroll
  for (int k = 0; k < 3; ++k) {
    double lo_k, hi_k;
    if (dc[k] == 0.0) {
      bool inside = oc[k] >= lo[k] && oc[k] <= hi[k];
      lo_k = inside ? -INFINITY : INFINITY;
      hi_k = inside ? INFINITY : -INFINITY;
    } else {
      double inv = ddiv(1.0, dc[k]);
      double t0 = dmul(dsub(lo[k], oc[k]), inv);
      double t1 = dmul(dsub(hi[k], oc[k]), inv);
      // np.minimum/np.maximum propagate NaN
      lo_k = (t0 != t0 || t1 != t1) ? NAN : fmin(t0, t1);
      hi_k = (t0 != t0 || t1 != t1) ? NAN : fmax(t0, t1);
    }
    a = (k == 0) ? lo_k : ((a != a || lo_k != lo_k) ? NAN : fmax(a, lo_k));
    b = (k == 0) ? hi_k : ((b != b || hi_k != hi_k) ? NAN : fmin(b, hi_k));
  }
  t_enter = a;
  t_exit = b;
}

// ---------------------------------------------------------------- PCG64
// numpy PCG64 = 128-bit LCG (multiplier 0x2360ED051FC65DA44385DF649FCCF645)
// with the XSL-RR 128->64 output taken after each step; Generator.random()
// is (next64 >> 11) * 2^-53.  Draw k is the output after k+1 steps.
struct u128 { uint64_t lo, hi; };

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
#else
  r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64) + a.hi * b.lo + a.lo * b.hi;
#endif
  return r;
}
__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
__host__ __device__ __forceinline__ uint64_t pcg_out(u128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned r = (unsigned)(s.hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// Jump table: step 2^b is  s -> mult[b] * s + plus[b]  (host-built per stream).
struct PcgStream {
  u128 state;          // seed state (before the first step)
  u128 mult[64];
  u128 plus[64];
};

__device__ __forceinline__ u128 pcg_jump(const PcgStream& st, uint64_t delta) {
  u128 s = st.state;
  for (int b = 0; delta; ++b, delta >>= 1)
    if (delta & 1ull) s = add128(mul128(st.mult[b], s), st.plus[b]);
  return s;
}
__device__ __forceinline__ double pcg_to_double(uint64_t v) {
  return (double)(v >> 11) * (1.0 / 9007199254740992.0);
}
// Two consecutive draws k, k+1 (the (.., 2) rows of rng.random((N, 2))).
__device__ __forceinline__ void pcg_pair(const PcgStream& st, uint64_t k, double& u0, double& u1) {
  u128 s = pcg_jump(st, k + 1);
  u0 = pcg_to_double(pcg_out(s));
  s = add128(mul128(st.mult[0], s), st.plus[0]);
  u1 = pcg_to_double(pcg_out(s));
}
__device__ __forceinline__ double pcg_single(const PcgStream& st, uint64_t k) {
  return pcg_to_double(pcg_out(pcg_jump(st, k + 1)));
}

// ---------------------------------------------------------------- network / field
enum Precision : int { PREC_FP32 = 0, PREC_BF16 = 1, PREC_FP32_SIMT = 2 };
enum Encoding : int { ENC_RAW5 = 0, ENC_PE6 = 1 };

struct NetDev {
  int n_layers;                    // weight layers (hidden ReLU layers + identity head)
  int widths[DDF_MAX_LAYERS + 1];  // widths[0] = network input width (5 or 65)
  int encoding;                    // Encoding
  double center[3];                // EXTENSION (config 5): object translation
  double scale;                    // EXTENSION: uniform object scale
  double inv_scale;                // 1 / scale, for the bf16 engines' input encoding (row_u_bf16)
  double albedo;                   // EXTENSION: per-object albedo
  // fp32 engine: row-major (out, in) effective weights and their transposes
  const float* w[DDF_MAX_LAYERS];
  const float* wt[DDF_MAX_LAYERS];
  const float* b[DDF_MAX_LAYERS];
  // bf16 tcgen05 engine: UMMA-ready pre-swizzled weight images (see mlp_umma.cuh)
  const void* wimg_fwd;
  const void* wimg_bwd;
  // fp32 mode on the tensor cores: 3xTF32 program + images (mlp_x3.cuh), or null
  const void* wimg_x3;
  int max_width;
};

struct FieldDev {
  int n_obj;
  int precision;
  double delta;
  double lo[3], hi[3];
  double step;        // 0.9 delta         (field.py:270)
  double thresh;      // 0.98 delta        (field.py:271)
  double backoff;     // 0.5 delta         (field.py:237)
  int max_steps;      // ceil(diag/step)+4 (field.py:272-273)
  bool composite;
  int is_mesh;        // 1: exact triangle-mesh field (OracleField), no networks
  NetDev net[DDF_MAX_OBJECTS];
};

// device error word bits (mapped to the reference's exceptions by the host)
enum DevError : int { DEVERR_SIGN_RULE = 1 };

}  // namespace ddf
