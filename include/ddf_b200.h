/* C ABI of the B200 DDF hot path (libddf_b200.so).
 *
 * The reference (ddfield, pure Python) has no FFI; its "plugin interface" for
 * this path is the duck-typed backend protocol that render.render_* calls
 * (ddfield/field.py:161-186, 248-317, 320) plus render.render_path
 * (ddfield/render.py:198-247) and the DDFN weight layout
 * (ddfield/neural.py:378-431).  Each entry point below replaces one of those
 * and cites it.  The Python shim paper_2306_16142_b200.field.CudaNeuralField
 * binds them with ctypes.
 *
 * Conventions
 *  - Array arguments are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *    C-contiguous, float64 unless stated; (N,3) arrays are row-major xyz.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    stream-ordered; ddf_render_path and ddf_render_mode synchronise the
 *    stream before returning because they report numeric errors,
 *    ddf_compact and ddf_rng_doubles synchronise too, and ddf_udf /
 *    ddf_udf_grid synchronise the device once
 *    whenever a handle first sees a new direction count (direction table).
 *  - One call at a time per field handle (its scratch is reused); handles are
 *    independent, so concurrent calls on different handles are fine.
 *    ddf_compact allocates its scratch per call (stream-ordered, on the
 *    device that owns `flags`).
 *  - Return value: DDF_OK or an error class mirroring ddfield/errors.py;
 *    ddf_last_error() holds the message (thread-local).
 */
#ifndef DDF_B200_H
#define DDF_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDF_OK 0
#define DDF_EUSAGE 1   /* ValueError / usage (cli.py:502-517 exit 1)       */
#define DDF_EDATA 2    /* DataError   (errors.py:12-13, exit 2)             */
#define DDF_ENUMERIC 3 /* NumericError (errors.py:16-17, exit 3)            */
#define DDF_ECUDA 4    /* CUDA runtime failure                             */

#define DDF_PREC_FP32 0      /* fp32-accurate MLP: 3xTF32 on tcgen05 (hidden <= 256 wide), else FFMA */
#define DDF_PREC_BF16 1      /* tcgen05 bf16 MLP, fp32 accumulate              */
#define DDF_PREC_FP32_SIMT 2 /* exact fp32 FFMA MLP (CUDA cores), any width    */

#define DDF_ENC_RAW5 0  /* neural.py:26-38 (x,y,z,az/pi-1,2pol/pi-1)      */
#define DDF_ENC_PE6 1   /* + 6-octave sin/cos encoding -> 65 inputs (configs 3-5) */

#define DDF_STAGE_STEPS 64    /* ddf_render_stats_t.primary_march_rows entries */
#define DDF_STAGE_BOUNCES 32  /* ddf_render_stats_t.bounce_*_rows entries        */

typedef struct ddf_field_s* ddf_field_t;

typedef struct {
  /* render.Camera after __post_init__ (render.py:33-51), computed by the host */
  double position[3], forward[3], right[3], up_ortho[3];
  double tan_half; /* tan(vfov/2) */
  double aspect;   /* width/height */
  int32_t width, height;
} ddf_camera_t;

typedef struct {
  /* render.RenderConfig fields used by render_path (render.py:106-124) */
  int32_t spp, bounces;
  double albedo, env_radiance;
  /* numpy PCG64 of default_rng([seed, 0x9A7]) (render.py:209): 128-bit state
     and increment as (lo, hi) u64 pairs, from bit_generator.state */
  uint64_t rng_state[2], rng_inc[2];
  /* EXTENSION (config 4): Russian roulette from this bounce index, -1 = off,
     with its own PCG64 stream */
  int32_t rr_start;
  uint64_t rr_state[2], rr_inc[2];
  /* image-tile sharding (config 4): tiles of tile x tile pixels, row-major,
     tile k owned by rank k % world; tile = 0 renders every pixel */
  int32_t tile, rank, world;
  /* path slots per wave (0 = default); larger waves mean fewer launches */
  int64_t max_wave_paths;
  /* 1: time every kernel class with CUDA events on `stream` (stats.ms_*) */
  int32_t profile;
  /* 1: replay the waves as a CUDA graph captured on the first call with the
     same camera, config and field (ignored when profile = 1 or stage_log is
     set).  The graph renders into the field's own film buffer, copied to
     accum at the end, so the caller's accumulator may move between calls. */
  int32_t graph;
  /* 1: never fuse a bounce ray's first march step with the next bounce's
     normal gradient (0 = fuse where the engine and regime allow; results
     are identical either way) */
  int32_t no_fuse;
  /* nullable: host array of ceil(W/tile) * ceil(H/tile) ranks, tile k owned
     by rank tile_owner[k] instead of k % world (the cost-balanced assignment
     of paper_2306_16142_b200/dist.py); read during the call only.  Which rank
     renders a pixel never changes its value (draws are addressed by global
     pixel index) */
  const int32_t* tile_owner;
  /* nullable, debug: DEVICE int32 buffer of stage_log_cap words receiving
     every compacted slot list of the render (the np.nonzero lists of
     render.py:225 and field.py:277).  Word 0 = words written after the
     2-word header, word 1 = 1 if a record did not fit.  Each record is
     {kind, bounce, step, s0, n_own, count, count slot ids}: kind 0 = primary
     march step, 1 = paths alive on entry to a bounce (after roulette; bucketed
     by object for composite fields), 2 = bounce-ray march step, 3 = the part
     of a bounce-ray march step 0 run by the fused trace+gradient kernel (kind
     2 of the same step holds the rest).  Slot id = (s - s0) * n_own + k for
     sample s of the wave starting at sample s0 and the k-th owned pixel.
     Setting it disables the CUDA-graph replay. */
  int32_t* stage_log;
  int64_t stage_log_cap;
} ddf_path_config_t;

typedef struct {
  /* render.RenderConfig fields used by render_depth / render_normal /
     render_shaded (render.py:106-124, 144-184) */
  int32_t mode;            /* 0 depth, 1 normal, 2 shaded                   */
  int32_t ambient;         /* shaded: flat albedo * env_radiance            */
  double background[3];
  double light_dir[3];     /* used as given (render.py:181)                 */
  double albedo, env_radiance;
} ddf_mode_config_t;

typedef struct {
  uint64_t forward_rows;   /* MLP forward rows evaluated (DDF queries)       */
  uint64_t gradient_rows;  /* MLP input-gradient rows (normals)             */
  uint64_t degenerate;     /* normals that fell back to -d (render.py:133)  */
  uint64_t path_samples;   /* owned pixels x spp                            */
  int32_t waves;
  uint64_t kernel_launches;     /* every kernel this call launched           */
  uint64_t forward_launches, gradient_launches;
  /* profile = 1 only: summed CUDA-event durations per kernel class */
  double ms_forward, ms_gradient, ms_compact, ms_other, ms_total;
  /* fused normal reuse: rows of the fused trace+gradient
     kernel (each a forward plus a backward chain), rows of the separate
     gradient pass actually executed (= gradient_rows when fusion is off; the
     reference's count of normal evaluations stays in gradient_rows), that
     kernel's launches and (profile = 1) time */
  uint64_t fused_rows, gradient_rows_executed, fused_launches;
  double ms_fused;
  /* per-stage row counts summed over spp (the lengths of the np.nonzero
     lists of render.py:225 and field.py:277): rows alive at primary march
     step j, rows alive on entry to bounce b (after roulette), and forward
     rows of bounce b's trace over all its march steps.  Steps and bounces
     past the array ends are not recorded. */
  uint64_t primary_march_rows[DDF_STAGE_STEPS];
  uint64_t bounce_alive_rows[DDF_STAGE_BOUNCES];
  uint64_t bounce_march_rows[DDF_STAGE_BOUNCES];
  /* profile = 1 only: the wavefront kernels of ms_other one by one
     (camera_kernel; roulette_kernel; bounce_kernel; after_primary_kernel +
     after_bounce_kernel; film_kernel) for their HBM roofline */
  double ms_camera, ms_roulette, ms_bounce, ms_after, ms_film;
  int32_t graph_replayed;  /* 1: this call replayed a captured CUDA graph     */
} ddf_render_stats_t;

/* NeuralField.__init__ (field.py:231-237): delta, AABB bounds (lo xyz, hi xyz). */
int ddf_field_create(double delta, const double bounds[6], int32_t precision, int32_t device,
                     ddf_field_t* out);
/* Adds one network.  MlpModel (neural.py:41-74) after effective_weights():
   `weights` = concatenation over layers of W_l (out, in) row-major float64,
   `biases` = concatenation of b_l.  HOST pointers.  center/scale/albedo are
   the EXTENSION object transform of config 5 (0, 1, unused for one net). */
int ddf_field_add_network(ddf_field_t f, const int32_t* widths, int32_t n_widths, const double* weights,
                          const double* biases, int32_t encoding, const double center[3], double scale,
                          double albedo);
int ddf_field_destroy(ddf_field_t f);
/* Switch the MLP engine of an existing field (DDF_PREC_*). */
int ddf_field_set_precision(ddf_field_t f, int32_t precision);
const char* ddf_last_error(void);

/* neural.forward_batch (neural.py:138-157) of network `net` on raw inputs
   x (n, widths[0]) -> out (n,) */
int ddf_mlp_forward(ddf_field_t f, int32_t net, const double* x, int64_t n, double* out, void* stream);
/* neural.input_gradient_batch (neural.py:229-249) -> out (n, widths[0]) */
int ddf_mlp_input_grad(ddf_field_t f, int32_t net, const double* x, int64_t n, double* out, void* stream);
/* NeuralField.query_batch (field.py:248-258): t (n,), hit (n,) uint8;
   pred (nullable) receives the raw network distance (config 1's output),
   obj (nullable) the min-composite object id */
int ddf_query(ddf_field_t f, const double* pos, const double* dirs, int64_t n, double* t, uint8_t* hit,
              double* pred, int32_t* obj, void* stream);
/* NeuralField.trace_batch (field.py:260-289): t (inf on miss), hit, obj (nullable) */
int ddf_trace(ddf_field_t f, const double* origins, const double* dirs, int64_t n, double* t, uint8_t* hit,
              int32_t* obj, void* stream);
/* NeuralField.normal_batch (field.py:295-317): t_hit and obj nullable;
   normals (n,3), valid (n,) uint8 */
int ddf_normal(ddf_field_t f, const double* origins, const double* dirs, const double* t_hit, const int32_t* obj,
               int64_t n, double* normals, uint8_t* valid, void* stream);
/* render.render_path (render.py:198-247): adds each owned pixel's radiance
   summed over spp (in sample order) into accum (W*H,) -- the caller divides
   by spp and replicates grey to RGB (render.py:244-247).  accum is zeroed
   first.  DDF_ENUMERIC on the normal sign rule (render.py:137-139). */
int ddf_render_path(ddf_field_t f, const ddf_camera_t* cam, const ddf_path_config_t* cfg, double* accum,
                    ddf_render_stats_t* stats, void* stream);

/* Exact triangle-mesh field: the reference's OracleField (field.py:191-200)
   over a TriangleMesh (mesh.py:19-67) with its BVH (mesh.py:94-166), built
   once from HOST arrays vertices (nv,3) f64 and faces (nf,3) int32.
   DDF_EDATA for an empty mesh or an out-of-range face index.  The handle
   works with ddf_query / ddf_trace (t, hit; obj receives the hit face id),
   ddf_normal (re-intersect, face normal, n . d < 0; t_hit and obj unused)
   and ddf_render_path (the BVH side of the paper's DDF-vs-BVH timing). */
int ddf_mesh_create(const double* vertices, int64_t n_vertices, const int32_t* faces, int64_t n_faces,
                    int32_t device, ddf_field_t* out);
/* mesh.intersect_rays (mesh.py:264-279) == _kernels.bvh_intersect_batch
   (_kernels.py:207-219): nearest hit with t in [t_min, t_max]; face -1 on a
   miss (t = inf, u = v = 0); ties on t go to the lower face index.  Device
   arrays; face/t/u/v nullable. */
int ddf_mesh_intersect(ddf_field_t f, const double* origins, const double* dirs, int64_t n, double t_min,
                       double t_max, int64_t* face, double* t, double* u, double* v, void* stream);

/* mesh.closest_distance (mesh.py:324-330) == _kernels.closest_dist_batch
   (_kernels.py:451-509): exact distance from each point (device (n,3) f64) to
   the mesh surface -> out (n,) f64.  OracleField.exact_distance. */
int ddf_mesh_closest(ddf_field_t f, const double* points, int64_t n, double* out, void* stream);

/* field.udf_many (field.py:418-488) for a neural backend: unsigned distance
   at n points (device (n,3) f64) = min over the n_dirs Halton sphere
   directions (field.py:126-141) of query_batch's t (+inf on a miss), then,
   when polish != 0, two rounds of golden-section search per angle
   (field.py:450-487).  out (n,) f64 device; +inf where every direction misses.
   n_dirs >= 1.  On a mesh handle (an exact backend) this is the exact
   closest-point distance, as udf_many's exact shortcut (field.py:431-433). */
int ddf_udf(ddf_field_t f, const double* points, int64_t n, int32_t n_dirs, int32_t polish, double* out,
            void* stream);
/* recon.udf_grid (recon.py:61-81): ddf_udf at the resolution^3 vertices of
   the grid over bbox = (lo x, y, z, hi x, y, z) (np.linspace per axis, C
   order, recon.py:53-58); out (resolution^3,) f64 device.  resolution >= 8. */
int ddf_udf_grid(ddf_field_t f, const double bbox[6], int32_t resolution, int32_t n_dirs, int32_t polish,
                 double* out, void* stream);

/* render.render_depth / render_normal / render_shaded (render.py:144-184)
   entirely on the device: pixel-centre rays (render.py:54-75), trace, the
   normals of the hit pixels (_hit_normals, render.py:127-141) and the shading.
   out: depth (H*W) f64, +inf on a miss; normal / shaded (H*W*3) f64 RGB, row
   major.  DDF_ENUMERIC on the normal sign rule. */
int ddf_render_mode(ddf_field_t f, const ddf_camera_t* cam, const ddf_mode_config_t* cfg, double* out, void* stream);

/* np.random.default_rng(...).random() draw k of a PCG64 stream given its
   (state, inc) (render.py:209,213,222): out[j] = draw idx[j] (device arrays). */
int ddf_rng_doubles(const uint64_t state[2], const uint64_t inc[2], const uint64_t* idx, int64_t n, double* out,
                    void* stream);
/* np.nonzero(flags) (field.py:277, render.py:225): ascending indices of the
   non-zero uint8 flags into list (device), count written to *count (device int32). */
int ddf_compact(const uint8_t* flags, int64_t n, int32_t* list, int32_t* count, void* stream);

/* Diagnostics: tcgen05 engine pipeline wait-cycle counters, collected when
   the environment variable DDF_DEBUG_UMMA has bit 1 set (16 u64 values). */
int ddf_debug_counters(uint64_t* out16, int32_t reset);
/* Diagnostics: the tcgen05 engines' event timeline of CTA 0 (builds with
   -DDDF_TRACE=1, empty otherwise): up to cap entries (clock64 << 16 | tag)
   copied to out (host); returns the count. */
int ddf_debug_trace(uint64_t* out, int32_t cap, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif
