"""ctypes binding of libddf_b200.so (include/ddf_b200.h) and its build recipe.

The library is built in-tree (``paper_2306_16142_b200/lib/libddf_b200.so``)
with nvcc for sm_100a only.  There is no CPU fallback: every entry point of the
package fails loudly when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import DataError, DdfError, NumericError

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
# DDF_B200_LIB: load another build of the same library (A/B timing)
LIB_PATH = os.environ.get("DDF_B200_LIB") or os.path.join(LIB_DIR, "libddf_b200.so")
HEADER = os.path.join(ROOT, "include", "ddf_b200.h")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
OBJ_DIR = os.path.join(HERE, "build")   # objects of the default flags; DDF_NVCC_EXTRA builds go to build/<tag>

DDF_OK, DDF_EUSAGE, DDF_EDATA, DDF_ENUMERIC, DDF_ECUDA = 0, 1, 2, 3, 4
PREC_FP32, PREC_BF16, PREC_FP32_SIMT = 0, 1, 2
PRECISIONS = {"fp32": PREC_FP32, "bf16": PREC_BF16, "fp32_simt": PREC_FP32_SIMT}
ENC_RAW5, ENC_PE6 = 0, 1
STAGE_STEPS, STAGE_BOUNCES = 64, 32     # DDF_STAGE_STEPS, DDF_STAGE_BOUNCES

EXPORTS = ("ddf_field_create", "ddf_field_add_network", "ddf_field_destroy", "ddf_field_set_precision",
           "ddf_last_error", "ddf_mlp_forward", "ddf_mlp_input_grad", "ddf_query", "ddf_trace",
           "ddf_normal", "ddf_render_path", "ddf_render_mode", "ddf_mesh_create", "ddf_mesh_intersect", "ddf_mesh_closest", "ddf_udf", "ddf_udf_grid", "ddf_rng_doubles", "ddf_compact",
           "ddf_debug_counters", "ddf_debug_trace")


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile the CUDA sources into the in-tree shared library: every
    translation unit (ddf_api.cu and the engine units eng_*.cu) in parallel
    to build/*.o, then one nvcc link.  A unit is recompiled when it or any
    header is newer than its object."""
    units = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cu")] + [HEADER]
    newest_header = max(os.path.getmtime(p) for p in headers)
    os.makedirs(OBJ_DIR, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("DDF_NVCC_EXTRA", "").split()
    obj_dir = OBJ_DIR if not extra else os.path.join(OBJ_DIR, "_".join(x.strip("-").replace("=", "") for x in extra))
    os.makedirs(obj_dir, exist_ok=True)
    objs, jobs = [], []
    for u in units:
        src = os.path.join(CSRC, u)
        obj = os.path.join(obj_dir, u[:-3] + ".o")
        objs.append(obj)
        stale = force or not os.path.exists(obj) or os.path.getmtime(obj) < max(newest_header, os.path.getmtime(src))
        if stale:
            cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", src, "-o", obj + ".tmp"]
            jobs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    errors = []
    for obj, proc in jobs:
        out, _ = proc.communicate()
        if proc.returncode != 0:
            errors.append(out)
        else:
            os.replace(obj + ".tmp", obj)
            if verbose and out:
                print(out)
    if errors:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errors))
    if not jobs and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(o) for o in objs):
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    res = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", tmp],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Camera_t(ctypes.Structure):
    _fields_ = [("position", ctypes.c_double * 3), ("forward", ctypes.c_double * 3),
                ("right", ctypes.c_double * 3), ("up_ortho", ctypes.c_double * 3),
                ("tan_half", ctypes.c_double), ("aspect", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class PathConfig_t(ctypes.Structure):
    _fields_ = [("spp", ctypes.c_int32), ("bounces", ctypes.c_int32),
                ("albedo", ctypes.c_double), ("env_radiance", ctypes.c_double),
                ("rng_state", ctypes.c_uint64 * 2), ("rng_inc", ctypes.c_uint64 * 2),
                ("rr_start", ctypes.c_int32),
                ("rr_state", ctypes.c_uint64 * 2), ("rr_inc", ctypes.c_uint64 * 2),
                ("tile", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("max_wave_paths", ctypes.c_int64), ("profile", ctypes.c_int32), ("graph", ctypes.c_int32),
                ("no_fuse", ctypes.c_int32), ("tile_owner", ctypes.POINTER(ctypes.c_int32)),
                ("stage_log", ctypes.POINTER(ctypes.c_int32)), ("stage_log_cap", ctypes.c_int64)]


class ModeConfig_t(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("ambient", ctypes.c_int32), ("background", ctypes.c_double * 3),
                ("light_dir", ctypes.c_double * 3), ("albedo", ctypes.c_double), ("env_radiance", ctypes.c_double)]


class RenderStats_t(ctypes.Structure):
    _fields_ = [("forward_rows", ctypes.c_uint64), ("gradient_rows", ctypes.c_uint64),
                ("degenerate", ctypes.c_uint64), ("path_samples", ctypes.c_uint64),
                ("waves", ctypes.c_int32), ("kernel_launches", ctypes.c_uint64),
                ("forward_launches", ctypes.c_uint64), ("gradient_launches", ctypes.c_uint64),
                ("ms_forward", ctypes.c_double), ("ms_gradient", ctypes.c_double),
                ("ms_compact", ctypes.c_double), ("ms_other", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("fused_rows", ctypes.c_uint64), ("gradient_rows_executed", ctypes.c_uint64),
                ("fused_launches", ctypes.c_uint64), ("ms_fused", ctypes.c_double),
                ("primary_march_rows", ctypes.c_uint64 * STAGE_STEPS),
                ("bounce_alive_rows", ctypes.c_uint64 * STAGE_BOUNCES),
                ("bounce_march_rows", ctypes.c_uint64 * STAGE_BOUNCES),
                ("ms_camera", ctypes.c_double), ("ms_roulette", ctypes.c_double), ("ms_bounce", ctypes.c_double),
                ("ms_after", ctypes.c_double), ("ms_film", ctypes.c_double), ("graph_replayed", ctypes.c_int32)]


def stats_dict(st: RenderStats_t) -> dict:
    """ddf_render_stats_t as a dict; the per-stage arrays become lists."""
    out = {}
    for k, _ in RenderStats_t._fields_:
        v = getattr(st, k)
        out[k] = list(v) if isinstance(v, ctypes.Array) else v
    return out


_lib = None


def lib():
    """Load (building first if needed and possible) the shared library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    L.ddf_last_error.restype = ctypes.c_char_p
    L.ddf_field_create.argtypes = [ctypes.c_double, ctypes.POINTER(ctypes.c_double), i32, i32, ctypes.POINTER(vp)]
    L.ddf_field_add_network.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), i32, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), i32, ctypes.POINTER(ctypes.c_double),
                                        ctypes.c_double, ctypes.c_double]
    L.ddf_field_destroy.argtypes = [vp]
    L.ddf_field_set_precision.argtypes = [vp, i32]
    L.ddf_mlp_forward.argtypes = [vp, i32, dp, i64, dp, vp]
    L.ddf_mlp_input_grad.argtypes = [vp, i32, dp, i64, dp, vp]
    L.ddf_query.argtypes = [vp, dp, dp, i64, dp, dp, dp, dp, vp]
    L.ddf_trace.argtypes = [vp, dp, dp, i64, dp, dp, dp, vp]
    L.ddf_normal.argtypes = [vp, dp, dp, dp, dp, i64, dp, dp, vp]
    L.ddf_render_path.argtypes = [vp, ctypes.POINTER(Camera_t), ctypes.POINTER(PathConfig_t), dp,
                                  ctypes.POINTER(RenderStats_t), vp]
    L.ddf_rng_doubles.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64), dp, i64, dp, vp]
    L.ddf_compact.argtypes = [dp, i64, dp, dp, vp]
    L.ddf_udf.argtypes = [vp, dp, i64, i32, i32, dp, vp]
    L.ddf_render_mode.argtypes = [vp, ctypes.POINTER(Camera_t), ctypes.POINTER(ModeConfig_t), dp, vp]
    L.ddf_mesh_create.argtypes = [vp, i64, vp, i64, i32, ctypes.POINTER(vp)]
    L.ddf_mesh_closest.argtypes = [vp, dp, i64, dp, vp]
    L.ddf_mesh_intersect.argtypes = [vp, dp, dp, i64, ctypes.c_double, ctypes.c_double, dp, dp, dp, dp, vp]
    L.ddf_udf_grid.argtypes = [vp, ctypes.POINTER(ctypes.c_double), i32, i32, i32, dp, vp]
    L.ddf_debug_counters.argtypes = [ctypes.POINTER(ctypes.c_uint64), i32]
    L.ddf_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_uint64), i32, i32]
    for name in EXPORTS:
        if name != "ddf_last_error":
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a C status onto the reference's exception classes (errors.py:8-17)."""
    if rc == DDF_OK:
        return
    msg = lib().ddf_last_error().decode("utf-8", "replace")
    if rc == DDF_EUSAGE:
        raise ValueError(msg)
    if rc == DDF_EDATA:
        raise DataError(msg)
    if rc == DDF_ENUMERIC:
        raise NumericError(msg)
    raise DdfError(f"CUDA failure: {msg}")
