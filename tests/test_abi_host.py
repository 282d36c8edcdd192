"""CPU-side checks: the C-ABI library builds, loads and exports every symbol
include/ddf_b200.h declares; host-side logic (DDFN I/O, camera, RNG seed
state, struct layouts) matches the reference.  No compute calls (no GPU)."""

import ctypes
import os
import re
import tempfile

import numpy as np
import pytest

from oracle import cpu_ddf as O
from paper_2306_16142_b200 import _lib
from paper_2306_16142_b200 import neural as N
from paper_2306_16142_b200.errors import DataError
from paper_2306_16142_b200 import render as R


def header_symbols():
    txt = open(_lib.HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(ddf_\w+)\(", txt, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_no_device_fails_loudly():
    """Without a GPU the product refuses to run (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    h = ctypes.c_void_p()
    b = (ctypes.c_double * 6)(-1, -1, -1, 1, 1, 1)
    rc = _lib.lib().ddf_field_create(1.0, b, 0, 0, ctypes.byref(h))
    assert rc == _lib.DDF_ECUDA
    assert b"no CUDA device" in _lib.lib().ddf_last_error()


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors == the C header's struct sizes and field offsets (gcc)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    src = tmp_path / "sz.c"
    fields = {"ddf_camera_t": _lib.Camera_t, "ddf_path_config_t": _lib.PathConfig_t,
              "ddf_render_stats_t": _lib.RenderStats_t, "ddf_mode_config_t": _lib.ModeConfig_t}
    body = []
    for cname, py in fields.items():
        body.append(f'printf("%zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            body.append(f'printf("%zu\\n", offsetof({cname}, {fname}));')
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ddf_b200.h"\nint main(){' + "".join(body) + "return 0;}")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.dirname(_lib.HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = []
    for py in fields.values():
        want.append(ctypes.sizeof(py))
        want += [getattr(py, f).offset for f, _ in py._fields_]
    assert got == want


def test_ddfn_roundtrip_matches_reference_bytes(golden):
    blob = golden["ddfn_bytes"].tobytes()
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "m.ddfn")
        open(p, "wb").write(blob)
        m, delta = N.load_model(p)
        q = os.path.join(td, "n.ddfn")
        N.save_model(m, delta, q)
        assert open(q, "rb").read() == blob
        for bad in (b"NOPE" + blob[4:], blob[:-8], blob + b"x", blob[:10]):
            open(q, "wb").write(bad)
            with pytest.raises(DataError):
                N.load_model(q)


def test_kaiming_matches_oracle():
    a = N.kaiming_uniform((65, 32, 1), 2)
    b = O.kaiming_uniform_net((65, 32, 1), 2)
    for x, y in zip(a.v + a.g, b.v + b.g):
        assert np.array_equal(x, y)
    assert N.encoding_of(a) == _lib.ENC_PE6


def test_camera_basis_and_structs_match_reference(golden):
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=24, height=16)
    oc = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=24, height=16)
    assert np.array_equal(cam.forward, oc.forward) and np.array_equal(cam.up_ortho, oc.up_ortho)
    c = R.camera_struct(cam)
    assert c.width == 24 and c.tan_half == np.tan(np.pi / 8)
    p = R.path_struct(R.RenderConfig(spp=3, bounces=2, seed=42))
    s, inc = O.pcg_seed_state(42)
    assert p.rng_state[0] + (p.rng_state[1] << 64) == s
    assert p.rng_inc[0] + (p.rng_inc[1] << 64) == inc


def test_render_config_validation():
    with pytest.raises(ValueError):
        R.RenderConfig(spp=0)
    with pytest.raises(ValueError):
        R.Camera(position=(0, 0, 0), look_at=(0, 0, 0))
