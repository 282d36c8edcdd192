"""CPU oracle for the DDF path-tracing hot path.  TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The shipped path
(``paper_2306_16142_b200``) never imports it and has no CPU fallback.

It is a float64 numpy restatement of the reference's hot path
(``/root/reference/pkg/src/ddfield``; paths below are relative to that
package).  Every function cites the reference lines it follows.  Where the
BASELINE configs ask for things the reference cannot express (65-D positional
encoding, Russian roulette, an 8-object min-composite scene) the restatement
extends the reference the way SURVEY.md Appendix A specifies; those parts are
marked EXTENSION and their parity is "parity with this restatement".

Pinning: ``tests/golden/make_golden.py`` runs the unmodified reference (it is
importable in the build container) and stores its outputs as fixtures;
``tests/test_oracle_golden.py`` checks this module against every fixture, and
against the live reference when ``/root/reference`` is present.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field as dc_field

import numpy as np

TWO_PI = 2.0 * np.pi
HIT_FRACTION = 0.98          # field.py:24  MISS_FRACTION
EVAL_CHUNK = 262_144         # neural.py:135 _EVAL_CHUNK
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645   # numpy PCG64 (XSL-RR 128/64) multiplier
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
RNG_TAG = 0x9A7              # render.py:209  default_rng([seed, 0x9A7])
RR_TAG = 0x5252              # EXTENSION: independent Russian-roulette stream
PE_OCTAVES = 6               # EXTENSION: configs 3-5 positional encoding


class OracleDataError(Exception):
    pass


class OracleNumericError(Exception):
    pass


# --------------------------------------------------------------------------
# weights (neural.py:41-95, 378-431)
# --------------------------------------------------------------------------

@dataclass
class Net:
    """One MLP as the reference stores it: V (out,in), g (out,), b (out,)."""
    widths: tuple
    v: list
    g: list
    b: list

    def effective(self):
        """neural.py:69-74  W = g * V / |V| row-wise, in float64."""
        out = []
        for v, g in zip(self.v, self.g):
            nrm = np.linalg.norm(v, axis=1)
            out.append(g[:, None] * v / nrm[:, None])
        return out

    @property
    def encoding(self) -> str:
        return "pe6" if self.widths[0] == 5 * (1 + 2 * PE_OCTAVES) else "raw5"


def kaiming_uniform_net(widths, seed: int) -> Net:
    """BASELINE configs' synthetic weights: per layer in
    order, V ~ U(+-sqrt(6/fan_in)) of shape (out, in) from default_rng(seed),
    g = |V| row norms (so W == V), b = 0."""
    rng = np.random.default_rng(seed)
    vs, gs, bs = [], [], []
    for i in range(len(widths) - 1):
        lim = np.sqrt(6.0 / widths[i])
        v = rng.uniform(-lim, lim, size=(widths[i + 1], widths[i]))
        vs.append(v)
        gs.append(np.linalg.norm(v, axis=1))
        bs.append(np.zeros(widths[i + 1]))
    return Net(tuple(int(w) for w in widths), vs, gs, bs)


def write_ddfn(net: Net, delta: float, path) -> None:
    """DDFN v1 layout (neural.py:378-390)."""
    blob = bytearray(b"DDFN")
    blob += struct.pack("<II", 1, len(net.widths))
    blob += struct.pack(f"<{len(net.widths)}I", *net.widths)
    blob += struct.pack("<d", float(delta))
    for v, g, b in zip(net.v, net.g, net.b):
        for a in (v, g, b):
            blob += np.ascontiguousarray(a, dtype="<f8").tobytes()
    with open(path, "wb") as fh:
        fh.write(bytes(blob))


def read_ddfn(path):
    """DDFN v1 reader with the reference's error cases (neural.py:393-431)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != b"DDFN":
        raise OracleDataError("not a DDFN checkpoint")
    try:
        ver, nw = struct.unpack_from("<II", blob, 4)
        if ver != 1:
            raise OracleDataError(f"unsupported checkpoint version {ver}")
        widths = struct.unpack_from(f"<{nw}I", blob, 12)
        (delta,) = struct.unpack_from("<d", blob, 12 + 4 * nw)
    except struct.error as exc:
        raise OracleDataError("truncated checkpoint header") from exc
    off = 20 + 4 * nw
    vs, gs, bs = [], [], []
    for i in range(nw - 1):
        o, n = widths[i + 1], widths[i]
        need = (o * n + 2 * o) * 8
        if off + need > len(blob):
            raise OracleDataError(f"truncated checkpoint (layer {i})")
        arr = np.frombuffer(blob, "<f8", count=o * n + 2 * o, offset=off)
        vs.append(arr[:o * n].reshape(o, n).copy())
        gs.append(arr[o * n:o * n + o].copy())
        bs.append(arr[o * n + o:].copy())
        off += need
    if off != len(blob):
        raise OracleDataError(f"{len(blob) - off} trailing bytes in checkpoint")
    return Net(tuple(widths), vs, gs, bs), float(delta)


# --------------------------------------------------------------------------
# angles and input encoding (field.py:69-112, neural.py:26-38)
# --------------------------------------------------------------------------

def dirs_to_angles(d):
    """field.py:77-82  (azimuth mod 2pi, polar from +z)."""
    d = np.atleast_2d(d)
    pol = np.arccos(np.clip(d[:, 2], -1.0, 1.0))
    az = np.arctan2(d[:, 1], d[:, 0]) % TWO_PI
    return np.stack([az, pol], axis=1)


def angles_to_dirs(a):
    """field.py:69-74."""
    a = np.atleast_2d(a)
    s = np.sin(a[:, 1])
    return np.stack([np.cos(a[:, 0]) * s, np.sin(a[:, 0]) * s, np.cos(a[:, 1])], axis=1)


def encode5(pos, ang):
    """neural.py:26-38: (x, y, z, az/pi - 1, 2*pol/pi - 1)."""
    pos = np.atleast_2d(pos)
    ang = np.atleast_2d(ang)
    u = np.empty((len(pos), 5))
    u[:, :3] = pos
    u[:, 3] = ang[:, 0] / np.pi - 1.0
    u[:, 4] = 2.0 * ang[:, 1] / np.pi - 1.0
    return u


def pe_encode(u):
    """EXTENSION (configs 3-5): 65-D sin/cos encoding of the
    five encoded inputs.  Column order (fixed, documented in DESIGN.md):
    [u_0..u_4, then for k = 0..5: sin(2^k pi u_0..4), cos(2^k pi u_0..4)]."""
    cols = [u]
    for k in range(PE_OCTAVES):
        arg = (2.0 ** k) * np.pi * u
        cols.append(np.sin(arg))
        cols.append(np.cos(arg))
    return np.concatenate(cols, axis=1)


def pe_chain(u, g65):
    """EXTENSION: d out / d u through pe_encode, given d out / d(65 inputs)."""
    g = g65[:, :5].copy()
    for k in range(PE_OCTAVES):
        f = (2.0 ** k) * np.pi
        arg = f * u
        base = 5 + 10 * k
        g += f * np.cos(arg) * g65[:, base:base + 5]
        g -= f * np.sin(arg) * g65[:, base + 5:base + 10]
    return g


def net_inputs(net: Net, u):
    return pe_encode(u) if net.encoding == "pe6" else u


# --------------------------------------------------------------------------
# MLP forward and input gradient (neural.py:138-157, 229-249)
# --------------------------------------------------------------------------

def mlp_forward(net: Net, x, ws=None):
    """neural.py:138-157 eval-mode forward: ReLU hidden layers, identity head,
    EVAL_CHUNK-row slabs."""
    x = np.atleast_2d(x)
    ws = net.effective() if ws is None else ws
    last = len(ws) - 1
    out = np.empty(len(x))
    for lo in range(0, len(x), EVAL_CHUNK):
        h = x[lo:lo + EVAL_CHUNK]
        for i, w in enumerate(ws):
            h = h @ w.T + net.b[i]
            if i != last:
                np.maximum(h, 0.0, out=h)
        out[lo:lo + EVAL_CHUNK] = h[:, 0]
    return out


def mlp_input_grad(net: Net, x, ws=None):
    """neural.py:229-249 generalised to any input width (the reference
    hard-codes 5 at neural.py:234): forward keeping ReLU masks, then
    d_h <- (d_h * mask) @ W down to the inputs."""
    x = np.atleast_2d(x)
    ws = net.effective() if ws is None else ws
    last = len(ws) - 1
    out = np.empty((len(x), x.shape[1]))
    for lo in range(0, len(x), EVAL_CHUNK):
        h = x[lo:lo + EVAL_CHUNK]
        masks = []
        for i, w in enumerate(ws):
            h = h @ w.T + net.b[i]
            if i != last:
                m = h > 0.0
                masks.append(m)
                h = h * m
        dh = np.ones((len(h), 1))
        for i in range(last, -1, -1):
            dz = dh if i == last else dh * masks[i]
            dh = dz @ ws[i]
        out[lo:lo + EVAL_CHUNK] = dh
    return out


def net_predict(net: Net, pos, ang, ws=None):
    """field.py:244-246 (_predict), plus the PE extension."""
    return mlp_forward(net, net_inputs(net, encode5(pos, ang)), ws)


def net_grad5(net: Net, pos, ang, ws=None):
    """field.py:291-293 (input_gradients) -> (N,5), plus the PE extension."""
    u = encode5(pos, ang)
    if net.encoding == "pe6":
        return pe_chain(u, mlp_input_grad(net, pe_encode(u), ws))
    return mlp_input_grad(net, u, ws)


# --------------------------------------------------------------------------
# the field: query / trace / normal (field.py:218-337)
# --------------------------------------------------------------------------

def ray_box(o, d, lo, hi):
    """field.py:323-337 vectorised slab test; enter > exit on a miss."""
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        t0 = (lo - o) * inv
        t1 = (hi - o) * inv
    a = np.minimum(t0, t1)
    b = np.maximum(t0, t1)
    z = d == 0.0
    if z.any():
        inside = (o >= lo) & (o <= hi)
        a = np.where(z, np.where(inside, -np.inf, np.inf), a)
        b = np.where(z, np.where(inside, np.inf, -np.inf), b)
    return a.max(axis=1), b.min(axis=1)


@dataclass
class Field:
    """A DDF backend: one network (the reference NeuralField, field.py:218-317)
    or, EXTENSION for config 5, several networks composed by min with
    per-object translation ``centers`` and uniform ``scale``."""
    nets: list
    delta: float
    bounds: np.ndarray = dc_field(default_factory=lambda: np.array([[-1.1] * 3, [1.1] * 3]))
    centers: np.ndarray | None = None
    scale: float = 1.0
    albedos: np.ndarray | None = None

    def __post_init__(self):
        self.bounds = np.asarray(self.bounds, dtype=np.float64)
        self._ws = [n.effective() for n in self.nets]
        if self.centers is None:
            self.centers = np.zeros((len(self.nets), 3))
        self.centers = np.asarray(self.centers, dtype=np.float64)
        self.normal_eval_backoff = 0.5 * self.delta      # field.py:237

    @property
    def composite(self) -> bool:
        return len(self.nets) > 1 or self.scale != 1.0 or bool(np.any(self.centers != 0.0))

    def predict(self, pos, ang):
        """Distance and object id.  Single net: field.py:244-246 exactly."""
        if not self.composite:
            return net_predict(self.nets[0], pos, ang, self._ws[0]), np.zeros(len(pos), np.int32)
        best = None
        obj = np.zeros(len(pos), np.int32)
        for j, net in enumerate(self.nets):
            dj = self.scale * net_predict(net, (pos - self.centers[j]) / self.scale, ang, self._ws[j])
            if best is None:
                best = dj
            else:
                take = dj < best
                obj[take] = j
                best = np.where(take, dj, best)
        return best, obj

    def grad5(self, pos, ang, obj):
        """field.py:291-293; composite: gradient of the object that was hit
        (d/dx of s*f((x-c)/s) = grad f)."""
        if not self.composite:
            return net_grad5(self.nets[0], pos, ang, self._ws[0])
        out = np.zeros((len(pos), 5))
        for j, net in enumerate(self.nets):
            sel = obj == j
            if sel.any():
                out[sel] = net_grad5(net, (pos[sel] - self.centers[j]) / self.scale, ang[sel], self._ws[j])
        return out

    # -- protocol ---------------------------------------------------------
    def query(self, pos, dirs):
        """field.py:248-258 query_batch: re-canonicalised angles, clamp,
        hit = clamp < 0.98 delta, t = max(clamp, 0)."""
        ang = dirs_to_angles(angles_to_dirs(dirs_to_angles(dirs)))
        pred, _ = self.predict(np.atleast_2d(pos), ang)
        c = np.clip(pred, -self.delta, self.delta)
        return np.maximum(c, 0.0), c < HIT_FRACTION * self.delta

    def trace(self, o, d, log=None):
        """field.py:260-289 sphere march with per-step np.nonzero compaction.
        Returns (t [inf on miss], hit, obj)."""
        o = np.atleast_2d(np.asarray(o, dtype=np.float64))
        d = np.atleast_2d(np.asarray(d, dtype=np.float64))
        n = len(o)
        ang = dirs_to_angles(d)
        te, tx = ray_box(o, d, self.bounds[0], self.bounds[1])
        alive = (te < tx) & (tx > 0.0)
        tacc = np.where(alive, np.maximum(te, 0.0), 0.0)
        tout = np.full(n, np.inf)
        hit = np.zeros(n, dtype=bool)
        obj = np.zeros(n, np.int32)
        step = 0.9 * self.delta
        thresh = HIT_FRACTION * self.delta
        diag = float(np.linalg.norm(self.bounds[1] - self.bounds[0]))
        for _ in range(int(np.ceil(diag / step)) + 4):
            if not alive.any():
                break
            idx = np.nonzero(alive)[0]
            if log is not None:
                log.append(idx.copy())
            p = o[idx] + tacc[idx, None] * d[idx]
            pred, oid = self.predict(p, ang[idx])
            c = np.clip(pred, -self.delta, self.delta)
            found = c < thresh
            sel = idx[found]
            tout[sel] = tacc[sel] + np.maximum(c[found], 0.0)
            hit[sel] = True
            obj[sel] = oid[found]
            alive[sel] = False
            tacc[idx[~found]] += step
            alive &= ~(alive & (tacc > tx))
        return tout, hit, obj

    def normal(self, o, d, t_hit=None, obj=None):
        """field.py:295-317: gradient at max(t - delta/2, 0) along the ray,
        normalised, flipped so n . d <= 0; |grad| < 1e-12 is invalid."""
        o = np.atleast_2d(o)
        d = np.atleast_2d(d)
        if t_hit is not None:
            back = np.maximum(np.asarray(t_hit) - self.normal_eval_backoff, 0.0)
            p = o + back[:, None] * d
        else:
            p = o
        if obj is None:
            obj = np.zeros(len(o), np.int32)
        g = self.grad5(p, dirs_to_angles(d), obj)[:, :3]
        nrm = np.linalg.norm(g, axis=1)
        valid = nrm >= 1e-12
        n = np.zeros_like(g)
        n[valid] = g[valid] / nrm[valid, None]
        dots = np.einsum("ij,ij->i", n, d)
        n[dots > 0.0] *= -1.0
        return n, valid


# --------------------------------------------------------------------------
# camera and sampling (render.py:22-75, 127-141, 187-195; field.py:103-112)
# --------------------------------------------------------------------------

@dataclass
class Cam:
    """render.py:22-51 pinhole camera."""
    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray = (0.0, 1.0, 0.0)
    vfov: float = np.pi / 3.0
    width: int = 256
    height: int = 256

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.look_at = np.asarray(self.look_at, dtype=np.float64)
        self.up = np.asarray(self.up, dtype=np.float64)
        f = self.look_at - self.position
        self.forward = f / np.linalg.norm(f)
        r = np.cross(self.forward, self.up)
        self.right = r / np.linalg.norm(r)
        self.up_ortho = np.cross(self.right, self.forward)


def camera_rays(cam: Cam, jitter, pix):
    """render.py:54-75 restricted to the global pixel indices ``pix``."""
    w, h = cam.width, cam.height
    px = (pix % w).astype(np.float64)
    py = (pix // w).astype(np.float64)
    tan_half = np.tan(cam.vfov / 2.0)
    aspect = w / h
    sx = (2.0 * (px + jitter[:, 0]) / w - 1.0) * tan_half * aspect
    sy = (1.0 - 2.0 * (py + jitter[:, 1]) / h) * tan_half
    d = cam.forward[None, :] + sx[:, None] * cam.right[None, :] + sy[:, None] * cam.up_ortho[None, :]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.broadcast_to(cam.position, d.shape).copy(), d


def frames(n):
    """field.py:103-112 smallest-component orthonormal frames."""
    axis = np.zeros((len(n), 3))
    axis[np.arange(len(n)), np.argmin(np.abs(n), axis=1)] = 1.0
    t1 = np.cross(n, axis)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    return t1, np.cross(n, t1)


def cosine_dirs(n, u):
    """render.py:187-195 cosine-weighted hemisphere about n."""
    r = np.sqrt(u[:, 0])
    phi = 2.0 * np.pi * u[:, 1]
    loc = np.stack([r * np.cos(phi), r * np.sin(phi), np.sqrt(np.maximum(0.0, 1.0 - u[:, 0]))], axis=1)
    t1, t2 = frames(n)
    return loc[:, 0, None] * t1 + loc[:, 1, None] * t2 + loc[:, 2, None] * n


def hit_normals(fld: Field, o, d, t, obj):
    """render.py:127-141 for an all-hit subset: degenerate -> -d, then the
    n . d < 0 sign rule raises."""
    n, valid = fld.normal(o, d, t_hit=t, obj=obj)
    bad = ~valid
    if bad.any():
        n[bad] = -d[bad]
    if not (np.einsum("ij,ij->i", n, d) < 0.0).all():
        raise OracleNumericError("normal sign rule violated: n . dir >= 0")
    return n


# --------------------------------------------------------------------------
# PCG64 (numpy's XSL-RR 128/64) as a counter-addressable stream
# --------------------------------------------------------------------------

def pcg_seed_state(seed: int, tag: int = RNG_TAG):
    """(state, inc) of numpy default_rng([seed, tag]) (render.py:209)."""
    st = np.random.PCG64(np.random.SeedSequence([seed, tag])).state["state"]
    return int(st["state"]), int(st["inc"])


def pcg_advance(state: int, inc: int, delta: int) -> int:
    """LCG jump-ahead: state after ``delta`` steps (O(log delta))."""
    am, ap, cm, cp = 1, 0, PCG_MULT, inc
    while delta > 0:
        if delta & 1:
            am = (am * cm) & M128
            ap = (ap * cm + cp) & M128
        cp = ((cm + 1) * cp) & M128
        cm = (cm * cm) & M128
        delta >>= 1
    return (am * state + ap) & M128


def pcg_output(state: int) -> int:
    """XSL-RR output of a post-step state."""
    hi, lo = state >> 64, state & M64
    x = hi ^ lo
    r = hi >> 58
    return ((x >> r) | (x << ((64 - r) & 63))) & M64


def pcg_double(seed_state, k: int) -> float:
    """Draw k (0-based) of the stream as numpy's Generator.random() makes it:
    (next64 >> 11) * 2^-53, next64 taken after k+1 steps."""
    s, inc = seed_state
    return (pcg_output(pcg_advance(s, inc, k + 1)) >> 11) * (1.0 / 9007199254740992.0)


def stream_block(seed: int, tag: int, k0: int, count: int):
    """``count`` consecutive doubles from draw index k0 (numpy advance)."""
    bg = np.random.PCG64(np.random.SeedSequence([seed, tag]))
    if k0:
        bg.advance(k0)
    return np.random.Generator(bg).random(count)


def draw_index(s: int, stage: int, n_pix: int, bounces: int) -> int:
    """first draw of (sample s, stage j) where stage 0 is the
    jitter and stage 1+b is bounce b; pixel i component c adds 2i + c."""
    return (s * (bounces + 1) + stage) * 2 * n_pix


# --------------------------------------------------------------------------
# the path tracer (render.py:198-247)
# --------------------------------------------------------------------------

@dataclass
class PathConfig:
    spp: int = 16
    bounces: int = 3
    albedo: float = 0.7
    env: float = 1.0
    seed: int = 0
    rr_start: int = -1          # EXTENSION: Russian roulette from this bounce index (-1 = off)


def render_path(fld: Field, cam: Cam, cfg: PathConfig, pix_range=None, log=None, pixels=None):
    """render.py:198-247 over the contiguous global pixel range ``pix_range``
    or the ascending pixel subset ``pixels`` (default: the whole film).  Random draws are addressed by global index so
    any range reproduces the full-frame stream.  Returns the (P,) grey value
    per pixel of the range (accum / spp, film summed in spp order).

    ``log`` (a list) receives, per spp, a dict with the ascending local
    indices alive at each primary march step ("primary_march"), alive on
    entry to each bounce ("bounce_alive"), and alive at each march step of
    each bounce's trace ("bounce_march", one list of steps per bounce), for
    compaction parity (render.py:225, field.py:277).
    EXTENSIONS: per-object albedo for composite fields; Russian roulette."""
    if cfg.bounces < 1:
        raise ValueError("path mode needs bounces >= 1")
    n_pix = cam.width * cam.height
    if pixels is not None:            # any ascending subset (e.g. one rank's tiles)
        pix = np.asarray(pixels, dtype=np.int64)
        i0, i1 = (int(pix.min()), int(pix.max()) + 1) if len(pix) else (0, 0)
    else:
        i0, i1 = (0, n_pix) if pix_range is None else pix_range
        pix = np.arange(i0, i1)
    P = len(pix)
    sel = pix - i0

    def block(tag, k0, per):
        """`per` draws per pixel for pixels i0..i1-1 from draw index k0, rows of pix."""
        b = stream_block(cfg.seed, tag, k0 + per * i0, per * (i1 - i0)).reshape(i1 - i0, per)
        return b[sel]
    accum = np.zeros(P)
    alb = None if fld.albedos is None else np.asarray(fld.albedos, dtype=np.float64)
    for s in range(cfg.spp):
        jit = block(RNG_TAG, draw_index(s, 0, n_pix, cfg.bounces), 2)
        o, d = camera_rays(cam, jit, pix)
        rad = np.zeros(P)
        thr = np.ones(P)
        tl = [] if log is not None else None
        t, hit, obj = fld.trace(o, d, tl)
        rad[~hit] = cfg.env
        alive = hit.copy()
        pos = o
        stages = []
        marches = []
        for b in range(cfg.bounces):
            u = block(RNG_TAG, draw_index(s, 1 + b, n_pix, cfg.bounces), 2)
            if cfg.rr_start >= 0 and b >= cfg.rr_start and alive.any():
                rr = block(RR_TAG, (s * cfg.bounces + b) * n_pix, 1)[:, 0]
                idx = np.nonzero(alive)[0]
                p = np.minimum(1.0, thr[idx])
                live = rr[idx] < p
                alive[idx[~live]] = False
                thr[idx[live]] = thr[idx[live]] / p[live]
            if not alive.any():
                continue
            idx = np.nonzero(alive)[0]
            if log is not None:
                stages.append(idx.copy())
            nrm = hit_normals(fld, pos[idx], d[idx], t[idx], obj[idx])
            hp = pos[idx] + t[idx, None] * d[idx] + 1e-6 * nrm
            thr[idx] *= cfg.albedo if alb is None else alb[obj[idx]]
            nd = cosine_dirs(nrm, u[idx])
            bl = [] if log is not None else None
            tn, hn, on = fld.trace(hp, nd, bl)
            if log is not None:
                marches.append([idx[j] for j in bl])
            esc = idx[~hn]
            rad[esc] += thr[esc] * cfg.env
            alive[esc] = False
            cont = idx[hn]
            pos[cont] = hp[hn]
            d[cont] = nd[hn]
            t[cont] = tn[hn]
            obj[cont] = on[hn]
            nxt = np.zeros(P, dtype=bool)
            nxt[cont] = True
            alive = nxt
        accum += rad
        if log is not None:
            log.append({"primary_march": tl, "bounce_alive": stages, "bounce_march": marches})
    return accum / cfg.spp


def stage_sequence(log):
    """The per-stage list lengths of a render_path log in the order the
    reference's render loop hands lists to the backend: (0, n) per march step
    (field.py:277), (1, n) per bounce's alive list (render.py:225)."""
    seq = []
    for rec in log:
        seq += [(0, len(lst)) for lst in rec["primary_march"]]
        for alive, steps in zip(rec["bounce_alive"], rec["bounce_march"]):
            seq.append((1, len(alive)))
            seq += [(0, len(lst)) for lst in steps]
    return seq


def film_rgb(value, cam: Cam):
    """render.py:244-247 grey -> (H, W, 3)."""
    return np.repeat(value[:, None], 3, axis=1).reshape(cam.height, cam.width, 3)


# --------------------------------------------------------------------------
# single-bounce render modes (render.py:144-184) for the GPU mode parity tests
# --------------------------------------------------------------------------

def render_mode(fld: Field, cam: Cam, mode: str, background=(0.0, 0.0, 0.0),
                light_dir=tuple(np.array([1.0, 1.0, 1.0]) / np.sqrt(3.0)), albedo=0.7, env=1.0, ambient=False,
                pixels=None):
    """render.py:144-184: "depth" -> (H, W) t (inf on miss); "normal" /
    "shaded" -> (H, W, 3).  Pixel-centre rays (render.py:62-63).  ``pixels``
    (ascending ids) renders only that subset and returns (P,) / (P, 3)."""
    pix = np.arange(cam.width * cam.height) if pixels is None else np.asarray(pixels, dtype=np.int64)
    n = len(pix)
    o, d = camera_rays(cam, np.full((n, 2), 0.5), pix)
    t, hit, obj = fld.trace(o, d)
    shape = (cam.height, cam.width) if pixels is None else (n,)
    if mode == "depth":
        return np.where(hit, t, np.inf).reshape(shape)
    nrm = np.zeros((n, 3))
    if hit.any():
        nrm[hit] = hit_normals(fld, o[hit], d[hit], t[hit], obj[hit])
    rgb = np.empty((n, 3))
    rgb[:] = np.asarray(background)
    if mode == "normal":
        rgb[hit] = 0.5 * (nrm[hit] + 1.0)
    elif ambient:
        rgb[hit] = albedo * env
    else:
        l = np.asarray(light_dir, dtype=np.float64)           # used as given (render.py:181)
        rgb[hit] = (albedo * np.maximum(nrm[hit] @ l, 0.0))[:, None]
    return rgb.reshape(shape + (3,))


# --------------------------------------------------------------------------
# unsigned distance from the DDF (field.py:115-141, 406-488; recon.py:53-72)
# --------------------------------------------------------------------------

GOLDEN = (np.sqrt(5.0) - 1.0) / 2.0      # field.py:406  _GOLDEN


def van_der_corput(idx, base: int):
    """field.py:115-123: radical inverse, digits accumulated low to high."""
    i = np.array(idx, dtype=np.int64)
    out = np.zeros(len(i))
    scale = 1.0 / base
    while (i > 0).any():
        out += scale * (i % base)
        i = i // base
        scale /= base
    return out


def sphere_directions(n: int):
    """field.py:126-141: Halton(2, 3) -> sphere (z = 1 - 2u, phi = 2 pi v)."""
    if n < 1:
        raise ValueError("need at least one direction")
    k = np.arange(1, n + 1)
    z = 1.0 - 2.0 * van_der_corput(k, 2)
    phi = TWO_PI * van_der_corput(k, 3)
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def _query_value(fld: Field, pos, dirs):
    """field.py:409-413 _eval_angles / 441-442: t on a hit, +inf on a miss."""
    t, hit = fld.query(pos, dirs)
    return np.where(hit, t, np.inf)


def udf_many(fld: Field, points, n_dirs: int = 512, polish: bool = True):
    """field.py:418-488 for a neural backend (exact_udf False).

    Stage 1: the minimum over the n_dirs sphere directions; ties resolve to the
    lowest direction index (the reference's chunked strict-< merge of per-chunk
    argmins yields exactly the global first argmin).  Stage 2 (polish): two
    rounds of golden-section search on the polar then azimuth angle, window
    +-3/sqrt(n_dirs) about the current best, 12 shrink steps, both probes
    re-evaluated every step, accepted only when strictly better."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    dirs = sphere_directions(n_dirs)
    n = len(pts)
    vals = _query_value(fld, np.repeat(pts, n_dirs, axis=0), np.tile(dirs, (n, 1))).reshape(n, n_dirs)
    arg = np.argmin(vals, axis=1)
    best = vals[np.arange(n), arg]
    if not polish:
        return best
    found = np.isfinite(best)
    if not found.any():
        return best
    p = pts[found]
    ang = dirs_to_angles(dirs[arg[found]])
    val = best[found].copy()
    half = 3.0 / np.sqrt(n_dirs)

    def probe(axis, x):
        a2 = np.empty_like(ang)
        a2[:, axis] = x
        a2[:, 1 - axis] = ang[:, 1 - axis]
        return _query_value(fld, p, angles_to_dirs(a2))

    for _ in range(2):
        for axis in (1, 0):
            lo, hi = ang[:, axis] - half, ang[:, axis] + half
            if axis == 1:
                lo, hi = np.clip(lo, 0.0, np.pi), np.clip(hi, 0.0, np.pi)
            x1, x2 = hi - GOLDEN * (hi - lo), lo + GOLDEN * (hi - lo)
            f1, f2 = probe(axis, x1), probe(axis, x2)
            for _ in range(12):
                right = f1 > f2
                lo = np.where(right, x1, lo)
                hi = np.where(right, hi, x2)
                x1, x2 = hi - GOLDEN * (hi - lo), lo + GOLDEN * (hi - lo)
                f1, f2 = probe(axis, x1), probe(axis, x2)
            xs = np.where(f1 < f2, x1, x2)
            fs = np.minimum(f1, f2)
            better = fs < val
            val[better] = fs[better]
            ang[better, axis] = xs[better]
    best[found] = val
    return best


def grid_points(bbox, resolution: int):
    """recon.py:53-58: per-axis linspace of the box corners, ij meshgrid,
    C order (z fastest)."""
    bbox = np.asarray(bbox, dtype=np.float64).reshape(2, 3)
    ax = np.linspace(bbox[0], bbox[1], resolution)
    x, y, z = np.meshgrid(ax[:, 0], ax[:, 1], ax[:, 2], indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)


def udf_grid(fld: Field, resolution: int = 64, n_dirs: int = 512, bounds=None, polish: bool = True):
    """recon.py:61-81: udf_many at every grid vertex -> (res, res, res)."""
    if resolution < 8:
        raise ValueError("resolution must be >= 8")
    box = np.asarray(bounds if bounds is not None else fld.bounds, dtype=np.float64).reshape(2, 3)
    return udf_many(fld, grid_points(box, resolution), n_dirs, polish).reshape((resolution,) * 3)


# --------------------------------------------------------------------------
# exact triangle-mesh field (field.py:144-200, mesh.py:264-279, _kernels.py:43-147)
# --------------------------------------------------------------------------

DET_EPS = 1e-9               # _kernels.py:16


def ray_tri(o, d, a, b, c):
    """_kernels.py:43-77 Moller-Trumbore, elementwise over broadcast arrays in
    the reference's operation order.  Returns (t, u, v); t = inf on a miss."""
    e1 = [b[..., k] - a[..., k] for k in range(3)]
    e2 = [c[..., k] - a[..., k] for k in range(3)]
    dx, dy, dz = d[..., 0], d[..., 1], d[..., 2]
    hx = dy * e2[2] - dz * e2[1]
    hy = dz * e2[0] - dx * e2[2]
    hz = dx * e2[1] - dy * e2[0]
    det = e1[0] * hx + e1[1] * hy + e1[2] * hz
    ok = ~((-DET_EPS < det) & (det < DET_EPS))
    with np.errstate(divide="ignore", invalid="ignore"):
        f = 1.0 / det
        sx, sy, sz = o[..., 0] - a[..., 0], o[..., 1] - a[..., 1], o[..., 2] - a[..., 2]
        u = f * (sx * hx + sy * hy + sz * hz)
        ok &= ~((u < 0.0) | (u > 1.0))
        qx = sy * e1[2] - sz * e1[1]
        qy = sz * e1[0] - sx * e1[2]
        qz = sx * e1[1] - sy * e1[0]
        v = f * (dx * qx + dy * qy + dz * qz)
        ok &= ~((v < 0.0) | (u + v > 1.0))
        t = f * (e2[0] * qx + e2[1] * qy + e2[2] * qz)
    return np.where(ok, t, np.inf), np.where(ok, u, 0.0), np.where(ok, v, 0.0)


class MeshField:
    """The reference's exact mesh backend (BruteForceField semantics, equal to
    OracleField): every query scans all faces; nearest t in [t_min, t_max],
    ties to the lower face index (_kernels.py:130-147)."""

    composite = False
    albedos = None

    def __init__(self, vertices, faces, chunk: int = 1 << 22):
        self.vertices = np.asarray(vertices, dtype=np.float64)
        self.faces = np.asarray(faces, dtype=np.int32)
        lo, hi = self.vertices.min(axis=0), self.vertices.max(axis=0)
        diag = float(np.linalg.norm(hi - lo))
        self.bounds = np.stack([lo - diag, hi + diag])                  # field.py:154-157
        self.grid_bounds = np.stack([lo - 0.05 * diag, hi + 0.05 * diag])
        tri = self.vertices[self.faces]
        self._a, self._b, self._c = tri[:, 0], tri[:, 1], tri[:, 2]
        self._chunk = chunk

    def intersect(self, o, d, t_min=0.0, t_max=np.inf):
        """mesh.intersect_rays (mesh.py:264-279) -> (face, t, u, v)."""
        o = np.atleast_2d(np.asarray(o, dtype=np.float64))
        d = np.atleast_2d(np.asarray(d, dtype=np.float64))
        n, m = len(o), len(self.faces)
        face = np.full(n, -1, np.int64)
        t_out, u_out, v_out = np.full(n, np.inf), np.zeros(n), np.zeros(n)
        step = max(1, self._chunk // max(m, 1))
        for s in range(0, n, step):
            oo, dd = o[s:s + step, None, :], d[s:s + step, None, :]
            t, u, v = ray_tri(oo, dd, self._a[None], self._b[None], self._c[None])
            t = np.where((t_min <= t) & (t <= t_max), t, np.inf)
            k = np.argmin(t, axis=1)                 # first minimum = lowest face index
            r = np.arange(len(k))
            tk = t[r, k]
            hit = np.isfinite(tk)
            face[s:s + step] = np.where(hit, k, -1)
            t_out[s:s + step] = tk
            u_out[s:s + step] = np.where(hit, u[r, k], 0.0)
            v_out[s:s + step] = np.where(hit, v[r, k], 0.0)
        return face, t_out, u_out, v_out

    def query(self, pos, dirs):
        """field.py:161-165."""
        face, t, _, _ = self.intersect(pos, dirs)
        return t, face >= 0

    def trace(self, o, d, log=None):
        """field.py:168 (trace_batch = query_batch); obj = the hit face."""
        face, t, _, _ = self.intersect(o, d)
        return t, face >= 0, face.astype(np.int32)

    def normal(self, o, d, t_hit=None, obj=None):
        """field.py:172-189: re-intersect, face normal, flipped so n . d <= 0."""
        d = np.atleast_2d(d)
        face, _, _, _ = self.intersect(o, d)
        valid = face >= 0
        n = np.zeros((len(d), 3))
        if valid.any():
            fv = self.faces[face[valid]]
            v = self.vertices
            nn = np.cross(v[fv[:, 1]] - v[fv[:, 0]], v[fv[:, 2]] - v[fv[:, 0]])
            nn /= np.linalg.norm(nn, axis=1, keepdims=True)
            dots = np.einsum("ij,ij->i", nn, d[valid])
            nn[dots > 0.0] *= -1.0
            n[valid] = nn
        return n, valid


def point_tri_dist_sq(p, a, b, c):
    """_kernels.py:363-424 (Ericson's closest-point region tests) elementwise
    over broadcast arrays, the first matching region in the reference's order."""
    with np.errstate(divide="ignore", invalid="ignore"):
        ab, ac, ap = b - a, c - a, p - a
        dot = lambda u, v: u[..., 0] * v[..., 0] + u[..., 1] * v[..., 1] + u[..., 2] * v[..., 2]  # noqa: E731
        d1, d2 = dot(ab, ap), dot(ac, ap)
        bp = p - b
        d3, d4 = dot(ab, bp), dot(ac, bp)
        vc = d1 * d4 - d3 * d2
        cp = p - c
        d5, d6 = dot(ab, cp), dot(ac, cp)
        vb = d5 * d2 - d1 * d6
        va = d3 * d6 - d5 * d4
        e1, e2 = d4 - d3, d5 - d6

        def frac(num, den):
            return np.where(den != 0.0, num / np.where(den != 0.0, den, 1.0), 0.0)

        w_ab = frac(d1, d1 - d3)[..., None]
        w_ac = frac(d2, d2 - d6)[..., None]
        w_bc = frac(e1, e1 + e2)[..., None]
        denom = va + vb + vc
        v_in = vb / np.where(denom == 0.0, 1.0, denom)
        w_in = vc / np.where(denom == 0.0, 1.0, denom)
        cands = [
            (d1 <= 0.0) & (d2 <= 0.0), dot(ap, ap),
            (d3 >= 0.0) & (d4 <= d3), dot(bp, bp),
            (vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0), None,
            (d6 >= 0.0) & (d5 <= d6), dot(cp, cp),
            (vb <= 0.0) & (d2 >= 0.0) & (d6 <= 0.0), None,
            (va <= 0.0) & (e1 >= 0.0) & (e2 >= 0.0), None,
            denom == 0.0, dot(ap, ap),
        ]
        e = ap - w_ab * ab
        cands[5] = dot(e, e)
        e = ap - w_ac * ac
        cands[9] = dot(e, e)
        e = bp - w_bc * (c - b)
        cands[11] = dot(e, e)
        e = ap - v_in[..., None] * ab - w_in[..., None] * ac
        out = dot(e, e)
        for k in range(len(cands) - 2, -1, -2):
            out = np.where(cands[k], cands[k + 1], out)
    return out


def _mesh_closest(self, points):
    """mesh.closest_distance (mesh.py:324-330) by a linear scan
    (_kernels.linear_closest_batch, _kernels.py:512-531)."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    out = np.empty(len(pts))
    step = max(1, self._chunk // max(len(self.faces), 1))
    for s in range(0, len(pts), step):
        d = point_tri_dist_sq(pts[s:s + step, None, :], self._a[None], self._b[None], self._c[None])
        out[s:s + step] = np.sqrt(d.min(axis=1))
    return out


MeshField.exact_distance = _mesh_closest
