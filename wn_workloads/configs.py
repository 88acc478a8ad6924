"""Seeded synthetic workloads C1..C5 in the libwn ABI layout.

This module is the ONE piece shared by the CPU oracle side and the CUDA side:
it only *constructs* inputs (control points, weights, CSR offsets, query
points) and holds none of the winding-number arithmetic of the method.  The
datasets of the paper (OpenClipArt20K, the BG dataset, CAD models; PAPER.md
§5.2, §5.4) are not in the container; these configs
stand in for them with the shapes/sizes/distributions recorded in DESIGN.md
("Input recipe") and in BASELINE.json `configs`.

Layout of a workload dict (all numpy, C-contiguous):
  ctrl_uv       float64 [n_ctrl, 2]   packed control points, stored coords
  ctrl_w        float64 [n_ctrl] or None (polynomial)
  seg_degree    int32   [n_segs]      1..5; ctrl offsets = excl. scan of deg+1
  loop_seg_off  int32   [n_loops+1]   CSR, segment order = loop orientation
  face_loop_off int32   [n_faces+1]   CSR
  face_periodic uint8   [n_faces]     bit0 = periodic in u, bit1 = in v
  face_domain   float64 [n_faces, 4]  (u0, Tu, v0, Tv)
  face_id       int32   [nq]
  uv            float64 [nq, 2]
  meta          dict    generator-side facts used by analytic pins

Periodic faces (C3, C3pq, the periodic C5 faces) come in two storage modes:
  exact=True  (default) every control point and the periods are quantised to
              the dyadic grid 2^-40 (Q40).  All lattice translates x + k*T are
              then exact in double arithmetic, so lifting and copy emission
              reproduce junction points bit-for-bit (reading R25).
  exact=False generic fp64 data: T = 2*pi (and pi) as plain doubles, control
              points unquantised.  Storing a segment translated by -k*T and
              lifting it back by +k*T rounds, so the junctions at seam
              crossings are NOT bit-continuous after lifting (the chain-break
              path of the library, reading R25).
Loops are stored seam-discontinuously: each segment is translated
by the lattice vector that puts its first control point into the fundamental
domain.
"""
from __future__ import annotations

import math

import numpy as np

Q40 = 2.0 ** -40


def quant(x):
    """Round to the 2^-40 dyadic grid (exact-translate grid for periodic faces)."""
    return np.round(np.asarray(x, dtype=np.float64) / Q40) * Q40


TWO_PI_Q = float(quant(2.0 * math.pi))   # quantised period used for "2*pi" domains
PI_Q = float(quant(math.pi))


def _qz(exact):
    """Coordinate rounding of a periodic generator: Q40 (exact=True) or none."""
    if exact:
        return quant
    return lambda x: np.asarray(x, dtype=np.float64)


def _periods(exact):
    """(2*pi, pi): Q40-quantised (exact=True) or the plain doubles."""
    return (TWO_PI_Q, PI_Q) if exact else (2.0 * math.pi, math.pi)

EPS_FP64 = 1e-10
EPS_FP32 = 1e-6


class _Builder:
    """Accumulates segments/loops/faces into the ABI arrays."""

    def __init__(self):
        self.ctrl = []
        self.w = []
        self.deg = []
        self.loop_off = [0]
        self.face_loop_off = [0]
        self.face_periodic = []
        self.face_domain = []
        self.n_loops = 0

    def seg(self, P, w=None):
        P = np.asarray(P, dtype=np.float64)
        n = P.shape[0] - 1
        assert 1 <= n <= 5
        self.ctrl.append(P)
        self.w.append(np.ones(n + 1) if w is None else np.asarray(w, dtype=np.float64))
        self.deg.append(n)

    def end_loop(self):
        self.loop_off.append(len(self.deg))
        self.n_loops += 1

    def end_face(self, periodic=0, domain=(0.0, 1.0, 0.0, 1.0)):
        self.face_loop_off.append(self.n_loops)
        self.face_periodic.append(periodic)
        self.face_domain.append(domain)

    def arrays(self, rational=True):
        ctrl = np.ascontiguousarray(np.concatenate(self.ctrl, axis=0))
        w = np.ascontiguousarray(np.concatenate(self.w)) if rational else None
        return dict(
            ctrl_uv=ctrl,
            ctrl_w=w,
            seg_degree=np.asarray(self.deg, dtype=np.int32),
            loop_seg_off=np.asarray(self.loop_off, dtype=np.int32),
            face_loop_off=np.asarray(self.face_loop_off, dtype=np.int32),
            face_periodic=np.asarray(self.face_periodic, dtype=np.uint8),
            face_domain=np.ascontiguousarray(np.asarray(self.face_domain, dtype=np.float64).reshape(-1, 4)),
        )


# ----------------------------------------------------------------------------
# small geometric helpers (input construction only)
# ----------------------------------------------------------------------------

def _bern_eval(P, w, t):
    """Rational Bezier point and derivative by the Bernstein basis (input recipe only:
    used to place C2's near-curve queries).  Independent of the oracle's de Casteljau."""
    n = P.shape[0] - 1
    t = np.asarray(t, dtype=np.float64)[:, None]
    B = np.stack([math.comb(n, j) * t[:, 0] ** j * (1 - t[:, 0]) ** (n - j) for j in range(n + 1)], 1)
    Xh = B @ (w[:, None] * P)
    Wh = B @ w
    if n >= 1:
        Bd = np.stack([math.comb(n - 1, j) * t[:, 0] ** j * (1 - t[:, 0]) ** (n - 1 - j) for j in range(n)], 1)
        dX = n * Bd @ (w[1:, None] * P[1:] - w[:-1, None] * P[:-1])
        dW = n * Bd @ (w[1:] - w[:-1])
    pt = Xh / Wh[:, None]
    d = (dX * Wh[:, None] - Xh * dW[:, None]) / (Wh ** 2)[:, None]
    return pt, d


def _perp(v):
    return np.stack([-v[..., 1], v[..., 0]], -1)


def _star_segments(rng, V, degs, jit_frac, rational):
    """Segments V_k -> V_{k+1} (cyclic) with degree degs[k]; interior control points
    on the edge plus a perpendicular jitter U(-jit_frac, jit_frac) * perp(edge).
    Junctions reuse the same V entries, so shared endpoints are bit-identical.
    Vectorised per degree; the random stream is consumed exactly as the
    per-segment form (jitter of segment k, then its weights, k = 0, 1, ...):
    uniform(low, high) = low + (high - low) * next_double."""
    n = V.shape[0]
    degs = np.asarray(degs, dtype=np.int64)
    cj = np.where(degs >= 2, degs - 1, 0)
    cw = degs + 1 if rational else np.zeros_like(degs)
    off = np.concatenate([[0], np.cumsum(cj + cw)])
    U = rng.random(int(off[-1]))
    A = V
    B = V[(np.arange(n) + 1) % n]
    E = B - A
    prp = _perp(E)
    out = [None] * n
    jlo, jsc = -jit_frac, jit_frac - (-jit_frac)
    wlo, wsc = 0.5, 2.0 - 0.5
    for d in np.unique(degs):
        d = int(d)
        ks = np.nonzero(degs == d)[0]
        jj = (np.arange(d + 1) / d)[None, :, None]
        P = A[ks, None, :] + jj * E[ks, None, :]
        if d >= 2:
            u = U[off[ks][:, None] + np.arange(d - 1)[None, :]]              # [m, d-1]
            P[:, 1:d] += (jlo + jsc * u)[:, :, None] * prp[ks, None, :]
        P[:, 0] = A[ks]
        P[:, d] = B[ks]
        if rational:
            W = wlo + wsc * U[off[ks][:, None] + cj[ks][:, None] + np.arange(d + 1)[None, :]]
        else:
            W = np.ones((len(ks), d + 1))
        for i, k in enumerate(ks):
            out[k] = (P[i], W[i])
    return out


def _star_vertices(rng, center, r_mean, r_jit, n, cw):
    ang = 2.0 * math.pi * np.arange(n) / n
    rad = r_mean + rng.uniform(-r_jit, r_jit, size=n)
    V = np.stack([center[0] + rad * np.cos(ang), center[1] + rad * np.sin(ang)], 1)
    return V[::-1].copy() if cw else V


def _circle_arcs(c, r, ccw=True):
    """Exact circle as 4 rational quadratic arcs, weights (1, sqrt(2)/2, 1)."""
    c = np.asarray(c, dtype=np.float64)
    E = [np.array([r, 0.0]), np.array([0.0, r]), np.array([-r, 0.0]), np.array([0.0, -r])]
    Cn = [np.array([r, r]), np.array([-r, r]), np.array([-r, -r]), np.array([r, -r])]
    arcs = []
    for k in range(4):
        P = np.stack([c + E[k], c + Cn[k], c + E[(k + 1) % 4]])
        arcs.append(P)
    w = np.array([1.0, math.sqrt(0.5), 1.0])
    if not ccw:
        arcs = [a[::-1].copy() for a in arcs[::-1]]
    return [(a, w.copy()) for a in arcs]


def _wrap_store(P, T_u, T_v, per_u, per_v, u0=0.0, v0=0.0, jit=None):
    """Store a lifted segment seam-discontinuously (R18): translate by the lattice
    vector that puts its first control point into [u0,u0+T) on periodic axes,
    plus (jit = (rng, K)) a random extra lattice vector in [-K, K]^2 -- any
    translate is valid storage (R18).  Exact for Q40-quantised coordinates and
    periods; rounds once per coordinate otherwise."""
    P = P.copy()
    if per_u:
        k = math.floor((P[0, 0] - u0) / T_u)
        if jit is not None:
            k += int(jit[0].integers(-jit[1], jit[1] + 1))
        P[:, 0] = P[:, 0] - k * T_u
    if per_v:
        k = math.floor((P[0, 1] - v0) / T_v)
        if jit is not None:
            k += int(jit[0].integers(-jit[1], jit[1] + 1))
        P[:, 1] = P[:, 1] - k * T_v
    return P


def _jit(seed, store_jitter):
    """Storage-translate jitter source (its own stream: the geometry stays the
    same whatever the jitter)."""
    return None if not store_jitter else (np.random.Generator(np.random.PCG64(10_000 + seed)), int(store_jitter))


def _graph_loop(rng, f, u_start, T, direction, n_seg, degs, rational, qz=quant):
    """Non-contractible loop following v = f(u) over one period, as Bezier segments
    whose control points sample the graph (monotone u => a graph).  direction=+1
    rightward (class (1,0)), -1 leftward (class (-1,0)).  qz = quant: all points
    Q40-quantised, the loop end equals start + direction*T exactly; otherwise
    the end is start + direction*T rounded once."""
    knots_u = qz(u_start + direction * T * np.arange(n_seg + 1) / n_seg)
    knots_u[-1] = qz(u_start) + direction * T          # closure (exact in Q40 arithmetic)
    knots_v = qz(f(knots_u))
    knots_v[-1] = knots_v[0]
    segs = []
    for k in range(n_seg):
        d = int(degs[k])
        ua, ub = knots_u[k], knots_u[k + 1]
        us = ua + (ub - ua) * np.arange(d + 1) / d
        P = np.stack([qz(us), qz(f(us))], 1)
        P[0] = (ua, knots_v[k])
        P[d] = (ub, knots_v[k + 1])
        w = rng.uniform(0.5, 2.0, size=d + 1) if rational else np.ones(d + 1)
        segs.append((P, w))
    return segs


def _hermite_graph_loop(f, fp, u_start, T, direction, n_seg, qz=quant):
    """Cubic Hermite fit to v = f(u) over one period (C3 separation loops)."""
    knots_u = qz(u_start + direction * T * np.arange(n_seg + 1) / n_seg)
    knots_u[-1] = qz(u_start) + direction * T
    knots_v = qz(f(knots_u))
    knots_v[-1] = knots_v[0]
    segs = []
    for k in range(n_seg):
        ua, ub = knots_u[k], knots_u[k + 1]
        h = ub - ua
        P0 = np.array([ua, knots_v[k]])
        P3 = np.array([ub, knots_v[k + 1]])
        P1 = qz(P0 + (h / 3.0) * np.array([1.0, fp(ua)]))
        P2 = qz(P3 - (h / 3.0) * np.array([1.0, fp(ub)]))
        segs.append((np.stack([P0, P1, P2, P3]), np.ones(4)))
    return segs


def _grid(lo, hi, n=64):
    """Cell-centred n x n grid, row-major (v outer, u inner)."""
    us = lo[0] + (np.arange(n) + 0.5) * ((hi[0] - lo[0]) / n)
    vs = lo[1] + (np.arange(n) + 0.5) * ((hi[1] - lo[1]) / n)
    U, Vv = np.meshgrid(us, vs)
    return np.stack([U.ravel(), Vv.ravel()], 1)


def _finish(b, face_id, uv, rational, name, meta, eps=EPS_FP64):
    d = b.arrays(rational=rational)
    d["face_id"] = np.ascontiguousarray(face_id, dtype=np.int32)
    d["uv"] = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
    d["name"] = name
    d["eps"] = eps
    d["meta"] = meta
    return d


# ----------------------------------------------------------------------------
# C1 — single planar face, 8-cubic jittered circle (BASELINE configs[0])
# ----------------------------------------------------------------------------

def gen_c1(seed=1, n_queries=10_000):
    rng = np.random.Generator(np.random.PCG64(seed))
    c = np.array([0.5, 0.5])
    r = 0.35
    h = (4.0 / 3.0) * math.tan(math.pi / 16.0) * r
    a = 2.0 * math.pi * np.arange(8) / 8
    E = c + r * np.stack([np.cos(a), np.sin(a)], 1)
    tang = np.stack([-np.sin(a), np.cos(a)], 1)
    Hp = E + h * tang           # outgoing handles
    Hm = E - h * tang           # incoming handles

    def jitter(q):
        d = q - c
        rho = np.hypot(d[..., 0], d[..., 1])
        beta = np.arctan2(d[..., 1], d[..., 0])
        rho = rho + rng.uniform(-0.05, 0.05, size=rho.shape)
        return c + rho[..., None] * np.stack([np.cos(beta), np.sin(beta)], -1)

    E, Hp, Hm = jitter(E), jitter(Hp), jitter(Hm)
    b = _Builder()
    for k in range(8):
        b.seg(np.stack([E[k], Hp[k], Hm[(k + 1) % 8], E[(k + 1) % 8]]))
    b.end_loop()
    b.end_face()
    uv = rng.uniform(0.0, 1.0, size=(n_queries, 2))
    meta = dict(star_centers=[(0.5, 0.5)], kind="C1")
    return _finish(b, np.zeros(n_queries), uv, False, "C1", meta)


# ----------------------------------------------------------------------------
# C2 — rational face with 4 holes, 10% near-curve queries (BASELINE configs[1])
# ----------------------------------------------------------------------------

def gen_c2(seed=2, n_queries=1_000_000, near_frac=0.10, near_off=1e-6):
    rng = np.random.Generator(np.random.PCG64(seed))
    c = np.array([0.5, 0.5])
    b = _Builder()
    allsegs = []
    centers = [tuple(c)]
    V = _star_vertices(rng, c, 0.40, 0.04, 32, cw=False)
    segs = _star_segments(rng, V, rng.integers(2, 6, size=32), 0.1, True)
    for P, w in segs:
        b.seg(P, w)
    b.end_loop()
    allsegs += segs
    for sx, sy in ((-1, -1), (1, -1), (1, 1), (-1, 1)):
        hc = c + 0.15 * np.array([sx, sy])
        centers.append(tuple(hc))
        V = _star_vertices(rng, hc, 0.07, 0.01, 12, cw=True)
        segs = _star_segments(rng, V, rng.integers(2, 6, size=12), 0.1, True)
        for P, w in segs:
            b.seg(P, w)
        b.end_loop()
        allsegs += segs
    b.end_face()
    outer = np.concatenate([P for P, _ in allsegs[:32]])
    lo, hi = outer.min(0), outer.max(0)
    n_near = int(round(n_queries * near_frac))
    n_uni = n_queries - n_near
    uv_u = lo + (hi - lo) * rng.uniform(0.0, 1.0, size=(n_uni, 2))
    si = rng.integers(0, len(allsegs), size=n_near)
    ts = rng.uniform(0.0, 1.0, size=n_near)
    off = rng.uniform(-near_off, near_off, size=n_near)
    uv_n = np.empty((n_near, 2))
    for s in np.unique(si):
        m = si == s
        P, w = allsegs[s]
        pt, d = _bern_eval(P, w, ts[m])
        nrm = _perp(d) / np.hypot(d[:, 0], d[:, 1])[:, None]
        uv_n[m] = pt + off[m, None] * nrm
    uv = np.concatenate([uv_u, uv_n])
    near = np.concatenate([np.zeros(n_uni, bool), np.ones(n_near, bool)])
    perm = rng.permutation(n_queries)
    meta = dict(star_centers=centers, near_mask=near[perm], kind="C2")
    return _finish(b, np.zeros(n_queries), uv[perm], True, "C2", meta)


# ----------------------------------------------------------------------------
# C3 — bi-periodic torus face (BASELINE configs[2]); layout = SURVEY R21
# ----------------------------------------------------------------------------

def gen_c3(seed=3, n_queries=1_000_000, exact=True, store_jitter=0):
    rng = np.random.Generator(np.random.PCG64(seed))
    T, PI_ = _periods(exact)
    qz = _qz(exact)
    b = _Builder()
    ph_a, ph_b = rng.uniform(0, 2 * math.pi, size=2)
    fa = lambda u: 4.6 + 0.3 * np.sin(u + ph_a)
    fpa = lambda u: 0.3 * math.cos(u + ph_a)
    fb = lambda u: T + 1.7 + 0.3 * np.sin(u + ph_b)      # lifted above alpha
    fpb = lambda u: 0.3 * math.cos(u + ph_b)
    ua = float(qz(rng.uniform(math.pi, 2 * math.pi)))
    ub = float(qz(rng.uniform(math.pi, 2 * math.pi)))
    loops = []
    loops.append(("alpha", _hermite_graph_loop(fa, fpa, ua, T, +1, 24, qz)))
    loops.append(("beta", _hermite_graph_loop(fb, fpb, ub, T, -1, 24, qz)))
    loops.append(("H1", [(qz(P), w) for P, w in _circle_arcs(qz([0.0, 0.0]), float(qz(0.6)), ccw=False)]))
    loops.append(("H2", [(qz(P), w) for P, w in _circle_arcs(qz([PI_, 0.0]), float(qz(0.6)), ccw=False)]))
    loops.append(("I3", [(qz(P), w) for P, w in _circle_arcs(qz([0.0, 3.0]), float(qz(0.5)), ccw=True)]))
    jit = _jit(seed, store_jitter)
    for _, segs in loops:
        for P, w in segs:
            b.seg(_wrap_store(P, T, T, True, True, jit=jit), w)
        b.end_loop()
    b.end_face(periodic=3, domain=(0.0, T, 0.0, T))
    uv = rng.uniform(0.0, 1.0, size=(n_queries, 2)) * T
    uv = np.minimum(uv, np.nextafter(T, 0.0))
    meta = dict(kind="C3", T=T, ph_a=ph_a, ph_b=ph_b, alpha_v=4.6, beta_v=1.7, amp=0.3, exact=exact,
                circles=[((0.0, 0.0), float(qz(0.6)), -1), ((PI_, 0.0), float(qz(0.6)), -1),
                         ((0.0, 3.0), float(qz(0.5)), +1)],
                alpha_knots=loops[0][1], beta_knots=loops[1][1])
    return _finish(b, np.zeros(n_queries), uv, True, "C3" if exact else "C3-generic", meta)


# ----------------------------------------------------------------------------
# C3pq — bi-periodic torus with a general coprime class (p,q) (SURVEY 8(f)
# NEXT-2; the paper's Dataset B has 2 <= p,q <= 5).  Not one of the five
# BASELINE configs: a parity case for the general band path.
# ----------------------------------------------------------------------------

def _band_frame(p, q, Tu, Tv):
    """Extension vector v = (p Tu, q Tv), the transverse vector w (w perpendicular
    to v, band coordinate nu(w) = 1 with nu(x) = p*y/Tv - q*x/Tu) -- input
    construction only."""
    v = np.array([p * Tu, q * Tv])
    L = math.hypot(v[0], v[1])
    w = np.array([-v[1], v[0]]) / L * (Tu * Tv / L)
    return v, w


def _hermite_band_loop(a0, v, w, f, fp, tau0, direction, n_seg, qz=quant):
    """x(tau) = a0 + tau v + f(tau) w over one period of tau (direction +1: tau0 ->
    tau0+1, class (p,q); -1: class -(p,q)), as cubic Hermite segments with
    control points rounded by qz; the end is the start + direction*v (exact in
    Q40 arithmetic, rounded once otherwise)."""
    taus = tau0 + direction * np.arange(n_seg + 1) / n_seg
    X = lambda t: a0 + t * v + f(t) * w
    dX = lambda t: v + fp(t) * w
    K = [qz(X(t)) for t in taus]
    K[-1] = K[0] + direction * v                     # closure
    segs = []
    for k in range(n_seg):
        h = taus[k + 1] - taus[k]
        P0, P3 = K[k], K[k + 1]
        P1 = qz(P0 + (h / 3.0) * dX(taus[k]))
        P2 = qz(P3 - (h / 3.0) * dX(taus[k + 1]))
        segs.append((np.stack([P0, P1, P2, P3]), np.ones(4)))
    return segs


def gen_c3pq(seed=6, p=2, q=1, n_queries=100_000, Tu=None, Tv=None, n_seg=None, beta_shift=(0, 1), exact=True,
             store_jitter=0):
    """Bi-periodic face whose separation loops alpha / beta have classes (p,q) /
    -(p,q): alpha at band coordinate nu = 0.2 + 0.05 sin(2 pi (2 tau) + phi_a),
    beta at nu = 0.6 + 0.05 sin(...) (the band between them is the interior),
    two CW hole circles inside the band (nu = 0.4) and one CCW island outside it
    (nu = 0.9).  beta is stored shifted by `beta_shift` tiles before wrapping so
    that pairing must find its proper translate.  All loops stored
    seam-discontinuous (R18); queries uniform in the fundamental domain."""
    rng = np.random.Generator(np.random.PCG64(seed))
    qz = _qz(exact)
    T2, _ = _periods(exact)
    Tu = T2 if Tu is None else float(qz(Tu))
    Tv = T2 if Tv is None else float(qz(Tv))
    assert math.gcd(abs(p), abs(q)) == 1
    if n_seg is None:
        n_seg = 12 * max(abs(p), abs(q), 1)
    v, w = _band_frame(p, q, Tu, Tv)
    s = float(np.linalg.norm(w))                     # distance per unit nu
    a0 = qz(rng.uniform(0, 1, size=2) * [Tu, Tv])
    ph_a, ph_b = rng.uniform(0, 2 * math.pi, size=2)
    A = 0.05
    fa = lambda t: 0.2 + A * np.sin(4 * math.pi * t + ph_a)
    fpa = lambda t: 4 * math.pi * A * math.cos(4 * math.pi * t + ph_a)
    fb = lambda t: 0.6 + A * np.sin(4 * math.pi * t + ph_b)
    fpb = lambda t: 4 * math.pi * A * math.cos(4 * math.pi * t + ph_b)
    tb = float(rng.uniform(0, 1))
    alpha = _hermite_band_loop(a0, v, w, fa, fpa, 0.0, +1, n_seg, qz)
    beta = _hermite_band_loop(a0, v, w, fb, fpb, tb, -1, n_seg, qz)
    shift = np.array([beta_shift[0] * Tu, beta_shift[1] * Tv])
    beta_stored = [(P + shift, wt) for P, wt in beta]
    r = float(qz(0.075 * s))
    circles = []
    for tau_c, nu_c, orient in ((0.3, 0.4, -1), (0.75, 0.4, -1), (0.5, 0.9, +1)):
        c = qz(a0 + tau_c * v + nu_c * w)
        circles.append((c, r, orient))
    b = _Builder()
    loops = [alpha, beta_stored] + [[(qz(P), wt) for P, wt in _circle_arcs(c, r, ccw=(o > 0))]
                                     for c, r, o in circles]
    jit = _jit(seed, store_jitter)
    for segs in loops:
        for P, wt in segs:
            b.seg(_wrap_store(P, Tu, Tv, True, True, jit=jit), wt)
        b.end_loop()
    b.end_face(periodic=3, domain=(0.0, Tu, 0.0, Tv))
    uv = rng.uniform(0.0, 1.0, size=(n_queries, 2)) * [Tu, Tv]
    uv = np.minimum(uv, np.nextafter(np.array([Tu, Tv]), 0.0))
    meta = dict(kind="C3pq", p=p, q=q, Tu=Tu, Tv=Tv, a0=a0, v=v, w=w, alpha=alpha, beta=beta, exact=exact,
                circles=[(tuple(c), r, o) for c, r, o in circles])
    return _finish(b, np.zeros(n_queries), uv, False, "C3pq(%d,%d)%s" % (p, q, "" if exact else "-generic"), meta)


# ----------------------------------------------------------------------------
# C4 — robustness set: gapped / open cubic loops (BASELINE configs[3])
# ----------------------------------------------------------------------------

def gen_c4(seed=4, n_faces=1000, q_per_face=256, n_deleted=None, sigma=1e-4):
    rng = np.random.Generator(np.random.PCG64(seed))
    if n_deleted is None:
        n_deleted = n_faces // 10
    deleted = set(rng.choice(n_faces, size=n_deleted, replace=False).tolist())
    b = _Builder()
    uvs = []
    fids = []
    for f in range(n_faces):
        c = np.array([0.5, 0.5])
        ang = 2.0 * math.pi * np.arange(64) / 64
        rad = 0.35 + rng.uniform(-0.05, 0.05, size=64)
        V = c + rad[:, None] * np.stack([np.cos(ang), np.sin(ang)], 1)
        skip = int(rng.integers(0, 64)) if f in deleted else -1
        pts = []
        for k in range(64):
            A, Bv = V[k], V[(k + 1) % 64]
            P1 = A + (V[(k + 1) % 64] - V[(k - 1) % 64]) / 6.0
            P2 = Bv - (V[(k + 2) % 64] - V[k]) / 6.0
            P0 = A + rng.normal(0.0, sigma, size=2)
            P3 = Bv + rng.normal(0.0, sigma, size=2)
            if k == skip:
                continue
            P = np.stack([P0, P1, P2, P3])
            b.seg(P)
            pts.append(P)
        b.end_loop()
        b.end_face()
        allp = np.concatenate(pts)
        lo, hi = allp.min(0), allp.max(0)
        uvs.append(lo + (hi - lo) * rng.uniform(0.0, 1.0, size=(q_per_face, 2)))
        fids.append(np.full(q_per_face, f))
    meta = dict(kind="C4", deleted=sorted(deleted), sigma=sigma)
    return _finish(b, np.concatenate(fids), np.concatenate(uvs), False, "C4", meta)


def to_fp32_inputs(wl):
    """C4-fp32 variant: inputs rounded to fp32, promoted back exactly."""
    out = dict(wl)
    out["ctrl_uv"] = wl["ctrl_uv"].astype(np.float32).astype(np.float64)
    if wl["ctrl_w"] is not None:
        out["ctrl_w"] = wl["ctrl_w"].astype(np.float32).astype(np.float64)
    out["uv"] = wl["uv"].astype(np.float32).astype(np.float64)
    out["face_domain"] = wl["face_domain"].astype(np.float32).astype(np.float64)
    out["eps"] = EPS_FP32
    out["name"] = wl["name"] + "-fp32"
    return out


# ----------------------------------------------------------------------------
# C5 — synthetic B-Rep batch / tessellation grid (BASELINE configs[4]); R22
# ----------------------------------------------------------------------------

def _n_segs(rng):
    return int(round(math.exp(rng.uniform(math.log(4.0), math.log(128.0)))))


def gen_c5(seed=5, n_faces=20_000, grid=64, periodic_frac=0.30, exact=True, store_jitter=0):
    rng = np.random.Generator(np.random.PCG64(seed))
    jit = _jit(seed, store_jitter)
    T, _ = _periods(exact)
    qz = _qz(exact)
    b = _Builder()
    uvs = []
    boxes = []   # per-face grid box (u_lo, v_lo, u_hi, v_hi): the implicit-grid form of the batch
    fids = []
    n_periodic = 0
    slots = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1)]
    for f in range(n_faces):
        L = min(int(rng.geometric(0.5)), 8)
        periodic = rng.random() < periodic_frac
        if not periodic:
            c = np.array([0.5, 0.5])
            n = _n_segs(rng)
            V = _star_vertices(rng, c, 0.42, 0.04, n, cw=False)
            pts = []
            for P, w in _star_segments(rng, V, rng.integers(1, 6, size=n), 0.05, True):
                b.seg(P, w)
                pts.append(P)
            b.end_loop()
            picks = rng.choice(9, size=L - 1, replace=False)
            for s in picks:
                hc = c + 0.15 * np.array(slots[s]) + rng.uniform(-0.005, 0.005, size=2)
                n = _n_segs(rng)
                V = _star_vertices(rng, hc, 0.06, 0.005, n, cw=True)
                for P, w in _star_segments(rng, V, rng.integers(1, 6, size=n), 0.05, True):
                    b.seg(P, w)
                b.end_loop()
            b.end_face(periodic=0, domain=(0.0, 1.0, 0.0, 1.0))
            allp = np.concatenate(pts)
            boxes.append((*allp.min(0), *allp.max(0)))
            uvs.append(_grid(allp.min(0), allp.max(0), grid))
        else:
            n_periodic += 1
            loops = []
            if L >= 2:
                kf = int(rng.integers(1, 4))
                pa, pb = rng.uniform(0, 2 * math.pi, size=2)
                fa = lambda u, kf=kf, pa=pa: 0.25 + 0.05 * np.sin(kf * u + pa)
                fb = lambda u, kf=kf, pb=pb: 0.75 + 0.05 * np.sin(kf * u + pb)
                na, nb = _n_segs(rng), _n_segs(rng)
                loops.append(_graph_loop(rng, fa, float(qz(rng.uniform(0, T))), T, +1, na,
                                         rng.integers(1, 6, size=na), True, qz))
                loops.append(_graph_loop(rng, fb, float(qz(rng.uniform(0, T))), T, -1, nb,
                                         rng.integers(1, 6, size=nb), True, qz))
                nh = L - 2
                for j in range(nh):
                    hu = 0.0 if j == 0 else j * T / nh + rng.uniform(-0.05, 0.05)
                    hc = qz([hu, 0.5 + rng.uniform(-0.1, 0.1)])
                    n = _n_segs(rng)
                    V = qz(_star_vertices(rng, hc, 0.06, 0.005, n, cw=True))
                    segs = _star_segments(rng, V, rng.integers(1, 6, size=n), 0.05, True)
                    loops.append([(qz(P), w) for P, w in segs])
            else:
                hc = qz([0.0, 0.5])
                n = _n_segs(rng)
                V = qz(_star_vertices(rng, hc, 0.3, 0.02, n, cw=False))
                segs = _star_segments(rng, V, rng.integers(1, 6, size=n), 0.05, True)
                loops.append([(qz(P), w) for P, w in segs])
            for segs in loops:
                for P, w in segs:
                    b.seg(_wrap_store(P, T, 1.0, True, False, jit=jit), w)
                b.end_loop()
            b.end_face(periodic=1, domain=(0.0, T, 0.0, 1.0))
            boxes.append((0.0, 0.0, T, 1.0))
            uvs.append(_grid((0.0, 0.0), (T, 1.0), grid))
        fids.append(np.full(grid * grid, f))
    meta = dict(kind="C5", n_periodic=n_periodic, grid=grid, exact=exact,
                grid_box=np.ascontiguousarray(np.asarray(boxes, dtype=np.float64).reshape(-1, 4)))
    return _finish(b, np.concatenate(fids), np.concatenate(uvs), True, "C5" if exact else "C5-generic", meta)


# ----------------------------------------------------------------------------
# NURBS ingest workload ("B-spline or NURBS
# curves can always be subdivided into (rational) Bezier segments").  Not a
# BASELINE config: a parity case for wn_build_faces_nurbs.  Layout (ABI of
# wn_build_faces_nurbs, include/wn.h):
#   ctrl_uv [n_ctrl,2], ctrl_w [n_ctrl], curve_degree [n_curves],
#   curve_ctrl_off [n_curves+1], knots [n_knots], curve_knot_off [n_curves+1],
#   loop_curve_off [n_loops+1], face_loop_off, face_periodic, face_domain,
#   face_id, uv.
# ----------------------------------------------------------------------------

def _clamped_knots(rng, n_ctrl, p, max_mult=None):
    """Clamped knot vector on [0,1] for n_ctrl control points of degree p with
    random interior knots, some repeated (multiplicity <= max_mult <= p)."""
    n_int = n_ctrl - p - 1
    max_mult = p if max_mult is None else max_mult
    ks = []
    while len(ks) < n_int:
        u = float(rng.uniform(0.02, 0.98))
        mult = int(rng.integers(1, max_mult + 1)) if rng.uniform() < 0.3 else 1
        ks.extend([u] * min(mult, n_int - len(ks)))
    ks = sorted(ks)
    return np.concatenate([np.zeros(p + 1), np.asarray(ks), np.ones(p + 1)])


def gen_nurbs(seed=7, n_faces=200, q_per_face=256, max_curves=3):
    """Faces bounded by closed loops made of 1..max_curves clamped NURBS curves
    (degree 1..5, 1..8 knot spans, weights U[0.5,2], random interior knot
    multiplicities): an outer star-like loop (CCW) about (0.5,0.5) of radius
    0.38 +- 0.04 and 0..2 CW holes of radius 0.07 at (0.5 +- 0.17, 0.5);
    queries uniform in the unit square."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ctrl, wts, deg, coff, knots, koff, lco, flo = [], [], [], [0], [], [0], [0], [0]
    n_loops = 0

    def loop(center, r_mean, r_jit, cw):
        nonlocal n_loops
        k = int(rng.integers(1, max_curves + 1))
        cuts = np.sort(rng.uniform(0, 2 * math.pi, size=k))
        th0 = cuts[0]
        bounds = list(cuts) + [th0 + 2 * math.pi]
        start_pt = None
        pts_prev_end = None
        curves = []
        for c in range(k):
            a, b_ = bounds[c], bounds[c + 1]
            p = int(rng.integers(1, 6))
            spans = int(rng.integers(1, 9))
            # control polygon fine enough (<= 30 deg per leg) that the curve
            # follows the star polygon (stays simple, encloses the centre)
            need = int(math.ceil((b_ - a) / (math.pi / 6))) + 1
            spans = max(spans, need - p)
            n_ctrl = p + spans
            th = np.linspace(a, b_, n_ctrl)
            rad = r_mean + rng.uniform(-r_jit, r_jit, size=n_ctrl)
            P = np.stack([center[0] + rad * np.cos(th), center[1] + rad * np.sin(th)], 1)
            if pts_prev_end is not None:
                P[0] = pts_prev_end
            pts_prev_end = P[-1].copy()
            if start_pt is None:
                start_pt = P[0].copy()
            w = rng.uniform(0.5, 2.0, size=n_ctrl)
            U = _clamped_knots(rng, n_ctrl, p)
            curves.append([P, w, p, U])
        curves[-1][0][-1] = start_pt          # closed loop: bit-identical junctions
        if cw:                                # reverse: curves in reverse order, each reversed
            curves = [[P[::-1].copy(), w[::-1].copy(), p, (1.0 - U[::-1]).copy()] for P, w, p, U in curves[::-1]]
        for P, w, p, U in curves:
            ctrl.append(P); wts.append(w); deg.append(p)
            coff.append(coff[-1] + len(P))
            knots.append(U); koff.append(koff[-1] + len(U))
        lco.append(lco[-1] + len(curves))
        n_loops += 1

    fids, uvs = [], []
    for f in range(n_faces):
        loop((0.5, 0.5), 0.38, 0.04, False)
        nh = int(rng.integers(0, 3))
        for h in range(nh):
            loop((0.5 + (0.17 if h == 0 else -0.17), 0.5), 0.07, 0.005, True)
        flo.append(n_loops)
        fids.append(np.full(q_per_face, f))
        uvs.append(rng.uniform(0, 1, size=(q_per_face, 2)))
    return dict(
        ctrl_uv=np.ascontiguousarray(np.concatenate(ctrl)), ctrl_w=np.ascontiguousarray(np.concatenate(wts)),
        curve_degree=np.asarray(deg, dtype=np.int32), curve_ctrl_off=np.asarray(coff, dtype=np.int32),
        knots=np.ascontiguousarray(np.concatenate(knots)), curve_knot_off=np.asarray(koff, dtype=np.int32),
        loop_curve_off=np.asarray(lco, dtype=np.int32), face_loop_off=np.asarray(flo, dtype=np.int32),
        face_periodic=np.zeros(n_faces, dtype=np.uint8),
        face_domain=np.tile(np.array([0.0, 1.0, 0.0, 1.0]), (n_faces, 1)),
        face_id=np.concatenate(fids).astype(np.int32), uv=np.ascontiguousarray(np.concatenate(uvs)),
        name="NURBS", eps=EPS_FP64, meta=dict(kind="NURBS"))


CONFIGS = {"C1": gen_c1, "C2": gen_c2, "C3": gen_c3, "C4": gen_c4, "C5": gen_c5}


def n_input_pairs(wl):
    """Sum over queries of the number of input segments of the query's face
    (the 'query*segment pairs' unit of BASELINE.json's metric)."""
    segs_per_loop = np.diff(wl["loop_seg_off"]).astype(np.int64)
    fl = wl["face_loop_off"]
    csum = np.concatenate([[0], np.cumsum(segs_per_loop)])
    segs_per_face = csum[fl[1:]] - csum[fl[:-1]]
    return int(segs_per_face[wl["face_id"]].sum())
