"""Independent test-side references used to PIN the oracle (never imported by
the oracle or the product).  Each is a textbook construction that shares no
code with oracle/wn_oracle.c:

  bern_eval        Bernstein-basis evaluation of a rational Bezier segment
  elevate          Bernstein degree elevation
  pip_crossing     textbook crossing-number point-in-polygon
  polyline_wn      dense-polyline angle sum (SPEC S:192-200 brute force)
  star_inside      analytic classification of star-shaped loops by bisection
                   on the monotone polar angle (SURVEY 8(c) pin table)
"""
import math

import numpy as np


def bern_eval(P, w, t):
    P = np.asarray(P, dtype=np.float64)
    n = P.shape[0] - 1
    w = np.ones(n + 1) if w is None else np.asarray(w, dtype=np.float64)
    t = np.atleast_1d(np.asarray(t, dtype=np.float64))
    B = np.stack([math.comb(n, j) * t ** j * (1.0 - t) ** (n - j) for j in range(n + 1)], 1)
    num = B @ (w[:, None] * P)
    den = B @ w
    return num / den[:, None]


def elevate(P, w):
    """Degree elevation n -> n+1 in homogeneous coordinates."""
    P = np.asarray(P, dtype=np.float64)
    n = P.shape[0] - 1
    w = np.ones(n + 1) if w is None else np.asarray(w, dtype=np.float64)
    H = np.concatenate([w[:, None] * P, w[:, None]], 1)
    Q = np.zeros((n + 2, 3))
    Q[0] = H[0]
    Q[n + 1] = H[n]
    for i in range(1, n + 1):
        a = i / (n + 1)
        Q[i] = a * H[i - 1] + (1 - a) * H[i]
    return Q[:, :2] / Q[:, 2:3], Q[:, 2].copy()


def pip_crossing(poly, p):
    """Textbook even-odd crossing number; returns winding parity (0/1) and the
    signed crossing count of the +x ray (== winding number for simple polygons)."""
    x, y = p
    wn = 0
    n = len(poly)
    for i in range(n):
        x0, y0 = poly[i]
        x1, y1 = poly[(i + 1) % n]
        if y0 <= y < y1:
            if (x1 - x0) * (y - y0) - (x - x0) * (y1 - y0) > 0:
                wn += 1
        elif y1 <= y < y0:
            if (x1 - x0) * (y - y0) - (x - x0) * (y1 - y0) < 0:
                wn -= 1
    return wn


def polyline_wn(pts, p):
    """Angle sum of a polyline about p (open polyline allowed), /2pi."""
    d = pts - np.asarray(p)[None, :]
    a, b = d[:-1], d[1:]
    cr = a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]
    dt = a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1]
    return np.arctan2(cr, dt).sum() / (2 * math.pi)


def sample_loop(segs, m):
    """Dense samples of a loop given as list of (P, w); m samples per segment."""
    out = []
    for P, w in segs:
        out.append(bern_eval(P, w, np.linspace(0.0, 1.0, m + 1))[:-1])
    out.append(bern_eval(segs[-1][0], segs[-1][1], np.array([1.0])))
    return np.concatenate(out)


def loops_of(wl):
    """List of loops, each a list of (P, w) in stored coordinates."""
    deg = wl["seg_degree"]
    off = np.concatenate([[0], np.cumsum(deg + 1)])
    loops = []
    lo = wl["loop_seg_off"]
    for l in range(len(lo) - 1):
        segs = []
        for s in range(lo[l], lo[l + 1]):
            P = wl["ctrl_uv"][off[s]:off[s + 1]]
            w = None if wl["ctrl_w"] is None else wl["ctrl_w"][off[s]:off[s + 1]]
            segs.append((P, w))
        loops.append(segs)
    return loops


def star_radius_fn(segs, c, m=64):
    """For a loop star-shaped about c: returns rho(theta) by locating the segment
    whose polar range contains theta (dense samples assert monotonicity) and
    bisecting on t.  Returns (rho_fn, ok_monotone, orientation)."""
    c = np.asarray(c)
    pieces = []
    total = 0.0
    for P, w in segs:
        ts = np.linspace(0.0, 1.0, m + 1)
        pts = bern_eval(P, w, ts) - c
        ang = np.unwrap(np.arctan2(pts[:, 1], pts[:, 0]))
        da = np.diff(ang)
        total += ang[-1] - ang[0]
        pieces.append((P, w, ang[0], ang[-1], da))
    orient = 1 if total > 0 else -1
    ok = all(np.all(orient * pc[4] > 0) for pc in pieces)

    def rho(theta):
        for P, w, a0, a1, _ in pieces:
            lo_a, hi_a = (a0, a1) if a1 > a0 else (a1, a0)
            # bring theta into the unwrapped range of this piece
            th = theta
            while th < lo_a:
                th += 2 * math.pi
            while th >= lo_a + 2 * math.pi:
                th -= 2 * math.pi
            if lo_a <= th <= hi_a:
                ta, tb = 0.0, 1.0
                fa = a0 - th
                for _ in range(80):
                    tm = 0.5 * (ta + tb)
                    q = bern_eval(P, w, np.array([tm]))[0] - c
                    am = math.atan2(q[1], q[0])
                    # unwrap am near a0..a1
                    base = a0 + (tm * (a1 - a0))
                    am += 2 * math.pi * round((base - am) / (2 * math.pi))
                    if (am - th) * (fa) > 0:
                        ta = tm
                    else:
                        tb = tm
                q = bern_eval(P, w, np.array([0.5 * (ta + tb)]))[0] - c
                return math.hypot(q[0], q[1])
        raise RuntimeError("theta not covered")
    return rho, ok, orient


def star_classify(segs, c, pts, m=64):
    """Winding of a star-shaped closed loop (+-1 inside, 0 outside) and the radial
    margin | |p-c| - rho(theta_p) | for each point."""
    rho, ok, orient = star_radius_fn(segs, c, m)
    assert ok, "loop not star-shaped about its centre"
    res = np.zeros(len(pts), dtype=np.int64)
    margin = np.zeros(len(pts))
    for i, p in enumerate(pts):
        d = np.asarray(p) - np.asarray(c)
        th = math.atan2(d[1], d[0])
        r = rho(th)
        rp = math.hypot(d[0], d[1])
        res[i] = orient if rp < r else 0
        margin[i] = abs(rp - r)
    return res, margin


def make_wl(faces, queries=None, face_ids=None, rational=True):
    """Build an ABI workload from faces = [(loops, periodic, domain)], loops =
    [[(P, w), ...], ...] in STORED coordinates."""
    from wn_workloads.configs import _Builder
    b = _Builder()
    for loops, periodic, domain in faces:
        for segs in loops:
            for P, w in segs:
                b.seg(np.asarray(P, dtype=np.float64), w)
            b.end_loop()
        b.end_face(periodic=periodic, domain=domain)
    d = b.arrays(rational=rational)
    if queries is None:
        queries = np.zeros((0, 2))
    queries = np.asarray(queries, dtype=np.float64).reshape(-1, 2)
    d["uv"] = np.ascontiguousarray(queries)
    d["face_id"] = np.ascontiguousarray(np.zeros(len(queries), np.int32) if face_ids is None
                                        else np.asarray(face_ids, np.int32))
    d["eps"] = 1e-10
    d["meta"] = {}
    return d


def circle_arcs(c, r, ccw=True):
    from wn_workloads.configs import _circle_arcs
    return _circle_arcs(np.asarray(c, dtype=np.float64), float(r), ccw)


def line_loop(p0, p1, n=1):
    """A straight loop p0 -> p1 split into n degree-1 segments."""
    p0 = np.asarray(p0, dtype=np.float64)
    p1 = np.asarray(p1, dtype=np.float64)
    pts = [p0 + (p1 - p0) * k / n for k in range(n + 1)]
    pts[0], pts[-1] = p0, p1
    return [(np.stack([pts[k], pts[k + 1]]), None) for k in range(n)]


def polygon_loop(V):
    V = np.asarray(V, dtype=np.float64)
    n = len(V)
    return [(np.stack([V[k], V[(k + 1) % n]]), None) for k in range(n)]


def deboor_eval(p, P, w, U, t):
    """NURBS point by the Cox-de Boor recursion (textbook definition of the
    B-spline basis, 0/0 := 0; half-open spans, t = U[-1] in the last span):
    C(t) = sum N_ip(t) w_i P_i / sum N_ip(t) w_i."""
    P = np.asarray(P, dtype=np.float64)
    n = len(P)
    w = np.ones(n) if w is None else np.asarray(w, dtype=np.float64)
    U = np.asarray(U, dtype=np.float64)
    m = len(U)
    # degree-0 basis
    N = np.zeros(m - 1)
    last = max(i for i in range(m - 1) if U[i] < U[i + 1])
    for i in range(m - 1):
        if U[i] <= t < U[i + 1] or (t == U[-1] and i == last):
            N[i] = 1.0
    for k in range(1, p + 1):
        N2 = np.zeros(m - 1 - k)
        for i in range(m - 1 - k):
            a = (t - U[i]) / (U[i + k] - U[i]) * N[i] if U[i + k] != U[i] else 0.0
            b = (U[i + k + 1] - t) / (U[i + k + 1] - U[i + 1]) * N[i + 1] if U[i + k + 1] != U[i + 1] else 0.0
            N2[i] = a + b
        N = N2
    N = N[:n]
    den = N @ w
    return (N * w) @ P / den
