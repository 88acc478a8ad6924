"""Oracle pins against closed forms and invariants the paper fixes:
polygons vs textbook crossing number (degree 1 and degree-elevated),
exact circles, the open circular arc, star-shaped analytic classification of
the generated loops, additivity / orientation, the gap-closure identity."""
import math

import numpy as np
import pytest

import oracle
from tests import helpers as H
from wn_workloads import configs as G


def _star_polygon(rng, n, c=(0.5, 0.5), r=0.3, jit=0.1):
    ang = np.sort(rng.uniform(0, 2 * np.pi, size=n))
    rad = r * (1 + rng.uniform(-jit, jit, size=n))
    return np.stack([c[0] + rad * np.cos(ang), c[1] + rad * np.sin(ang)], 1)


@pytest.mark.parametrize("elevated", [False, True])
def test_polygons_vs_crossing_number(elevated):
    """Degree-1 polygons (and the same edges degree-elevated to cubic) give the
    textbook crossing-number winding exactly (integer, residual < 1e-13)."""
    rng = np.random.default_rng(10)
    for trial in range(15):
        V = _star_polygon(rng, int(rng.integers(3, 12)))
        if trial % 2:
            V = V[::-1]
        loop = H.polygon_loop(V)
        if elevated:
            el = []
            for P, w in loop:
                P2, w2 = H.elevate(P, w)
                P3, w3 = H.elevate(P2, w2)
                P3[0], P3[-1] = P[0], P[-1]
                el.append((P3, w3))
            loop = el
        q = rng.uniform(0, 1, size=(300, 2))
        wl = H.make_wl([([loop], 0, (0, 1, 0, 1))], q)
        r = oracle.query(wl)
        for i, p in enumerate(q):
            ref = H.pip_crossing(V, p)
            if r["comparable"][i]:
                assert abs(r["w"][i] - ref) < 1e-13


@pytest.mark.parametrize("ccw", [True, False])
def test_exact_circle(ccw):
    c, rad = np.array([0.4, 0.55]), 0.3
    arcs = H.circle_arcs(c, rad, ccw)
    rng = np.random.default_rng(11)
    q = rng.uniform(0, 1, size=(3000, 2))
    r = oracle.query(H.make_wl([([arcs], 0, (0, 1, 0, 1))], q))
    d = np.hypot(*(q - c).T)
    ok = np.abs(d - rad) > 1e-9
    expect = np.where(d < rad, 1.0 if ccw else -1.0, 0.0)
    assert np.all(np.abs(r["w"][ok] - expect[ok]) < 1e-12)
    assert r["comparable"][ok].all()


def test_open_arc_closed_form():
    """omega(arc) = [p in circular segment] + omega(p, start, end) for a CCW
    circular arc of angle < pi (single rational quadratic)."""
    rng = np.random.default_rng(12)
    for a in (0.4, 1.3, 2.6):
        c, rad, a0 = np.array([0.5, 0.5]), 0.3, rng.uniform(0, 2 * np.pi)
        S = c + rad * np.array([math.cos(a0), math.sin(a0)])
        E = c + rad * np.array([math.cos(a0 + a), math.sin(a0 + a)])
        M = c + (rad / math.cos(a / 2)) * np.array([math.cos(a0 + a / 2), math.sin(a0 + a / 2)])
        arc = [(np.stack([S, M, E]), np.array([1.0, math.cos(a / 2), 1.0]))]
        q = rng.uniform(0, 1, size=(2000, 2))
        r = oracle.query(H.make_wl([([arc], 0, (0, 1, 0, 1))], q))
        d = np.hypot(*(q - c).T)
        cr = (E - S)[0] * (q[:, 1] - S[1]) - (E - S)[1] * (q[:, 0] - S[0])
        inseg = (d < rad) & (cr < 0)
        ch = np.array([oracle.chord(p, S, E) for p in q])
        ok = (np.abs(d - rad) > 1e-9) & (np.abs(cr) > 1e-9)
        assert np.all(np.abs(r["w"][ok] - (inseg[ok] + ch[ok])) < 1e-12)


def _star_check(wl, centers, nq=400, seed=0):
    loops = H.loops_of(wl)
    rng = np.random.default_rng(seed)
    q = wl["uv"][rng.choice(len(wl["uv"]), size=min(nq, len(wl["uv"])), replace=False)]
    total = np.zeros(len(q), dtype=np.int64)
    margin = np.full(len(q), np.inf)
    for segs, c in zip(loops, centers):
        res, mg = H.star_classify(segs, c, q)
        total += res
        margin = np.minimum(margin, mg)
    r = oracle.query(wl, face_id=np.zeros(len(q), np.int32), uv=q)
    ok = margin > 1e-9
    assert ok.mean() > 0.95
    assert np.all(np.abs(r["w"][ok] - total[ok]) < 1e-12)
    assert np.all(r["flag"][ok] == (total[ok] != 0))


def test_star_c1():
    wl = G.gen_c1(n_queries=2000)
    _star_check(wl, wl["meta"]["star_centers"])


def test_star_c2():
    wl = G.gen_c2(n_queries=4000)
    _star_check(wl, wl["meta"]["star_centers"], nq=300)


def test_star_c5_nonperiodic_faces():
    wl = G.gen_c5(n_faces=6, grid=8)
    loops = H.loops_of(wl)
    fo = wl["face_loop_off"]
    checked = 0
    for f in range(len(fo) - 1):
        if wl["face_periodic"][f]:
            continue
        sub = dict(wl)
        m = wl["face_id"] == f
        q = wl["uv"][m]
        total = np.zeros(len(q), dtype=np.int64)
        margin = np.full(len(q), np.inf)
        for l in range(fo[f], fo[f + 1]):
            segs = loops[l]
            allp = np.concatenate([P for P, _ in segs])
            # star centre: outer loop (0.5,0.5); holes: mean of their vertices
            c = (0.5, 0.5) if l == fo[f] else tuple(np.mean([P[0] for P, _ in segs], 0))
            res, mg = H.star_classify(segs, c, q)
            total += res
            margin = np.minimum(margin, mg)
        r = oracle.query(sub, face_id=np.full(len(q), f, np.int32), uv=q)
        ok = margin > 1e-9
        assert np.all(np.abs(r["w"][ok] - total[ok]) < 1e-12)
        checked += 1
    assert checked >= 2


def test_orientation_reversal_and_additivity():
    wl = G.gen_c2(n_queries=500)
    loops = H.loops_of(wl)
    q = wl["uv"]
    r = oracle.query(wl)
    rev = [[(P[::-1].copy(), None if w is None else w[::-1].copy()) for P, w in segs[::-1]] for segs in loops]
    r2 = oracle.query(H.make_wl([(rev, 0, (0, 1, 0, 1))], q))
    ok = r["comparable"]
    assert np.all(np.abs(r["w"][ok] + r2["w"][ok]) < 1e-12)
    # additivity over loops: one face per loop, same queries
    parts = np.zeros(len(q))
    for segs in loops:
        parts += oracle.query(H.make_wl([([segs], 0, (0, 1, 0, 1))], q))["w"]
    assert np.all(np.abs(r["w"][ok] - parts[ok]) < 1e-12)


def test_gap_closure_identity_c4():
    """omega_open + sum_gaps omega(p, e_i, s_{i+1}) is an integer,
    and that integer matches a dense-polyline crossing count of the closed-up curve."""
    wl = G.gen_c4(n_faces=12, q_per_face=40, n_deleted=3)
    loops = H.loops_of(wl)
    r = oracle.query(wl)
    for f in range(12):
        segs = loops[f]
        m = wl["face_id"] == f
        q = wl["uv"][m]
        w = r["w"][m]
        gaps = np.zeros(len(q))
        n = len(segs)
        for i in range(n):
            e = segs[i][0][-1]
            s = segs[(i + 1) % n][0][0]
            gaps += np.array([oracle.chord(p, e, s) for p in q])
        tot = w + gaps
        ok = r["comparable"][m]
        assert np.all(np.abs(tot[ok] - np.round(tot[ok])) < 1e-12)
        dense = H.sample_loop(segs, 64)
        closed = []
        for i in range(n):
            closed.append(H.sample_loop([segs[i]], 64))
        poly = np.concatenate(closed)
        for j in np.nonzero(ok)[0][:10]:
            assert round(tot[j]) == H.pip_crossing(poly, q[j])
