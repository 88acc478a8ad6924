"""Pins of the oracle's NURBS ingest (NURBS curves "can always be
subdivided into (rational) Bezier segments"; SPEC decompose_bspline): the
decomposition reproduces an independent Cox-de Boor evaluation of the spline,
SPEC's worked examples, and the exact NURBS circle's winding numbers."""
import math

import numpy as np
import pytest

import oracle
from tests import helpers as H
from wn_workloads import configs as G


def _spans(U, p):
    br = np.unique(U[p:len(U) - p])
    return list(zip(br[:-1], br[1:]))


def _check_curve(p, P, w, U, rng, nt=60, tol=1e-12):
    segs = oracle.nurbs_decompose(p, P, w, U)
    spans = _spans(U, p)
    assert len(segs) == len(spans)
    for _ in range(nt):
        j = int(rng.integers(len(spans)))
        a, b = spans[j]
        s = float(rng.uniform())
        t = a + s * (b - a)
        s = (t - a) / (b - a)
        ref = H.deboor_eval(p, P, w, U, t)
        got = H.bern_eval(segs[j][0], segs[j][1], s)[0]
        assert np.max(np.abs(got - ref)) < tol, (p, t, got, ref)
    # end points exact, interior junctions shared
    assert np.array_equal(segs[0][0][0], P[0]) and np.array_equal(segs[-1][0][-1], P[-1])
    for j in range(len(segs) - 1):
        assert np.array_equal(segs[j][0][-1], segs[j + 1][0][0])
    return segs


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_decompose_vs_cox_de_boor(p):
    rng = np.random.default_rng(100 + p)
    for trial in range(6):
        n_ctrl = p + 1 + int(rng.integers(0, 9))
        P = rng.uniform(-1, 1, size=(n_ctrl, 2))
        w = rng.uniform(0.5, 2.0, size=n_ctrl)
        U = G._clamped_knots(rng, n_ctrl, p)
        _check_curve(p, P, w, U, rng)
        _check_curve(p, P, None, U, rng)


def test_single_span_is_identity():
    """SPEC: knots 0,0,0,0,1,1,1,1 (degree 3) -> one identical segment."""
    P = np.array([[0.0, 0.0], [1.0, 2.0], [3.0, 2.0], [4.0, 0.0]])
    w = np.array([1.0, 0.5, 2.0, 1.0])
    segs = oracle.nurbs_decompose(3, P, w, np.array([0, 0, 0, 0, 1, 1, 1, 1.0]))
    assert len(segs) == 1
    assert np.allclose(segs[0][0], P, atol=1e-15, rtol=0) and np.allclose(segs[0][1], w, atol=1e-15, rtol=0)


def test_two_span_uniform_cubic_junction():
    """SPEC: two-span uniform cubic B-spline -> two segments whose junction is the
    spline at the interior knot."""
    P = np.array([[0.0, 0.0], [1.0, 1.0], [2.0, -1.0], [3.0, 1.0], [4.0, 0.0]])
    U = np.array([0, 0, 0, 0, 0.5, 1, 1, 1, 1.0])
    segs = oracle.nurbs_decompose(3, P, None, U)
    assert len(segs) == 2
    assert np.max(np.abs(segs[0][0][-1] - H.deboor_eval(3, P, None, U, 0.5))) < 1e-15
    # the textbook junction of a uniform cubic: (P1 + 4 P2 + P3) / 6 ... with
    # clamped ends the interior knot point is (P1 + 2 P2 + P3) / 4 here
    assert np.max(np.abs(segs[0][0][-1] - (P[1] + 2 * P[2] + P[3]) / 4)) < 1e-15


def _nurbs_circle(c, r):
    s = math.sqrt(0.5)
    Q = np.array([[1, 0], [1, 1], [0, 1], [-1, 1], [-1, 0], [-1, -1], [0, -1], [1, -1], [1, 0]], dtype=np.float64)
    P = np.asarray(c) + r * Q
    w = np.array([1, s, 1, s, 1, s, 1, s, 1.0])
    U = np.array([0, 0, 0, 0.25, 0.25, 0.5, 0.5, 0.75, 0.75, 1, 1, 1.0])
    return P, w, U


def test_nurbs_circle_exact_winding():
    """The 9-point degree-2 NURBS circle decomposes into four exact circular
    arcs; its winding number is 1 inside, 0 outside (closed form)."""
    c, r = np.array([0.5, 0.5]), 0.3
    P, w, U = _nurbs_circle(c, r)
    segs = _check_curve(2, P, w, U, np.random.default_rng(1))
    for Ps, ws in segs:
        pts = H.bern_eval(Ps, ws, np.linspace(0, 1, 33))
        assert np.max(np.abs(np.hypot(*(pts - c).T) - r)) < 1e-15
    wl = dict(ctrl_uv=P, ctrl_w=w, curve_degree=np.array([2], np.int32), curve_ctrl_off=np.array([0, 9], np.int32),
              knots=U, curve_knot_off=np.array([0, 12], np.int32), loop_curve_off=np.array([0, 1], np.int32),
              face_loop_off=np.array([0, 1], np.int32), face_periodic=np.zeros(1, np.uint8),
              face_domain=np.array([[0.0, 1.0, 0.0, 1.0]]))
    bz = oracle.nurbs_to_bezier_workload(wl)
    q = np.random.default_rng(2).uniform(0, 1, size=(2000, 2))
    d = np.hypot(*(q - c).T)
    keep = np.abs(d - r) > 1e-9
    res = oracle.query(bz, face_id=np.zeros(len(q), np.int32), uv=q)
    assert np.array_equal(res["w"][keep].round(), (d[keep] < r).astype(float))
    assert np.max(np.abs(res["w"][keep] - (d[keep] < r))) < 1e-12


def test_generated_nurbs_faces_closed_integral():
    """gen_nurbs loops are closed (bit-identical junctions): every comparable
    winding number is an integer, and the outer loop's interior is inside."""
    wl = G.gen_nurbs(n_faces=12, q_per_face=64)
    bz = oracle.nurbs_to_bezier_workload(wl)
    r = oracle.query(bz)
    cm = r["comparable"]
    assert cm.mean() > 0.99
    assert np.max(np.abs(r["w"][cm] - np.round(r["w"][cm]))) < 1e-12
    assert set(np.round(r["w"][cm]).astype(int)) <= {0, 1}
    centre = oracle.query(bz, face_id=np.arange(12, dtype=np.int32), uv=np.tile([[0.5, 0.5]], (12, 1)))
    assert np.all(centre["w"].round() == 1)


@pytest.mark.parametrize("p", [1, 3])
def test_overclamped_end_knot_rejected(p):
    """A (p+2)-fold end knot is not a clamped knot vector of degree p (the
    curve's end points would not be P_0 / P_n): rejected, not decomposed into
    a bogus extra segment (e.g. p=1, U=[0,0,1,1,1])."""
    if p == 1:
        P = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]])
        U = np.array([0.0, 0.0, 1.0, 1.0, 1.0])
    else:
        P = np.random.default_rng(3).uniform(-1, 1, size=(6, 2))
        U = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 0.5, 1.0, 1.0, 1.0, 1.0])   # 5-fold start knot
    with pytest.raises(ValueError):
        oracle.nurbs_decompose(p, P, None, U)
