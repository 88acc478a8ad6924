"""Pins of the oracle's primitives against values fixed by the paper / SPEC and
against independent textbook constructions (tests/helpers.py).  -m "not gpu"."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests import helpers as H

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))


@pytest.mark.parametrize("case", GOLD["chord"])
def test_chord_worked_values(case):
    assert oracle.chord(case["p"], case["a"], case["b"]) == pytest.approx(case["omega"], abs=1e-15)


def test_chord_antisymmetry_and_range():
    rng = np.random.default_rng(0)
    for _ in range(200):
        p, a, b = rng.normal(size=(3, 2))
        w1 = oracle.chord(p, a, b)
        w2 = oracle.chord(p, b, a)
        assert -0.5 < w1 <= 0.5
        assert w1 == pytest.approx(-w2, abs=1e-15)


@pytest.mark.parametrize("case", GOLD["eval"])
def test_eval_worked_values(case):
    pt = oracle.evaluate(np.array(case["P"], float), case["w"], case["t"])
    assert np.allclose(pt, case["pt"], atol=1e-15)


def test_eval_endpoints_exact_and_vs_bernstein():
    rng = np.random.default_rng(1)
    for n in range(1, 6):
        for _ in range(20):
            P = rng.uniform(-1, 1, size=(n + 1, 2))
            w = rng.uniform(0.5, 2.0, size=n + 1)
            assert np.array_equal(oracle.evaluate(P, w, 0.0), P[0])
            assert np.array_equal(oracle.evaluate(P, w, 1.0), P[n])
            for t in rng.uniform(0, 1, size=5):
                assert np.allclose(oracle.evaluate(P, w, t), H.bern_eval(P, w, t)[0], atol=1e-13)


def test_rational_quadratic_arc_on_circle():
    # closed form: weights (1, cos(a/2), 1) with the tangent-intersection middle
    # control point give an exact circular arc of angle a
    for a in (0.3, 1.0, math.pi / 2, 2.5):
        r, c = 0.7, np.array([0.2, -0.1])
        P0 = c + r * np.array([1.0, 0.0])
        P2 = c + r * np.array([math.cos(a), math.sin(a)])
        P1 = c + (r / math.cos(a / 2)) * np.array([math.cos(a / 2), math.sin(a / 2)])
        P = np.stack([P0, P1, P2])
        w = np.array([1.0, math.cos(a / 2), 1.0])
        for t in np.linspace(0, 1, 17):
            q = oracle.evaluate(P, w, t)
            assert abs(np.hypot(*(q - c)) - r) < 1e-14


def test_derivative_vs_finite_difference():
    rng = np.random.default_rng(2)
    for n in range(1, 6):
        P = rng.uniform(-1, 1, size=(n + 1, 2))
        w = rng.uniform(0.5, 2.0, size=n + 1)
        for t in (0.1, 0.37, 0.5, 0.9):
            h = 1e-6
            fd = (H.bern_eval(P, w, t + h)[0] - H.bern_eval(P, w, t - h)[0]) / (2 * h)
            assert np.allclose(oracle.derivative(P, w, t), fd, atol=1e-7)


def test_segment_winding_far_point_is_chord():
    P = np.array([[0.0, 0.0], [0.3, 0.4], [0.7, -0.2], [1.0, 0.0]])
    val, near, dl, pieces = oracle.segment_winding(P, None, (0.5, 3.0))
    assert pieces == 1 and not near
    assert val == oracle.chord((0.5, 3.0), P[0], P[-1])


def test_segment_winding_vs_dense_polyline():
    """brute force by a dense polyline (1e5 pieces) for
    points at distance >= 0.01 from the curve, within 1e-6."""
    rng = np.random.default_rng(3)
    checked = 0
    for _ in range(40):
        n = int(rng.integers(1, 6))
        P = rng.uniform(0, 1, size=(n + 1, 2))
        w = rng.uniform(0.5, 2.0, size=n + 1)
        pts = H.bern_eval(P, w, np.linspace(0, 1, 100001))
        for p in rng.uniform(-0.2, 1.2, size=(5, 2)):
            if np.min(np.hypot(*(pts - p).T)) < 0.01:
                continue
            val, near, dl, _ = oracle.segment_winding(P, w, p)
            assert not near
            assert abs(val - H.polyline_wn(pts, p)) < 1e-6
            checked += 1
    assert checked > 50


def test_segment_winding_near_point_certificate():
    P = np.array([[0.0, 0.0], [0.5, 1.0], [1.0, 0.0]])
    on = H.bern_eval(P, None, 0.3)[0]
    val, near, dl, _ = oracle.segment_winding(P, None, on, delta=1e-9)
    assert near  # a point on the curve can never be certified
    val, near, dl, _ = oracle.segment_winding(P, None, on + np.array([0.0, 1e-6]), delta=1e-9)
    assert not near and dl > 1e-9
