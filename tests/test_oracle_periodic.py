"""Oracle pins for the periodic machinery (Sec. 4.3-4.5, App. B/C):
homology, line / extended-curve worked values, uni-contractible translates,
bi-periodic strip, Eq. 5 N vs 2N, tile periodicity, pairing, and the C3
torus closed form."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests import helpers as H
from wn_workloads import configs as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))


@pytest.mark.parametrize("case", GOLD["homology"])
def test_homology_examples(case):
    s, e = np.array(case["start"]), np.array(case["end"])
    T = case["T"]
    # a two-segment loop start -> mid -> end, stored seam-discontinuously:
    mid = 0.5 * (s + e)
    seg1 = np.stack([s, mid])
    seg2 = np.stack([mid, e])
    k = np.floor(mid / T)
    seg2s = seg2 - k * np.array(T)        # store second segment wrapped
    wl = H.make_wl([([[(seg1, None), (seg2s, None)]], 3, (0.0, T[0], 0.0, T[1]))])
    sh, cl, bb = oracle.lift(wl)
    assert tuple(cl[0]) == tuple(case["class"])
    assert tuple(sh[1]) == tuple(k.astype(int))


def test_lift_generated_classes():
    wl = G.gen_c3(n_queries=10)
    sh, cl, bb = oracle.lift(wl)
    assert [tuple(c) for c in cl] == [(1, 0), (-1, 0), (0, 0), (0, 0), (0, 0)]
    # lifted loops are continuous: every junction bit-identical (Q40 data)
    wl5 = G.gen_c5(n_faces=40, grid=4)
    sh5, cl5, _ = oracle.lift(wl5)
    fo, lo = wl5["face_loop_off"], wl5["loop_seg_off"]
    for f in range(len(fo) - 1):
        cls = [tuple(cl5[l]) for l in range(fo[f], fo[f + 1])]
        if wl5["face_periodic"][f]:
            nc = [c for c in cls if c != (0, 0)]
            assert sorted(nc) in ([], [(-1, 0), (1, 0)])
        else:
            assert all(c == (0, 0) for c in cls)


def _uni_face(loops, T=1.0):
    return (loops, 1, (0.0, T, 0.0, 1.0))


@pytest.mark.parametrize("case", GOLD["line"])
def test_extended_straight_segment(case):
    b, v = np.array(case["base"]), np.array(case["v"])
    loop = H.line_loop(b, b + v, n=3)
    wl = H.make_wl([_uni_face([loop])], [case["p"]])
    r = oracle.query(wl, strict=False)      # a lone extended curve is a primitive, not a valid face
    assert r["w"][0] == pytest.approx(case["omega"], abs=1e-14)
    assert oracle.query(wl)["face_err"][0] == 2   # Prop. 1: unbalanced set rejected when strict


@pytest.mark.parametrize("case", GOLD["uni_contractible_circle"])
def test_uni_contractible_circle(case):
    arcs = H.circle_arcs(case["center"], case["r"], ccw=True)
    wl = H.make_wl([_uni_face([arcs])], [case["p"]])
    r = oracle.query(wl, reduce=False)
    assert r["w"][0] == pytest.approx(case["omega"], abs=1e-12)


@pytest.mark.parametrize("shift_beta", [0, -1, 1])
@pytest.mark.parametrize("case", GOLD["bi_strip"])
def test_bi_periodic_strip(case, shift_beta):
    """Strip between v=0.25 (rightward) and v=0.75 (leftward), both axes of
    period 1; beta optionally stored one tile off so that pairing (Algs. 7-9)
    must find the proper translate."""
    a, b = case["lines_v"]
    alpha = H.line_loop((0.0, a), (1.0, a), n=2)
    beta = [(P + np.array([0.0, shift_beta]), w) for P, w in H.line_loop((1.0, b), (0.0, b), n=2)]
    beta = [(P - np.array([np.floor(P[0, 0]), 0.0]), w) for P, w in beta]  # store wrapped in u
    wl = H.make_wl([([alpha, beta], 3, (0.0, 1.0, 0.0, 1.0))], [case["p"]])
    r = oracle.query(wl)
    assert r["face_err"][0] == 0
    assert r["w"][0] == pytest.approx(case["omega"], abs=1e-12)


@pytest.mark.parametrize("exact", [True, False])
def test_eq5_N_vs_2N_and_tile_periodicity(exact):
    """exact=False: generic fp64 periodic data (T = 2 pi as a plain double,
    segments stored at random lattice translates): lifted junctions at seam
    crossings are not bit-continuous, the loops' closures carry ulp-size
    defects; Eq. 5 still converges and values stay integers to ~1e-12 away
    from the curves."""
    wl = G.gen_c5(n_faces=30, grid=6, exact=exact, store_jitter=0 if exact else 2)
    per = np.nonzero(wl["face_periodic"])[0]
    assert len(per) >= 3
    m = np.isin(wl["face_id"], per)
    fid, q = wl["face_id"][m], wl["uv"][m]
    r1 = oracle.query(wl, face_id=fid, uv=q, N5=4)
    r2 = oracle.query(wl, face_id=fid, uv=q, N5=8)
    ok = r1["comparable"] & r2["comparable"]
    assert ok.mean() > 0.9
    assert np.max(np.abs(r1["w"][ok] - r2["w"][ok])) < (1e-13 if exact else 1e-11)
    # far truncations (N = 64 against 128) agree with the default N = 8:
    # Eq. 5 does not depend on where the copies are cut off
    r64 = oracle.query(wl, face_id=fid, uv=q, N5=64)
    r128 = oracle.query(wl, face_id=fid, uv=q, N5=128)
    okN = ok & r64["comparable"] & r128["comparable"]
    assert okN.mean() > 0.9
    assert np.max(np.abs(r64["w"][okN] - r128["w"][okN])) < (1e-12 if exact else 1e-10)
    assert np.max(np.abs(r2["w"][okN] - r128["w"][okN])) < (1e-12 if exact else 1e-10)
    # tile periodicity: the unreduced point one period away gives the same value
    T = wl["face_domain"][fid, 1]
    r3 = oracle.query(wl, face_id=fid, uv=q + np.stack([T, 0 * T], 1), reduce=False)
    ok &= r3["comparable"]
    assert np.max(np.abs(r1["w"][ok] - r3["w"][ok])) < 1e-9
    # and every comparable value is an integer (closed / balanced loops)
    assert np.max(np.abs(r1["w"][ok] - np.round(r1["w"][ok]))) < (1e-12 if exact else 1e-10)


def test_c3_pairing_finds_proper_translate():
    wl = G.gen_c3(n_queries=10)
    pr, ps, fe = oracle.pairs(wl)
    assert fe[0] == 0
    assert pr[0] == 1 and tuple(ps[0]) == (0, 1)   # beta lifted +1 tile in v sits above alpha


def _graph_v(segs, u, T):
    """v of a graph loop (monotone in u) at u, searched over lattice copies."""
    for P, w in segs:
        for k in (-2, -1, 0, 1, 2):
            Pk = P + np.array([k * T, 0.0])
            lo, hi = sorted((Pk[0, 0], Pk[-1, 0]))
            if lo <= u <= hi:
                ta, tb = 0.0, 1.0
                inc = Pk[-1, 0] > Pk[0, 0]
                for _ in range(70):
                    tm = 0.5 * (ta + tb)
                    x = H.bern_eval(Pk, w, tm)[0, 0]
                    if (x < u) == inc:
                        ta = tm
                    else:
                        tb = tm
                return H.bern_eval(Pk, w, 0.5 * (ta + tb))[0, 1]
    raise RuntimeError


@pytest.mark.parametrize("exact", [True, False])
def test_c3_torus_closed_form(exact):
    """C3 analytic classification: inside iff in the band between
    alpha (v = f_a(u)) and the proper translate of beta (v = f_b(u) + T),
    modulo the lattice, minus the two CW holes, plus the CCW island.
    exact=False: generic fp64 data (T = 2 pi plain, random storage translates;
    lifted junctions not bit-continuous): the ulp-size gaps perturb the value
    by at most ~defect / (2 pi distance), so the pin uses a 1e-5 margin and a
    1e-9 tolerance there."""
    wl = G.gen_c3(n_queries=600, exact=exact, store_jitter=0 if exact else 2)
    meta = wl["meta"]
    T = meta["T"]
    rng = np.random.default_rng(5)
    q = wl["uv"]
    r = oracle.query(wl)
    alpha = meta["alpha_knots"]
    beta = meta["beta_knots"]
    n_ok = 0
    for i, p in enumerate(q):
        fa = _graph_v(alpha, p[0], T)
        fb = _graph_v(beta, p[0], T)          # lifted beta: ~ T + 1.7
        v = p[1]
        inband = any(fa < v + k * T < fb for k in (-1, 0, 1))
        marg = min(abs(v + k * T - f) for k in (-1, 0, 1) for f in (fa, fb))
        total = 1 if inband else 0
        for (c, rad, orient) in meta["circles"]:
            d = min(math.hypot(p[0] - c[0] - i_ * T, p[1] - c[1] - j_ * T) for i_ in (-1, 0, 1) for j_ in (-1, 0, 1))
            marg = min(marg, abs(d - rad))
            if d < rad:
                total += orient
        if marg > (1e-7 if exact else 1e-5) and r["comparable"][i]:
            assert abs(r["w"][i] - total) < (1e-12 if exact else 1e-9), (p, r["w"][i], total)
            n_ok += 1
    assert n_ok > 550


def _ext_gcd_rep(p, q, m):
    """A lattice translate (i, j) with p*j - q*i = m (brute force over a small box)."""
    for i in range(-abs(p) - 1, abs(p) + 2):
        for j in range(-abs(q) - 1, abs(q) + 2):
            if p * j - q * i == 1:
                return m * i, m * j
    raise RuntimeError


def _band_f(segs, tau, a0, v, nu0):
    """nu-offset of a band loop (a graph over tau: tau is monotone along every
    Hermite segment) at band-coordinate tau, by bisection on the Bernstein form."""
    vv = float(v @ v)
    for P, w in segs:
        ta_, tb_ = ((P[[0, -1]] - a0) @ v) / vv
        lo, hi = min(ta_, tb_), max(ta_, tb_)
        if lo <= tau <= hi:
            a, b = 0.0, 1.0
            inc = tb_ > ta_
            for _ in range(70):
                tm = 0.5 * (a + b)
                x = H.bern_eval(P, w, tm)[0]
                if (((x - a0) @ v) / vv < tau) == inc:
                    a = tm
                else:
                    b = tm
            x = H.bern_eval(P, w, 0.5 * (a + b))[0]
            return nu0(x)
    raise RuntimeError(tau)


@pytest.mark.parametrize("pq,T,exact", [((2, 1), None, True), ((3, 2), None, True), ((1, -2), None, True),
                                        ((2, 3), (2 * math.pi, math.pi), True), ((3, -2), None, False),
                                        ((2, 3), (2 * math.pi, math.pi), False)])
def test_c3pq_general_class_closed_form(pq, T, exact):
    """General bi-periodic class (p,q) (Prop. 2, Eq. 8):
    the face interior is the band between alpha and the proper translate of
    beta, modulo the lattice, minus two CW holes plus one CCW island.  Band
    membership in band coordinates (tau along v, nu across), by bisection on
    the loops as graphs over tau -- independent of the oracle's Eq. 5/8 sums."""
    p, q = pq
    kw = {} if T is None else dict(Tu=T[0], Tv=T[1])
    wl = G.gen_c3pq(p=p, q=q, n_queries=250, exact=exact, store_jitter=0 if exact else 2, **kw)
    meta = wl["meta"]
    Tu, Tv, v, a0 = meta["Tu"], meta["Tv"], meta["v"], meta["a0"]
    s = float(np.linalg.norm(meta["w"]))
    nu = lambda x: p * x[1] / Tv - q * x[0] / Tu
    nu0 = lambda x: nu(x) - nu(a0)
    vv = float(v @ v)
    r = oracle.query(wl)
    n_ok = 0
    for k, x in enumerate(wl["uv"]):
        tx = float((x - a0) @ v) / vv
        nx = nu0(x)
        inband, marg = False, 1e9
        for m in range(int(math.floor(nx)) - 2, int(math.floor(nx)) + 3):
            i, j = _ext_gcd_rep(p, q, m)
            dt = (i * Tu * v[0] + j * Tv * v[1]) / vv
            t = tx - dt
            fa = _band_f(meta["alpha"], t - math.floor(t), a0, v, nu0)
            tb0 = ((meta["beta"][-1][0][-1] - a0) @ v) / vv      # beta's tau range [tb0, tb0 + 1]
            tt = t - math.floor(t - tb0)
            fb = _band_f(meta["beta"], tt, a0, v, nu0)
            if fa + m < nx < fb + m:
                inband = True
            marg = min(marg, abs(nx - fa - m) * s, abs(nx - fb - m) * s)
        total = 1 if inband else 0
        for c, rad, orient in meta["circles"]:
            i0, j0 = round((x[0] - c[0]) / Tu), round((x[1] - c[1]) / Tv)
            d = min(math.hypot(x[0] - c[0] - i_ * Tu, x[1] - c[1] - j_ * Tv)
                    for i_ in (i0 - 1, i0, i0 + 1) for j_ in (j0 - 1, j0, j0 + 1))
            marg = min(marg, abs(d - rad))
            if d < rad:
                total += orient
        if marg > (1e-7 if exact else 1e-5) and r["comparable"][k]:
            assert abs(r["w"][k] - total) < (1e-12 if exact else 1e-9), (x, r["w"][k], total)
            n_ok += 1
    assert n_ok > 230


@pytest.mark.parametrize("pq", [(2, 1), (-3, 2)])
def test_c3pq_tile_periodicity_and_pairing_invariance(pq):
    """omega(p) = omega(p + Tu e1) = omega(p + Tv e2) (unreduced), and the
    value does not depend on which lattice translate beta is stored at."""
    wl = G.gen_c3pq(p=pq[0], q=pq[1], n_queries=120)
    wl2 = G.gen_c3pq(p=pq[0], q=pq[1], n_queries=120, beta_shift=(3, -2))
    Tu, Tv = wl["meta"]["Tu"], wl["meta"]["Tv"]
    q = wl["uv"]
    r1 = oracle.query(wl)
    r2 = oracle.query(wl, uv=q + [Tu, 0.0], reduce=False)
    r3 = oracle.query(wl, uv=q + [0.0, -Tv], reduce=False)
    r4 = oracle.query(wl2)
    ok = r1["comparable"] & r2["comparable"] & r3["comparable"] & r4["comparable"]
    assert ok.mean() > 0.95
    for rr in (r2, r3, r4):
        assert np.max(np.abs(r1["w"][ok] - rr["w"][ok])) < 1e-9
    assert np.max(np.abs(r1["w"][ok] - np.round(r1["w"][ok]))) < 1e-12
    assert set(np.round(r1["w"][ok]).astype(int)) <= {-1, 0, 1}
