"""GPU <-> oracle parity on generic fp64 periodic data, the ABI's options and
the boundary's input-lifetime contract (-m gpu).

Generic periodic data (wn_workloads exact=False, store_jitter=2): periods 2 pi
and pi as plain doubles, unquantised control points, every segment stored at a
random lattice translate (R18).  Lifting x + k T then rounds, so junctions at
seam crossings are NOT bit-continuous and loop closures carry ulp-size
defects: the chain-break path (K_MOVEG gap terms), un-culled copies and open
contractible loops (CLOSEG) run here, in both angle modes, with the hierarchy
on and off (PAPER P:420-429 covering space, P:445-461 gamma(t+T) = gamma(t)+v,
P:463-483 Eq. 5, Eq. 8).

Options: rule = 1 ("positive", reading R10), the recursion depth
cap (R6; Lemma 2) and the on-boundary tolerance eps (Alg. 1 line 1
P:311; the paper's eps sweep P:765-774)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2510_25159_b200 as wn  # noqa: E402
from tests import helpers as H  # noqa: E402
from wn_workloads import configs as G  # noqa: E402

TOL64 = 1e-9
DELTA64 = 1e-9


def _gpu(wl, face_id=None, uv=None, **kw):
    faces = wn.Faces.from_workload(wl, **kw)
    r = faces.query(wl["face_id"] if face_id is None else face_id, wl["uv"] if uv is None else uv)
    torch.cuda.synchronize()
    out = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    info = faces.info()
    faces.close()
    return out[0], out[1], info


def _check(wl, w, fl, min_cmp=0.9, rule=0):
    r = oracle.query(wl, delta=DELTA64, tol=TOL64, rule=rule)
    cm = r["comparable"]
    assert cm.mean() >= min_cmp, cm.mean()
    assert not np.any(fl[cm] == 2), "GPU on-boundary on a certified-far query"
    assert not np.any(fl[cm] == 3)
    bad = np.nonzero(fl[cm] != r["flag"][cm])[0]
    assert bad.size == 0, (bad.size, w[cm][bad[:5]], r["w"][cm][bad[:5]])
    err = np.abs(w[cm] - r["w"][cm])
    assert err.max() <= TOL64, err.max()
    return r


def _breaks(wl):
    """Junctions that are not bit-continuous after the oracle's lifting."""
    sh, cl, _ = oracle.lift(wl)
    deg = wl["seg_degree"]
    off = np.concatenate([[0], np.cumsum(deg + 1)])
    P, lo, fo = wl["ctrl_uv"], wl["loop_seg_off"], wl["face_loop_off"]
    dom, per = wl["face_domain"], wl["face_periodic"]
    face_of = np.searchsorted(fo, np.arange(len(lo) - 1), side="right") - 1
    n = 0
    for l in range(len(lo) - 1):
        f = face_of[l]
        for s in range(lo[l] + 1, lo[l + 1]):
            a = P[off[s] - 1].copy()
            b = P[off[s]].copy()
            for ax in (0, 1):
                if per[f] >> ax & 1:
                    a[ax] = a[ax] + sh[s - 1, ax] * dom[f, 1 + 2 * ax]
                    b[ax] = b[ax] + sh[s, ax] * dom[f, 1 + 2 * ax]
            n += int(not np.array_equal(a, b))
    return n


@pytest.mark.parametrize("angle_mode,hierarchy", [(0, True), (1, True), (0, False), (1, False)])
def test_c3_generic_fp64(angle_mode, hierarchy):
    wl = G.gen_c3(n_queries=40_000, exact=False, store_jitter=2)
    assert _breaks(wl) > 5              # the chain-break path really runs
    w, fl, info = _gpu(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    _check(wl, w, fl, min_cmp=0.99)
    assert info["n_bands"] > 0 and info["n_copy_groups"] > 0


def test_c3_generic_full_size_sampled():
    """C3 at BASELINE size (1M queries), generic data, bench launch configuration."""
    wl = G.gen_c3(exact=False, store_jitter=2)
    w, fl, _ = _gpu(wl)
    idx = np.random.default_rng(4).choice(len(w), 40_000, replace=False)
    wl2 = dict(wl)
    wl2["face_id"], wl2["uv"] = wl["face_id"][idx], wl["uv"][idx]
    _check(wl2, w[idx], fl[idx], min_cmp=0.99)


@pytest.mark.parametrize("angle_mode,hierarchy", [(0, True), (1, True), (0, False), (1, False)])
def test_c5_generic_reduced(angle_mode, hierarchy):
    wl = G.gen_c5(n_faces=200, grid=24, exact=False, store_jitter=2)
    assert _breaks(wl) > 50
    w, fl, info = _gpu(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    _check(wl, w, fl, min_cmp=0.97)
    assert info["n_copy_groups"] > 0 and info["n_bands"] == 0


@pytest.mark.parametrize("pq,angle_mode,hierarchy", [((2, 1), 0, True), ((3, -2), 1, True), ((3, -2), 0, False),
                                                      ((1, 2), 1, False)])
def test_c3pq_generic(pq, angle_mode, hierarchy):
    wl = G.gen_c3pq(p=pq[0], q=pq[1], n_queries=10_000, exact=False, store_jitter=2, beta_shift=(2, -1))
    w, fl, _ = _gpu(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    _check(wl, w, fl, min_cmp=0.99)


def test_generic_periodic_reduction_equals_in_tile():
    """Queries given one period away (unreduced) equal the in-tile queries on
    generic data too (reduction into the base tile)."""
    wl = G.gen_c3(n_queries=4000, exact=False, store_jitter=2)
    T = wl["meta"]["T"]
    w, fl, _ = _gpu(wl)
    w2, fl2, _ = _gpu(wl, uv=wl["uv"] + np.array([T, -2 * T]))
    ok = fl != 2
    assert np.array_equal(fl[ok], fl2[ok])
    assert np.max(np.abs(w[ok] - w2[ok])) < 1e-9


# ----------------------------------------------------------------------------
# options of wn_options_t
# ----------------------------------------------------------------------------

def _reversed(wl):
    """Every loop reversed (segments in reverse order, each reversed): omega -> -omega."""
    out = dict(wl)
    deg = wl["seg_degree"]
    off = np.concatenate([[0], np.cumsum(deg + 1)])
    lo = wl["loop_seg_off"]
    ctrl, wts, degs = [], [], []
    for l in range(len(lo) - 1):
        for s in range(lo[l + 1] - 1, lo[l] - 1, -1):
            ctrl.append(wl["ctrl_uv"][off[s]:off[s + 1]][::-1])
            if wl["ctrl_w"] is not None:
                wts.append(wl["ctrl_w"][off[s]:off[s + 1]][::-1])
            degs.append(deg[s])
    out["ctrl_uv"] = np.ascontiguousarray(np.concatenate(ctrl))
    out["ctrl_w"] = np.ascontiguousarray(np.concatenate(wts)) if wts else None
    out["seg_degree"] = np.asarray(degs, np.int32)
    return out


def test_rule_positive():
    """rule = 1 (positive: round(w) >= 1) vs rule = 0 (nonzero) on a face whose
    loops are all reversed (omega = -1 inside): nonzero says inside, positive
    says outside; both match the oracle under the same rule."""
    wl = _reversed(G.gen_c2(n_queries=40_000))
    w0, f0, _ = _gpu(wl, rule=0)
    w1, f1, _ = _gpu(wl, rule=1)
    r0 = _check(wl, w0, f0, min_cmp=0.85, rule=0)
    r1 = _check(wl, w1, f1, min_cmp=0.85, rule=1)
    cm = r0["comparable"]
    neg = cm & (np.round(r0["w"]) == -1)
    assert neg.sum() > 1000
    assert np.all(f0[neg] == 1) and np.all(f1[neg] == 0)
    assert np.array_equal(w0[cm], w1[cm])                 # the rule changes the flag only
    # the unreversed face: positive and nonzero agree (omega in {0, 1})
    wl2 = G.gen_c2(n_queries=20_000)
    wa, fa, _ = _gpu(wl2, rule=1)
    _check(wl2, wa, fa, min_cmp=0.85, rule=1)


def test_depth_cap():
    """max_depth (R6): pairs whose recursion would go deeper than the cap report
    on-boundary (flag 2); every other query still matches the oracle; the
    number of capped queries does not grow with the cap, and at a cap above
    the deepest recursion of the batch none remain."""
    wl = G.gen_c2(n_queries=30_000)
    faces = wn.Faces.from_workload(wl)
    faces.set_counters(True)
    faces.query(wl["face_id"], wl["uv"])
    dmax = faces.counters()["max_depth"]
    faces.close()
    assert 8 < dmax < 48
    prev = None
    for cap in (4, 8, 12, dmax - 1, dmax):
        w, fl, _ = _gpu(wl, max_depth=cap)
        n2 = int((fl == 2).sum())
        r = oracle.query(wl, delta=DELTA64, tol=TOL64)
        cm = r["comparable"] & (fl != 2)
        assert np.array_equal(fl[cm], r["flag"][cm])
        assert np.max(np.abs(w[cm] - r["w"][cm])) <= TOL64
        assert np.all(np.isnan(w[fl == 2]))
        if prev is not None:
            assert n2 <= prev
        prev = n2
        if cap == 4:
            assert n2 > 0
        if cap == dmax:
            assert not np.any(fl[r["comparable"]] == 2)
        if cap == dmax - 1:
            assert n2 > 0


def test_eps_sweep_on_boundary_fraction():
    """The on-boundary tolerance eps (Alg. 1 line 1) swept as in the
    paper's Fig. on C2 (10% of the points within 1e-6 of a curve):
    the on-boundary fraction does not increase as eps decreases and vanishes
    at 1e-10 on the uniform points; a query is flagged only if the oracle's
    certified distance lower bound is below eps, and never when it is above;
    every other comparable query matches the oracle."""
    wl = G.gen_c2(n_queries=60_000)
    near = wl["meta"]["near_mask"]
    r = oracle.query(wl, delta=DELTA64, tol=TOL64)
    dl = r["dist_lb"]
    fracs = []
    for eps in (1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-10):
        w, fl, _ = _gpu(wl, eps=eps)
        onb = fl == 2
        fracs.append(onb.mean())
        assert np.all(dl[onb] < eps * (1 + 1e-9) + 1e-15), eps        # flagged => within eps of the curve
        assert not np.any(onb & (dl > eps * (1 + 1e-6))), eps           # farther than eps => not flagged
        cm = r["comparable"] & ~onb
        assert np.array_equal(fl[cm], r["flag"][cm])
        assert np.max(np.abs(w[cm] - r["w"][cm])) <= TOL64
    assert all(a >= b for a, b in zip(fracs, fracs[1:])), fracs
    assert fracs[0] > fracs[-1]
    w, fl, _ = _gpu(wl, eps=1e-10)
    assert not np.any(fl[~near] == 2)


# ----------------------------------------------------------------------------
# boundary: inputs may be freed / overwritten as soon as wn_build_faces returns
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("gen", ["c5", "c3"])
def test_inputs_clobbered_after_build(gen):
    """"Inputs may be freed after it returns".  The caller's device
    arrays are overwritten with garbage on ANOTHER stream right after
    wn_build_faces returns (no synchronisation with the build's stream); the
    handle's results still match the oracle."""
    wl = (G.gen_c5(n_faces=300, grid=16, exact=False, store_jitter=1) if gen == "c5"
          else G.gen_c3(n_queries=20_000, exact=False, store_jitter=2))
    dev = torch.device("cuda", 0)
    T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    geo = [T(wl["ctrl_uv"], torch.float64), T(wl["ctrl_w"], torch.float64), T(wl["seg_degree"], torch.int32),
           T(wl["loop_seg_off"], torch.int32), T(wl["face_loop_off"], torch.int32),
           T(wl["face_periodic"], torch.uint8), T(wl["face_domain"], torch.float64)]
    torch.cuda.synchronize()
    build_stream = torch.cuda.Stream(dev)
    side = torch.cuda.Stream(dev)
    faces = wn.Faces.build(*geo, stream=build_stream)
    with torch.cuda.stream(side):                     # not ordered after the build's stream
        geo[0].fill_(float("nan"))
        geo[1].fill_(-1.0)
        geo[2].fill_(9)
        geo[3].fill_(-7)
        geo[4].fill_(1 << 30)
        geo[5].fill_(255)
        geo[6].fill_(float("inf"))
    side.synchronize()
    with torch.cuda.stream(build_stream):
        r = faces.query(wl["face_id"], wl["uv"])
    build_stream.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    _check(wl, w, fl, min_cmp=0.97)


def test_nurbs_overclamped_end_knot_rejected():
    """A (p+2)-fold end knot is rejected by the device validation (WN_ERR_GEOM)
    like the oracle rejects it, instead of producing a bogus segment."""
    P = np.array([[0.2, 0.2], [0.8, 0.2], [0.8, 0.8], [0.2, 0.8], [0.2, 0.2]])
    with pytest.raises(wn.WNError) as e:
        wn.nurbs_to_bezier(P, None, np.array([1], np.int32), np.array([0, 5], np.int32),
                           np.array([0.0, 0.0, 0.3, 0.6, 1.0, 1.0, 1.0]), np.array([0, 7], np.int32))
    assert e.value.status == 2
    with pytest.raises(ValueError):
        oracle.nurbs_decompose(1, P, None, np.array([0.0, 0.0, 0.3, 0.6, 1.0, 1.0, 1.0]))


@pytest.mark.parametrize("precision", [0, 1])
def test_recursion_bounds_sound(precision):
    """The bounds the shipped recursion uses (BaseCold written by K1 in the
    build, read back with wn_recursion_bounds) are sound: B >= max |gamma'|,
    every piece bound Bq[q] >= max |gamma'| on [q/8, (q+1)/8] and every
    tabulated depth-1..3 node span >= the node's arc length (Lemma 1 P:335-345,
    Eq. 2, R9, R29), by dense sampling with the oracle's evaluation
    and derivative (2048 intervals)."""
    rng = np.random.default_rng(17 + precision)
    segs = []
    for _ in range(200):
        n = int(rng.integers(1, 6))
        P = rng.uniform(-1, 1, size=(n + 1, 2))
        w = rng.uniform(0.5, 2.0, size=n + 1) if rng.random() < 0.8 else np.exp(rng.uniform(-3, 3, n + 1))
        segs.append((P, w))
    # one open loop of unrelated segments (a valid, if odd, face: gaps are chain breaks)
    wl = H.make_wl([([segs], 0, (0, 1, 0, 1))])
    faces = wn.Faces.from_workload(wl, precision=precision)
    rb = faces.recursion_bounds(len(segs)).cpu().numpy()
    faces.close()
    ts = np.linspace(0, 1, 2049)
    for (P, w), row in zip(segs, rb):
        sp = np.array([np.hypot(*oracle.derivative(P, w, t)) for t in ts])
        pts = np.array([oracle.evaluate(P, w, t) for t in ts])
        arc = np.hypot(*np.diff(pts, axis=0).T)
        assert row[0] >= sp.max() * (1 - 1e-12)
        for q in range(8):
            m = (ts >= q / 8) & (ts <= (q + 1) / 8)
            assert row[1 + q] >= sp[m].max() * (1 - 1e-12), (q, row[1 + q], sp[m].max())
        for d in (1, 2, 3):
            L = 2048 >> d
            for k in range(1 << d):
                assert row[9 + (1 << d) - 2 + k] >= arc[k * L:(k + 1) * L].sum() * (1 - 1e-9), (d, k)


def test_unaligned_flag_output():
    """An output flag array at an odd address (k_finish's scalar path) gives
    the same results as an aligned one, with parity against the oracle."""
    wl = G.gen_c2(n_queries=30_000)
    faces = wn.Faces.from_workload(wl)
    n = len(wl["face_id"])
    wbuf = torch.empty(n, dtype=torch.float64, device="cuda")
    fbuf = torch.empty(n + 1, dtype=torch.uint8, device="cuda")[1:]     # odd address
    r = faces.query(wl["face_id"], wl["uv"], out=(wbuf, fbuf))
    r2 = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    assert np.array_equal(fl, r2.flag.cpu().numpy())
    faces.close()
    _check(wl, w, fl, min_cmp=0.85)


def test_bad_period_rejected():
    """A periodic axis needs a finite start and a finite period > 0 (device-side
    input validation, WN_ERR_GEOM naming the first bad face and axis)."""
    wl = G.gen_c3(n_queries=10)
    for bad in ((0.0, 0.0, 0.0, wl["meta"]["T"]), (0.0, wl["meta"]["T"], np.nan, wl["meta"]["T"]),
                (0.0, -1.0, 0.0, 1.0)):
        w2 = dict(wl)
        w2["face_domain"] = np.array([bad], dtype=np.float64)
        with pytest.raises(wn.WNError) as e:
            wn.Faces.from_workload(w2)
        assert e.value.status == 2 and "period" in str(e.value)
