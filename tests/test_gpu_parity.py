"""GPU <-> oracle parity through the C ABI (-m gpu).

Contract (BASELINE.json north_star): on every query the oracle
certifies as COMPARABLE (farther than delta from every curve, winding farther
than tol from a half-integer) the inside/outside flag is bit-exact and
|omega_gpu - omega_oracle| <= 1e-9 (fp64) / 1e-4 (fp32, oracle on the fp32-
rounded inputs, R19); the GPU never reports on-boundary there."""
import numpy as np
import pytest
import torch

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2510_25159_b200 as wn  # noqa: E402
from tests import helpers as H  # noqa: E402
from wn_workloads import configs as G  # noqa: E402

TOL64, TOL32 = 1e-9, 1e-4
DELTA64, DELTA32 = 1e-9, 1e-5


def _gpu(wl, face_id=None, uv=None, **kw):
    faces = wn.Faces.from_workload(wl, **kw)
    r = faces.query(wl["face_id"] if face_id is None else face_id, wl["uv"] if uv is None else uv)
    torch.cuda.synchronize()
    out = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    return out


def _check(wl, w, fl, idx=None, fp32=False, min_cmp=0.9, **okw):
    fid = wl["face_id"] if idx is None else wl["face_id"][idx]
    uv = wl["uv"] if idx is None else wl["uv"][idx]
    delta, tol = (DELTA32, TOL32) if fp32 else (DELTA64, TOL64)
    r = oracle.query(wl, face_id=fid, uv=uv, delta=delta, tol=tol, **okw)
    if idx is not None:
        w, fl = w[idx], fl[idx]
    cm = r["comparable"]
    assert cm.mean() >= min_cmp, cm.mean()
    assert not np.any(fl[cm] == 2), "GPU on-boundary on a certified-far query"
    assert not np.any(fl[cm] == 3)
    bad = np.nonzero(fl[cm] != r["flag"][cm])[0]
    assert bad.size == 0, (bad.size, w[cm][bad[:5]], r["w"][cm][bad[:5]], uv[cm][bad[:5]])
    err = np.abs(w[cm] - r["w"][cm])
    assert err.max() <= tol, (err.max(), uv[cm][np.argmax(err)])
    return err.max(), cm.mean()


@pytest.mark.parametrize("angle_mode", [0, 1])
def test_c1_full(angle_mode):
    wl = G.gen_c1()
    w, fl = _gpu(wl, angle_mode=angle_mode)
    _check(wl, w, fl, min_cmp=0.999)


@pytest.mark.parametrize("angle_mode,hierarchy", [(0, True), (1, True), (0, False)])
def test_c2_sampled(angle_mode, hierarchy):
    wl = G.gen_c2(n_queries=60_000)
    w, fl = _gpu(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    _check(wl, w, fl, min_cmp=0.85)
    # the near-curve shell (1e-6) is part of the batch
    assert wl["meta"]["near_mask"].sum() > 5000


def test_c2_full_size_sampled():
    """BASELINE configs[1] at full size (1M queries) in the bench launch
    configuration; the oracle checks a 40k sample."""
    wl = G.gen_c2()
    w, fl = _gpu(wl)
    idx = np.random.default_rng(0).choice(len(w), 40_000, replace=False)
    _check(wl, w, fl, idx=idx, min_cmp=0.85)
    assert np.all(fl != 3)


@pytest.mark.parametrize("angle_mode,hierarchy", [(0, True), (1, True), (0, False)])
def test_c3_torus(angle_mode, hierarchy):
    wl = G.gen_c3(n_queries=20_000)
    w, fl = _gpu(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    _check(wl, w, fl, min_cmp=0.99)


def test_c4_fp64():
    wl = G.gen_c4(n_faces=200, n_deleted=20)
    w, fl = _gpu(wl)
    _check(wl, w, fl, min_cmp=0.95)


def test_c4_fp32():
    wl = G.to_fp32_inputs(G.gen_c4(n_faces=200, n_deleted=20))
    w, fl = _gpu(wl, precision=1)
    _check(wl, w, fl, fp32=True, min_cmp=0.95)


@pytest.mark.parametrize("angle_mode,hierarchy", [(0, True), (1, True), (0, False), (1, False)])
def test_c5_reduced(angle_mode, hierarchy):
    wl = G.gen_c5(n_faces=120, grid=32)
    w, fl = _gpu(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    _check(wl, w, fl, min_cmp=0.97)


def test_c5_full_size_sampled():
    """BASELINE configs[4] at full size (20,000 faces x 64x64 grid = 81.92M
    queries), sampled oracle check."""
    wl = G.gen_c5()
    w, fl = _gpu(wl)
    idx = np.random.default_rng(1).choice(len(w), 20_000, replace=False)
    _check(wl, w, fl, idx=idx, min_cmp=0.97)


def test_c3_full_size_sampled():
    """BASELINE configs[2] at full size (1M queries on the bi-periodic torus),
    sampled oracle check."""
    wl = G.gen_c3()
    w, fl = _gpu(wl)
    assert np.all(fl != 3)
    idx = np.random.default_rng(2).choice(len(w), 20_000, replace=False)
    _check(wl, w, fl, idx=idx, min_cmp=0.99)


@pytest.mark.parametrize("fp32", [False, True])
def test_c4_full_size_sampled(fp32):
    """BASELINE configs[3] at full size (1,000 gapped / open loops, 256k
    queries), fp64 and fp32 (oracle on the fp32-rounded inputs, R19), sampled."""
    wl = G.gen_c4()
    if fp32:
        wl = G.to_fp32_inputs(wl)
    w, fl = _gpu(wl, precision=1 if fp32 else 0)
    idx = np.random.default_rng(3).choice(len(w), 30_000, replace=False)
    _check(wl, w, fl, idx=idx, fp32=fp32, min_cmp=0.95)


# ----------------------------------------------------------------------------
# edge cases
# ----------------------------------------------------------------------------

def test_unsorted_batch_equals_sorted():
    wl = G.gen_c4(n_faces=50, q_per_face=300, n_deleted=5)   # 300: ragged tiles
    w, fl = _gpu(wl)
    perm = np.random.default_rng(2).permutation(len(w))
    w2, fl2 = _gpu(wl, face_id=wl["face_id"][perm], uv=wl["uv"][perm])
    assert np.array_equal(fl2, fl[perm])
    assert np.array_equal(np.isnan(w2), np.isnan(w[perm]))
    ok = ~np.isnan(w2)
    assert np.max(np.abs(w2[ok] - w[perm][ok])) < 1e-12


def test_invalid_queries_flag3_and_empty():
    wl = G.gen_c1(n_queries=100)
    fid = wl["face_id"].copy()
    uv = wl["uv"].copy()
    fid[3] = 7
    fid[5] = -1
    uv[9, 0] = np.nan
    w, fl = _gpu(wl, face_id=fid, uv=uv)
    assert fl[3] == 3 and fl[5] == 3 and fl[9] == 3
    assert np.isnan(w[3]) and np.isnan(w[9])
    assert np.all(fl[[0, 1, 2, 4, 6, 7, 8]] != 3)
    faces = wn.Faces.from_workload(wl)
    r = faces.query(np.zeros(0, np.int32), np.zeros((0, 2)))
    assert r.winding.numel() == 0


def test_on_boundary_exact_vertex():
    wl = G.gen_c1(n_queries=10)
    uv = wl["uv"].copy()
    uv[0] = wl["ctrl_uv"][0]          # a segment end point: d = 0 < eps (Alg. 1 line 1)
    w, fl = _gpu(wl, uv=uv)
    assert fl[0] == 2 and np.isnan(w[0])


def test_periodic_reduction_equals_in_tile():
    wl = G.gen_c3(n_queries=3000)
    T = wl["meta"]["T"]
    w, fl = _gpu(wl)
    shifted = wl["uv"] + np.array([T, -2 * T])
    w2, fl2 = _gpu(wl, uv=shifted)
    ok = fl != 2
    assert np.array_equal(fl[ok], fl2[ok])
    assert np.max(np.abs(w[ok] - w2[ok])) < 1e-9


def test_single_extended_curve_nonstrict():
    """Worked values S:301-302 / P:480-481 through the GPU (strict=0)."""
    loop = H.line_loop((0.0, 0.5), (1.0, 0.5), n=3)
    wl = H.make_wl([([loop], 1, (0.0, 1.0, 0.0, 1.0))], [(0.3, 0.8), (0.3, 0.2)])
    w, fl = _gpu(wl, strict=False)
    assert w[0] == pytest.approx(0.5, abs=1e-14) and w[1] == pytest.approx(-0.5, abs=1e-14)
    with pytest.raises(wn.WNError) as ei:
        wn.Faces.from_workload(wl)
    assert ei.value.status == 3 and ei.value.face_status[0] == 2


def test_bad_geometry_rejected():
    wl = G.gen_c1(n_queries=10)
    bad = dict(wl)
    bad["ctrl_w"] = np.ones(len(wl["ctrl_uv"]))
    bad["ctrl_w"][4] = -1.0
    with pytest.raises(wn.WNError) as ei:
        wn.Faces.from_workload(bad)
    assert ei.value.status == 2
    bad2 = dict(wl)
    bad2["seg_degree"] = wl["seg_degree"].copy()
    bad2["seg_degree"][0] = 7
    with pytest.raises(wn.WNError) as ei:
        wn.Faces.from_workload(bad2)
    assert ei.value.status == 1


@pytest.mark.gpu
def test_bad_csr_rejected_without_fault():
    # the device kernels run before the host validates the CSR offsets: they
    # must clamp every index (a fault here would poison the context)
    wl = G.gen_c2(n_queries=100)
    ns, nl = len(wl["seg_degree"]), len(wl["loop_seg_off"]) - 1
    for lso in (np.r_[wl["loop_seg_off"][:-1], ns + 1000],          # past the segment array
                np.r_[0, np.full(nl, -5)],                          # decreasing / negative
                np.r_[0, np.full(nl, 10 ** 9)]):
        bad = dict(wl)
        bad["loop_seg_off"] = lso.astype(np.int32)
        with pytest.raises(wn.WNError) as ei:
            wn.Faces.from_workload(bad)
        assert ei.value.status == 1
    nf = len(wl["face_loop_off"]) - 1
    bad = dict(wl)
    bad["face_loop_off"] = np.r_[0, np.full(nf, nl + 77)].astype(np.int32)
    with pytest.raises(wn.WNError):
        wn.Faces.from_workload(bad)
    # the context is still healthy
    faces = wn.Faces.from_workload(wl)
    r = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    assert r.flag.cpu().numpy().max() <= 3


def test_counters_and_info():
    wl = G.gen_c2(n_queries=20_000)
    faces = wn.Faces.from_workload(wl)
    faces.set_counters(True)
    faces.query(wl["face_id"], wl["uv"])
    c = faces.counters()
    info = faces.info()
    assert info["n_seg_records"] == 80
    assert c["pairs_tested"] > 0 and c["hard_pairs"] > 0 and c["max_depth"] <= 48
    assert wn.last_query_launches() >= 1


def test_k1_derivative_bounds_sound():
    """Lemma 1 soundness: B >= max |gamma'| sampled densely (oracle's
    derivative), every piece bound >= the sampled speed on its piece, and
    S0 >= the true arc length (so the root ellipse contains the curve)."""
    rng = np.random.default_rng(7)
    segs = []
    for _ in range(300):
        n = int(rng.integers(1, 6))
        P = rng.uniform(-1, 1, size=(n + 1, 2))
        w = rng.uniform(0.5, 2.0, size=n + 1) if rng.random() < 0.8 else np.exp(rng.uniform(-3, 3, n + 1))
        segs.append((P, w))
    wl = H.make_wl([([segs], 0, (0, 1, 0, 1))])
    out = wn.segment_prep(wl["ctrl_uv"], wl["ctrl_w"], wl["seg_degree"]).cpu().numpy()
    ts = np.linspace(0, 1, 2049)
    for (P, w), row in zip(segs, out):
        sp = np.array([np.hypot(*oracle.derivative(P, w, t)) for t in ts])
        assert row[0] >= sp.max() * (1 - 1e-12), (row[0], sp.max())
        for q in range(8):
            m = (ts >= q / 8) & (ts <= (q + 1) / 8)
            assert row[2 + q] >= sp[m].max() * (1 - 1e-12)
        pts = np.array([oracle.evaluate(P, w, t) for t in ts])
        seg = np.hypot(*np.diff(pts, axis=0).T)
        arc = seg.sum()
        assert row[1] >= arc * (1 - 1e-9)
        assert row[1] <= row[0] + 1e-15
        # piece polygon lengths bound the pieces' arc lengths (256 samples each)
        for q in range(8):
            assert row[10 + q] >= seg[q * 256:(q + 1) * 256].sum() * (1 - 1e-9)
        assert row[1] <= row[10:18].sum() * (1 + 1e-12)


def test_hard_pair_queue_overflow_path(monkeypatch):
    """Force the global hard-pair queue to overflow: the affected queries go
    through k_overflow and must still match the oracle."""
    monkeypatch.setenv("WN_HQ_CAP", "64")
    wl = G.gen_c2(n_queries=20_000)
    w, fl = _gpu(wl)
    _check(wl, w, fl, min_cmp=0.85)
    wl3 = G.gen_c3(n_queries=5_000)
    w, fl = _gpu(wl3)
    _check(wl3, w, fl, min_cmp=0.99)


@pytest.mark.gpu
def test_query_host_streamed_equals_device():
    """wn_query_host (chunked copy-in / query / copy-out on overlapping streams)
    gives exactly the device-resident query's results, for pinned and pageable
    inputs and chunk sizes that leave a ragged last chunk and reuse every slot."""
    wl = G.gen_c5(n_faces=300, grid=24, seed=11)
    faces = wn.Faces.from_workload(wl)
    ref = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    rw, rf = ref.winding.cpu().numpy(), ref.flag.cpu().numpy()
    n = len(wl["face_id"])
    for chunk, pin in ((0, True), (7777, True), (n // 3 + 1, False), (n, True)):
        fid = torch.from_numpy(wl["face_id"])
        uv = torch.from_numpy(wl["uv"])
        if pin:
            fid, uv = fid.pin_memory(), uv.pin_memory()
        r = faces.query_host(fid, uv, chunk=chunk)
        assert np.array_equal(r.flag.numpy(), rf), chunk
        assert np.array_equal(np.nan_to_num(r.winding.numpy(), nan=9.0), np.nan_to_num(rw, nan=9.0)), chunk
    # classification only (h_winding = NULL): the same flags, no winding copy
    r = faces.query_host(torch.from_numpy(wl["face_id"]).pin_memory(), torch.from_numpy(wl["uv"]).pin_memory(),
                         chunk=7777, winding=False)
    assert r.winding is None and np.array_equal(r.flag.numpy(), rf)
    faces.close()


@pytest.mark.parametrize("pq,angle_mode,hierarchy,dom", [
    ((2, 1), 0, True, None), ((2, 1), 1, True, None), ((3, 2), 0, True, None), ((3, 2), 0, False, None),
    ((1, -2), 0, True, None), ((-2, 3), 1, False, None), ((2, 3), 0, True, (6.283185307179586, 3.141592653589793)),
    ((5, 2), 0, True, None)])
def test_c3pq_general_class(pq, angle_mode, hierarchy, dom):
    """General bi-periodic classes (p,q) (Prop. 2, Eq. 8):
    slanted band lines, band copies along v, pairing over the band index."""
    kw = {} if dom is None else dict(Tu=dom[0], Tv=dom[1])
    wl = G.gen_c3pq(p=pq[0], q=pq[1], n_queries=8_000, **kw)
    w, fl = _gpu(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    _check(wl, w, fl, min_cmp=0.99)


def test_c3pq_beta_stored_off_tile():
    """Pairing must find the proper beta translate wherever beta is stored."""
    wl = G.gen_c3pq(p=3, q=-2, n_queries=6_000, beta_shift=(4, 3))
    w, fl = _gpu(wl)
    _check(wl, w, fl, min_cmp=0.99)


def _grid_uv(boxes, nu, nv):
    """Explicit uv of an implicit grid batch, by the formula include/wn.h documents."""
    out = []
    for b in np.asarray(boxes, dtype=np.float64).reshape(-1, 4):
        us = b[0] + (np.arange(nu) + 0.5) * ((b[2] - b[0]) / nu)
        vs = b[1] + (np.arange(nv) + 0.5) * ((b[3] - b[1]) / nv)
        U, V = np.meshgrid(us, vs)
        out.append(np.stack([U.ravel(), V.ravel()], 1))
    return np.concatenate(out)


@pytest.mark.parametrize("angle_mode", [0, 1])
def test_grid_query_c5_reduced(angle_mode):
    """wn_query_grid (implicit cell-centred grids, Sec. 5.4.3 tessellation,
    P:884-895) = wn_query on the explicit points, and parity with the oracle."""
    wl = G.gen_c5(n_faces=120, grid=32)
    gb = wl["meta"]["grid_box"]
    faces = wn.Faces.from_workload(wl, angle_mode=angle_mode)
    rg = faces.query_grid(np.arange(len(gb)), gb, 32, 32)
    re_ = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    wg, fg = rg.winding.cpu().numpy(), rg.flag.cpu().numpy()
    we, fe = re_.winding.cpu().numpy(), re_.flag.cpu().numpy()
    faces.close()
    assert np.array_equal(fg, fe)
    tol = 0.0 if angle_mode == 0 else 1e-12     # angle mode: atomic fp64 sums in any order
    assert np.nanmax(np.abs(wg - we)) <= tol
    _check(wl, wg, fg, min_cmp=0.97)


def test_grid_query_nonsquare_periodic_and_invalid():
    """Rectangular grids (nu != nv) on the C3 torus, an invalid face id and a
    non-finite box (flag 3), grids in any face order."""
    wl = G.gen_c3(n_queries=10)
    T = wl["meta"]["T"]
    boxes = np.array([[0.0, 0.0, T, T], [1.0, 2.0, 3.5, 2.5], [0.0, 0.0, 1.0, 1.0], [np.nan, 0.0, 1.0, 1.0]])
    gf = np.array([0, 0, 5, 0], dtype=np.int32)
    nu, nv = 37, 23
    faces = wn.Faces.from_workload(wl)
    r = faces.query_grid(gf, boxes, nu, nv)
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    G_ = nu * nv
    assert np.all(fl[2 * G_:] == 3) and np.all(np.isnan(w[2 * G_:]))
    uv = _grid_uv(boxes[:2], nu, nv)
    wl2 = dict(wl)
    wl2["face_id"] = np.zeros(len(uv), dtype=np.int32)
    wl2["uv"] = uv
    _check(wl2, w[:2 * G_], fl[:2 * G_], min_cmp=0.99)


def test_grid_query_c5_full_size_equals_explicit():
    """BASELINE configs[4] at full size: all 81.92M grid results equal the
    explicit-uv results (crossing mode: bit-identical)."""
    wl = G.gen_c5()
    gb = wl["meta"]["grid_box"]
    faces = wn.Faces.from_workload(wl)
    re_ = faces.query(wl["face_id"], wl["uv"])
    rg = faces.query_grid(np.arange(len(gb)), gb, 64, 64)
    torch.cuda.synchronize()
    assert torch.equal(rg.flag, re_.flag)
    assert torch.equal(rg.winding, re_.winding)
    faces.close()


def test_nurbs_decompose_matches_oracle():
    """wn_nurbs_to_bezier (device knot insertion) = the oracle's own
    decomposition: same segment counts and degrees, control points and weights
    to rounding, bit-exact curve ends and junctions."""
    wl = G.gen_nurbs(n_faces=60)
    cso, bz, bw, bd = wn.nurbs_to_bezier(wl["ctrl_uv"], wl["ctrl_w"], wl["curve_degree"], wl["curve_ctrl_off"],
                                         wl["knots"], wl["curve_knot_off"])
    torch.cuda.synchronize()
    cso, bz, bw, bd = cso.cpu().numpy(), bz.cpu().numpy(), bw.cpu().numpy(), bd.cpu().numpy()
    ref = oracle.nurbs_to_bezier_workload(wl)
    assert np.array_equal(bd, ref["seg_degree"])
    assert bz.shape == ref["ctrl_uv"].shape
    assert np.max(np.abs(bz - ref["ctrl_uv"])) < 1e-12
    assert np.max(np.abs(bw / ref["ctrl_w"] - 1.0)) < 1e-12
    # curve ends exact, consecutive segments share their junction bit for bit
    off = np.concatenate([[0], np.cumsum(bd + 1)])
    co = wl["curve_ctrl_off"]
    for c in range(len(wl["curve_degree"])):
        s0, s1 = cso[c], cso[c + 1]
        assert np.array_equal(bz[off[s0]], wl["ctrl_uv"][co[c]])
        assert np.array_equal(bz[off[s1] - 1], wl["ctrl_uv"][co[c + 1] - 1])
        for s in range(s0, s1 - 1):
            assert np.array_equal(bz[off[s + 1] - 1], bz[off[s + 1]])


@pytest.mark.parametrize("angle_mode,hierarchy", [(0, True), (1, False)])
def test_nurbs_faces_parity(angle_mode, hierarchy):
    """wn_build_faces_nurbs + wn_query vs the oracle on its own Bezier form."""
    wl = G.gen_nurbs(n_faces=150)
    faces = wn.Faces.from_nurbs_workload(wl, angle_mode=angle_mode, hierarchy=hierarchy)
    r = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    _check(oracle.nurbs_to_bezier_workload(wl), w, fl, min_cmp=0.99)


def test_nurbs_invalid_knots_rejected():
    wl = G.gen_nurbs(n_faces=3)
    bad = dict(wl)
    kn = wl["knots"].copy()
    kn[1] = 0.5            # first curve no longer clamped / non-decreasing
    bad["knots"] = kn
    with pytest.raises(wn.WNError) as e:
        wn.Faces.from_nurbs_workload(bad)
    assert e.value.status == 2


def test_spatial_regrouping_is_a_permutation(monkeypatch):
    """The in-kernel Morton regrouping of a unit's queries (random-order batch:
    it engages) permutes whole queries: results are bit-identical to the
    given order (crossing mode: integer sums)."""
    wl = G.gen_c2(n_queries=200_000)
    faces = wn.Faces.from_workload(wl)
    r1 = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    monkeypatch.setenv("WN_NO_SPATIAL", "1")
    r2 = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    faces.close()
    assert torch.equal(r1.flag, r2.flag)
    same = (r1.winding == r2.winding) | (torch.isnan(r1.winding) & torch.isnan(r2.winding))
    assert bool(same.all())


# ----------------------------------------------------------------------------
# degenerate geometry and large faces
# ----------------------------------------------------------------------------

def test_degenerate_segments_and_loops():
    """Zero-length segments (all control points equal), collinear control
    points, a closed loop of ONE segment (coincident end points: its root
    ellipse foci coincide), a two-segment lens, faces with no loops and a loop
    of degree-1 segments only: parity with the oracle, and the loop-free face
    is 0 everywhere."""
    rng = np.random.default_rng(11)
    c = np.array([0.5, 0.5])
    # square with a zero-length and a collinear cubic inserted on its edges
    sq = [(np.array([[0.2, 0.2], [0.8, 0.2]]), None),
          (np.array([[0.8, 0.2], [0.8, 0.2], [0.8, 0.2], [0.8, 0.2]]), None),       # zero length
          (np.array([[0.8, 0.2], [0.8, 0.4], [0.8, 0.6], [0.8, 0.8]]), None),       # collinear cubic
          (np.array([[0.8, 0.8], [0.2, 0.8]]), None),
          (np.array([[0.2, 0.8], [0.2, 0.2]]), None)]
    # one-segment closed loop (quintic teardrop), rational weights
    P = np.array([[0.5, 0.3], [0.9, 0.1], [0.9, 0.9], [0.1, 0.9], [0.1, 0.1], [0.5, 0.3]])
    drop = [(P, rng.uniform(0.5, 2.0, 6))]
    # two-segment lens
    lens = [(np.array([[0.3, 0.5], [0.5, 0.8], [0.7, 0.5]]), None), (np.array([[0.7, 0.5], [0.5, 0.2], [0.3, 0.5]]), None)]
    faces = [([sq], 0, (0, 1, 0, 1)), ([drop], 0, (0, 1, 0, 1)), ([lens], 0, (0, 1, 0, 1)), ([], 0, (0, 1, 0, 1))]
    nq = 4000
    q = rng.uniform(0, 1, size=(len(faces) * nq, 2))
    fid = np.repeat(np.arange(len(faces)), nq).astype(np.int32)
    wl = H.make_wl(faces, q, fid)
    w, fl = _gpu(wl)
    _check(wl, w, fl, min_cmp=0.99)
    assert np.all(w[fid == 3] == 0.0) and np.all(fl[fid == 3] == 0)


def test_large_face_multichunk():
    """One face whose record program spans many 32-KB shared-memory chunks
    (an 8,000-segment rational star loop plus 50 holes): staging chunk by
    chunk, hierarchy subtrees and skips that cross chunk boundaries."""
    rng = np.random.default_rng(12)
    from wn_workloads.configs import _star_segments, _star_vertices
    outer = _star_segments(rng, _star_vertices(rng, (0.5, 0.5), 0.42, 0.02, 8000, False),
                           rng.integers(1, 6, 8000), 0.05, True)
    loops = [outer]
    for k in range(50):
        cc = (0.2 + 0.6 * ((k % 10) + 0.5) / 10, 0.3 + 0.4 * ((k // 10) + 0.5) / 5)
        loops.append(_star_segments(rng, _star_vertices(rng, cc, 0.02, 0.002, 12, True),
                                    rng.integers(1, 6, 12), 0.05, True))
    q = rng.uniform(0.05, 0.95, size=(30_000, 2))
    wl = H.make_wl([(loops, 0, (0, 1, 0, 1))], q)
    faces = wn.Faces.from_workload(wl)
    assert faces.info()["max_face_records"] > 3 * 1024
    r = faces.query(wl["face_id"], wl["uv"])
    torch.cuda.synchronize()
    w, fl = r.winding.cpu().numpy(), r.flag.cpu().numpy()
    faces.close()
    idx = np.random.default_rng(0).choice(len(w), 3000, replace=False)
    _check(wl, w, fl, idx=idx, min_cmp=0.95)


def test_bucketing_runs_and_group_boundaries():
    """K4 (a3) on batches built to stress the histogram's 16-id groups: runs of
    a face's queries of length 1, 15, 16, 17, 31, 32, 33, 48 and 1,000+ placed
    at and off group boundaries, invalid ids (-1, n_faces) inside long runs and
    at group edges, a descending face id exactly at a group boundary after a
    long sorted prefix (the batch must be detected unsorted) and a repeated
    face after other faces.  Valid queries match the oracle; invalid ids are
    flagged 3."""
    wl = G.gen_c4(n_faces=40, q_per_face=200, n_deleted=4)
    rng = np.random.default_rng(21)
    pool = {f: np.nonzero(wl["face_id"] == f)[0] for f in range(40)}
    lens = [1, 15, 16, 17, 31, 32, 33, 48, 1024, 1040, 7, 16, 16, 64]
    fids, src = [], []
    for k, L in enumerate(lens):
        f = k % 40 if k != 9 else 3          # face 3 again after others
        fids.append(np.full(L, f, np.int32))
        src.append(rng.choice(pool[f], L))
    # a descending step exactly at a group boundary (prefix length is a multiple of 16)
    pre = sum(len(a) for a in fids)
    pad = (-pre) % 16
    fids.append(np.full(pad + 32, 39, np.int32))
    src.append(rng.choice(pool[39], pad + 32))
    fids.append(np.full(48, 2, np.int32))
    src.append(rng.choice(pool[2], 48))
    fid = np.concatenate(fids)
    idx = np.concatenate(src)
    assert (pre + pad + 32) % 16 == 0
    uv = wl["uv"][idx].copy()
    bad = [int(np.cumsum(lens)[8]) - 500, int(np.cumsum(lens)[8]) - 512, 0, len(fid) - 1, pre + pad + 16]
    fid[bad[0]] = -1
    fid[bad[1]] = 40
    fid[bad[2]] = 41
    fid[bad[3]] = -7
    fid[bad[4]] = 40
    w, fl = _gpu(wl, face_id=fid, uv=uv)
    assert np.all(fl[bad] == 3) and np.all(np.isnan(w[bad]))
    ok = np.ones(len(fid), bool)
    ok[bad] = False
    assert np.all(fl[ok] != 3)
    wl2 = dict(wl)
    wl2["face_id"], wl2["uv"] = fid[ok], uv[ok]
    _check(wl2, w[ok], fl[ok], min_cmp=0.95)
